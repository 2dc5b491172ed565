// residuals.cuh -- PDE residuals on output jets and their transposes (the
// reverse-pass seeds). Reference: residual_components (losses.cpp:26-75);
// ns_steady follows PAPER.md:785-789 (extension, absent from the reference).
//
// o[s*F + f] is output field f on stream s of the PDE's stream layout.
#pragma once
#include "jets.cuh"

namespace pnx {

enum Pde : int { PDE_ADVECTION = 0, PDE_ALLEN_CAHN = 1, PDE_BURGERS = 2, PDE_MAXWELL = 3, PDE_NS = 4, PDE_MAXWELL_EH = 5 };

template <int P> struct PdeTraits;
template <> struct PdeTraits<PDE_ADVECTION> { static constexpr int L = LAY_XT, F = 1, K = 1; };
template <> struct PdeTraits<PDE_ALLEN_CAHN> { static constexpr int L = LAY_AC, F = 1, K = 1; };
template <> struct PdeTraits<PDE_BURGERS> { static constexpr int L = LAY_XT, F = 1, K = 1; };
template <> struct PdeTraits<PDE_MAXWELL> { static constexpr int L = LAY_MX, F = 3, K = 3; };
template <> struct PdeTraits<PDE_NS> { static constexpr int L = LAY_NS, F = 3, K = 3; };
template <> struct PdeTraits<PDE_MAXWELL_EH> { static constexpr int L = LAY_MX, F = 3, K = 3; };

struct PdeConst {
    float c, eps, mu, inv_re;
};

// r[k] from output jets.
template <int P>
__device__ __forceinline__ void residual(const float* o, float* r, const PdeConst& pc) {
    constexpr int F = PdeTraits<P>::F;
#define O(s, f) o[(s) * F + (f)]
    if constexpr (P == PDE_ADVECTION) {  // u_t + c u_x   (losses.cpp:36-41)
        r[0] = O(2, 0) + pc.c * O(1, 0);
    } else if constexpr (P == PDE_ALLEN_CAHN) {  // u_t - 1e-4 u_xx + 5u^3 - 5u  (:42-50)
        const float u = O(0, 0);
        r[0] = (O(2, 0) - 1e-4f * O(3, 0)) + (5.0f * (u * (u * u)) - 5.0f * u);
    } else if constexpr (P == PDE_BURGERS) {  // u_t + u u_x  (:51-56)
        r[0] = O(2, 0) + O(0, 0) * O(1, 0);
    } else if constexpr (P == PDE_MAXWELL) {  // (:57-72) fields Ez,Hx,Hy; streams x,y,t
        r[0] = pc.eps * O(3, 0) - (O(1, 2) - O(2, 1));
        r[1] = pc.mu * O(3, 1) + O(2, 0);
        r[2] = pc.mu * O(3, 2) - O(1, 0);
    } else if constexpr (P == PDE_MAXWELL_EH) {  // TE (Ex, Ey, Hz): SURVEY 8(a) a10c, extension
        r[0] = pc.eps * O(3, 0) - O(2, 2);              // eps Ex_t = Hz_y
        r[1] = pc.eps * O(3, 1) + O(1, 2);              // eps Ey_t = -Hz_x
        r[2] = pc.mu * O(3, 2) - (O(2, 0) - O(1, 1));   // mu Hz_t = Ex_y - Ey_x
    } else {  // NS steady: fields u,v,p; streams u, _x, _y, _xx, _yy
        const float u = O(0, 0), v = O(0, 1);
        r[0] = O(1, 0) + O(2, 1);
        r[1] = u * O(1, 0) + v * O(2, 0) + O(1, 2) - pc.inv_re * (O(3, 0) + O(4, 0));
        r[2] = u * O(1, 1) + v * O(2, 1) + O(2, 2) - pc.inv_re * (O(3, 1) + O(4, 1));
    }
#undef O
}

// ob = (dr/do)^T rb
template <int P>
__device__ __forceinline__ void residual_seed(const float* o, const float* rb, float* ob,
                                              const PdeConst& pc) {
    constexpr int F = PdeTraits<P>::F;
    constexpr int S = Streams<PdeTraits<P>::L>::S;
#pragma unroll
    for (int i = 0; i < S * F; ++i) ob[i] = 0.0f;
#define O(s, f) o[(s) * F + (f)]
#define OB(s, f) ob[(s) * F + (f)]
    if constexpr (P == PDE_ADVECTION) {
        OB(2, 0) = rb[0];
        OB(1, 0) = pc.c * rb[0];
    } else if constexpr (P == PDE_ALLEN_CAHN) {
        const float u = O(0, 0);
        OB(2, 0) = rb[0];
        OB(3, 0) = -1e-4f * rb[0];
        OB(0, 0) = (15.0f * u * u - 5.0f) * rb[0];
    } else if constexpr (P == PDE_BURGERS) {
        OB(2, 0) = rb[0];
        OB(0, 0) = O(1, 0) * rb[0];
        OB(1, 0) = O(0, 0) * rb[0];
    } else if constexpr (P == PDE_MAXWELL) {
        OB(3, 0) += pc.eps * rb[0];
        OB(1, 2) += -rb[0];
        OB(2, 1) += rb[0];
        OB(3, 1) += pc.mu * rb[1];
        OB(2, 0) += rb[1];
        OB(3, 2) += pc.mu * rb[2];
        OB(1, 0) += -rb[2];
    } else if constexpr (P == PDE_MAXWELL_EH) {
        OB(3, 0) += pc.eps * rb[0];
        OB(2, 2) += -rb[0];
        OB(3, 1) += pc.eps * rb[1];
        OB(1, 2) += rb[1];
        OB(3, 2) += pc.mu * rb[2];
        OB(2, 0) += -rb[2];
        OB(1, 1) += rb[2];
    } else {
        const float u = O(0, 0), v = O(0, 1);
        const float ux = O(1, 0), uy = O(2, 0), vx = O(1, 1), vy = O(2, 1);
        const float rc = rb[0], ru = rb[1], rv = rb[2], ir = pc.inv_re;
        OB(1, 0) += rc + u * ru;
        OB(2, 1) += rc + v * rv;
        OB(0, 0) += ux * ru + vx * rv;
        OB(0, 1) += uy * ru + vy * rv;
        OB(2, 0) += v * ru;
        OB(1, 2) += ru;
        OB(3, 0) += -ir * ru;
        OB(4, 0) += -ir * ru;
        OB(1, 1) += u * rv;
        OB(2, 2) += rv;
        OB(3, 1) += -ir * rv;
        OB(4, 1) += -ir * rv;
    }
#undef O
#undef OB
}

}  // namespace pnx
