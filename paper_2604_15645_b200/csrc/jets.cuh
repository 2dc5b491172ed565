// jets.cuh -- compile-time Taylor-stream layouts and the per-element jet rules
// (forward + transpose) for the activations of the reference model
// (model.cpp:168-174: tanh, sin(w0 z), z*sigmoid(z)).
//
// A "stream" is one Taylor coefficient carried through the network per point:
// the value, d/dx_a (order 1) or d2/dx_a^2 (order 2). Which streams a PDE needs
// mirrors the derivative_wrt_input calls of residual_components
// (losses.cpp:36-72). Layouts are compile-time so every stream index folds into
// registers.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace pnx {

// Stream layouts. order: 0 value, 1 first, 2 pure second; axis: coordinate
// index; partner: index of the first-order stream of the same axis (order 2).
enum Layout : int {
    LAY_V = 0,    // {u}                                    (IC/BC only)
    LAY_XT = 1,   // {u, u_0, u_1}                          advection, burgers
    LAY_AC = 2,   // {u, u_0, u_1, u_00}                    allen-cahn
    LAY_MX = 3,   // {u, u_0, u_1, u_2}                     maxwell TE (x, y, t)
    LAY_NS = 4,   // {u, u_0, u_1, u_00, u_11}              steady NS (x, y)
};

template <int L> struct Streams;
template <> struct Streams<LAY_V> {
    static constexpr int S = 1;
    __host__ __device__ static constexpr int order(int) { return 0; }
    __host__ __device__ static constexpr int axis(int) { return -1; }
    __host__ __device__ static constexpr int partner(int) { return -1; }
};
template <> struct Streams<LAY_XT> {
    static constexpr int S = 3;
    __host__ __device__ static constexpr int order(int s) { return s == 0 ? 0 : 1; }
    __host__ __device__ static constexpr int axis(int s) { return s - 1; }
    __host__ __device__ static constexpr int partner(int) { return -1; }
};
template <> struct Streams<LAY_AC> {
    static constexpr int S = 4;
    __host__ __device__ static constexpr int order(int s) { return s == 0 ? 0 : (s == 3 ? 2 : 1); }
    __host__ __device__ static constexpr int axis(int s) { return s == 0 ? -1 : (s == 3 ? 0 : s - 1); }
    __host__ __device__ static constexpr int partner(int s) { return s == 3 ? 1 : -1; }
};
template <> struct Streams<LAY_MX> {
    static constexpr int S = 4;
    __host__ __device__ static constexpr int order(int s) { return s == 0 ? 0 : 1; }
    __host__ __device__ static constexpr int axis(int s) { return s - 1; }
    __host__ __device__ static constexpr int partner(int) { return -1; }
};
template <> struct Streams<LAY_NS> {
    static constexpr int S = 5;
    __host__ __device__ static constexpr int order(int s) { return s == 0 ? 0 : (s >= 3 ? 2 : 1); }
    __host__ __device__ static constexpr int axis(int s) { return s == 0 ? -1 : (s >= 3 ? s - 3 : s - 1); }
    __host__ __device__ static constexpr int partner(int s) { return s == 3 ? 1 : (s == 4 ? 2 : -1); }
};

enum Act : int { ACT_TANH = 0, ACT_SINE = 1, ACT_SWISH = 2, ACT_NONE = 3 };

// Storage convention of a hidden layer's jets Z[s]: for tanh layers the value
// stream holds t = tanh(z0) (applied once, in the producing epilogue), the
// other streams hold the pre-activation jets z_a, z_aa. Every consumer (next
// layer's prologue, the reverse epilogue, the weight gradient, the head) needs
// exactly t and z_a, z_aa. sine/swish layers store z0 itself.
template <int ACT>
__device__ __forceinline__ float store_value(float z0) {
    if constexpr (ACT == ACT_TANH) return tanhf(z0);
    return z0;
}

// h = act(z) on all S streams of one (point, feature) element.
template <int L, int ACT>
__device__ __forceinline__ void act_fwd(const float* z, float* h, float w0) {
    using St = Streams<L>;
    constexpr int S = St::S;
    if constexpr (ACT == ACT_NONE) {
#pragma unroll
        for (int s = 0; s < S; ++s) h[s] = z[s];
    } else if constexpr (ACT == ACT_TANH) {
        const float t = z[0];  // stored as tanh(z0)
        const float d = 1.0f - t * t;
        h[0] = t;
#pragma unroll
        for (int s = 1; s < S; ++s) {
            if (St::order(s) == 1) {
                h[s] = d * z[s];
            } else {
                const float za = z[St::partner(s)];
                h[s] = d * (z[s] - 2.0f * t * za * za);
            }
        }
    } else if constexpr (ACT == ACT_SINE) {
        float sn, cs;
        sincosf(w0 * z[0], &sn, &cs);
        h[0] = sn;
#pragma unroll
        for (int s = 1; s < S; ++s) {
            if (St::order(s) == 1) {
                h[s] = w0 * cs * z[s];
            } else {
                const float za = z[St::partner(s)];
                h[s] = w0 * cs * z[s] - w0 * w0 * sn * za * za;
            }
        }
    } else {  // swish
        const float z0 = z[0];
        const float q = 1.0f / (1.0f + expf(-z0));
        const float sp = q * (1.0f - q);
        const float f1 = q + z0 * sp;
        const float f2 = sp * (2.0f + z0 * (1.0f - 2.0f * q));
        h[0] = z0 * q;
#pragma unroll
        for (int s = 1; s < S; ++s) {
            if (St::order(s) == 1) {
                h[s] = f1 * z[s];
            } else {
                const float za = z[St::partner(s)];
                h[s] = f1 * z[s] + f2 * za * za;
            }
        }
    }
}

// zbar = (d act / d z)^T hbar on all streams of one element (transpose of act_fwd).
template <int L, int ACT>
__device__ __forceinline__ void act_bwd(const float* z, const float* hb, float* zb, float w0) {
    using St = Streams<L>;
    constexpr int S = St::S;
    if constexpr (ACT == ACT_NONE) {
#pragma unroll
        for (int s = 0; s < S; ++s) zb[s] = hb[s];
    } else if constexpr (ACT == ACT_TANH) {
        const float t = z[0];  // stored as tanh(z0)
        const float d = 1.0f - t * t;
        float tbar = hb[0], dbar = 0.0f;
#pragma unroll
        for (int s = 1; s < S; ++s) zb[s] = 0.0f;
#pragma unroll
        for (int s = 1; s < S; ++s) {
            if (St::order(s) == 1) {
                zb[s] += d * hb[s];
                dbar += z[s] * hb[s];
            } else {
                const int p = St::partner(s);
                const float za = z[p], zaa = z[s];
                zb[s] += d * hb[s];
                zb[p] += -4.0f * t * d * za * hb[s];
                dbar += (zaa - 2.0f * t * za * za) * hb[s];
                tbar += -2.0f * d * za * za * hb[s];
            }
        }
        tbar += -2.0f * t * dbar;
        zb[0] = d * tbar;
    } else if constexpr (ACT == ACT_SINE) {
        float sn, cs;
        sincosf(w0 * z[0], &sn, &cs);
        float sbar = hb[0], cbar = 0.0f;
#pragma unroll
        for (int s = 1; s < S; ++s) zb[s] = 0.0f;
#pragma unroll
        for (int s = 1; s < S; ++s) {
            if (St::order(s) == 1) {
                zb[s] += w0 * cs * hb[s];
                cbar += w0 * z[s] * hb[s];
            } else {
                const int p = St::partner(s);
                const float za = z[p], zaa = z[s];
                zb[s] += w0 * cs * hb[s];
                cbar += w0 * zaa * hb[s];
                zb[p] += -2.0f * w0 * w0 * sn * za * hb[s];
                sbar += -w0 * w0 * za * za * hb[s];
            }
        }
        zb[0] = w0 * cs * sbar - w0 * sn * cbar;
    } else {  // swish
        const float z0 = z[0];
        const float q = 1.0f / (1.0f + expf(-z0));
        const float sp = q * (1.0f - q);
        const float spp = sp * (1.0f - 2.0f * q);
        const float sppp = spp * (1.0f - 2.0f * q) - 2.0f * sp * sp;
        const float f1 = q + z0 * sp;
        const float f2 = 2.0f * sp + z0 * spp;
        const float f3 = 3.0f * spp + z0 * sppp;
        float f1bar = 0.0f, f2bar = 0.0f;
#pragma unroll
        for (int s = 1; s < S; ++s) zb[s] = 0.0f;
#pragma unroll
        for (int s = 1; s < S; ++s) {
            if (St::order(s) == 1) {
                zb[s] += f1 * hb[s];
                f1bar += z[s] * hb[s];
            } else {
                const int p = St::partner(s);
                const float za = z[p], zaa = z[s];
                zb[s] += f1 * hb[s];
                f1bar += zaa * hb[s];
                zb[p] += 2.0f * f2 * za * hb[s];
                f2bar += za * za * hb[s];
            }
        }
        zb[0] = hb[0] * f1 + f1bar * f2 + f2bar * f3;
    }
}

}  // namespace pnx
