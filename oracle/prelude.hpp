// Force-included (g++ -include) into every reference translation unit when
// building the CPU oracle in oracle/_ref. TEST INFRASTRUCTURE ONLY.
//
// The shipped reference does not compile as-is: trainer.cpp:507 and :510 call
// `apply_update` before its definition at trainer.cpp:643, and no header
// declares it. This prelude supplies the missing declaration without editing
// the read-only sources. Nothing else is changed.
#pragma once
#include "pinnlab/trainer.hpp"

namespace pinnlab {
void apply_update(Adam& adam, const ExponentialLr& sched, long epoch, Model& model,
                  std::vector<Model>& replicas, const std::vector<Tensor>& grads,
                  const TrainConfig& cfg, TrainResult& result);
}  // namespace pinnlab
