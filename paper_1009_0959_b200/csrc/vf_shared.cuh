// vf_shared.cuh -- cross-window pair sharing for the angular criterion
// (SURVEY.md 8(f1)).  Placeholder: not yet applicable (returns -100 so the
// per-window kernel runs).
#pragma once
#include <cuda_runtime.h>

#include "vf_window.cuh"

namespace vf {

inline int launch_shared(const Launch&, int, int, int, cudaStream_t) { return -100; }

}  // namespace vf
