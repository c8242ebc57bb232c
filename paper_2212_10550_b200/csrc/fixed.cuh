// fixed.cuh -- fixed-point gradient accumulation (deterministic mode, arfx_model_set_deterministic).
// A contribution c is rounded to the nearest multiple of 2^-46 (1.4e-14) and summed as
// int64: integer addition is exact and associative, so the sum does not depend on the
// order of the atomics that build it. |sums| must stay below 2^17, far above any SPEC-loss
// gradient. One conversion back to f32 per element when the sum is consumed.
#pragma once
#include <cuda_runtime.h>

namespace arfx {
constexpr float kFixScale = 70368744177664.0f;  // 2^46
constexpr double kFixInv = 1.0 / 70368744177664.0;

__device__ __forceinline__ long long f32_to_fix(float c) { return __float2ll_rn(c * kFixScale); }
__device__ __forceinline__ float fix_to_f32(long long a) {
  return __double2float_rn(__dmul_rn(__ll2double_rn(a), kFixInv));
}
}  // namespace arfx
