// peaks.cu -- measured pipe roofs for the kernels MEASURED_PEAKS.json has no denominator
// for: the deformer and march are FP64 add/mul issue-bound (explicit __dadd_rn /
// __dmul_rn, no FMA -- bit-exactness forbids contraction), the exact MLP is FP32
// add/mul issue-bound. Each thread runs 8 independent dependent chains of
// x = x*a + b as separate mul + add (2 flops), enough ILP to saturate the pipe.
#include <cuda_runtime.h>

#include "model.h"

namespace arfx {
namespace {

__global__ void fp64_peak_kernel(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = __dadd_rn(__dmul_rn(x[k], a), b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

__global__ void fp32_peak_kernel(float* out, int iters, float a, float b) {
  float x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3f + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = __fadd_rn(__fmul_rn(x[k], a), b);
  }
  float s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678f) out[0] = s;
}

}  // namespace

// returns TFLOP/s counting each add and each mul as one flop
void measure_pipe_peaks(double* fp64_tflops, double* fp32_tflops) {
  int dev = 0, sms = 148;
  ARFX_CUDA(cudaGetDevice(&dev));
  ARFX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  DevBuf<double> o64;
  DevBuf<float> o32;
  o64.alloc(1);
  o32.alloc(1);
  cudaEvent_t e0, e1;
  ARFX_CUDA(cudaEventCreate(&e0));
  ARFX_CUDA(cudaEventCreate(&e1));
  const int threads = 256, blocks = sms * 8;
  const int it64 = 4096, it32 = 16384;
  float best64 = 1e30f, best32 = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    ARFX_CUDA(cudaEventRecord(e0));
    fp64_peak_kernel<<<blocks, threads>>>(o64.ptr, it64, 0.999999, 1e-7);
    ARFX_CUDA(cudaEventRecord(e1));
    ARFX_CUDA(cudaEventSynchronize(e1));
    float ms;
    ARFX_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    if (rep) best64 = ms < best64 ? ms : best64;
    ARFX_CUDA(cudaEventRecord(e0));
    fp32_peak_kernel<<<blocks, threads>>>(o32.ptr, it32, 0.999999f, 1e-7f);
    ARFX_CUDA(cudaEventRecord(e1));
    ARFX_CUDA(cudaEventSynchronize(e1));
    ARFX_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    if (rep) best32 = ms < best32 ? ms : best32;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const double thr = static_cast<double>(blocks) * threads;
  *fp64_tflops = thr * it64 * 8 * 2 / (best64 * 1e-3) / 1e12;
  *fp32_tflops = thr * it32 * 8 * 2 / (best32 * 1e-3) / 1e12;
}

}  // namespace arfx
