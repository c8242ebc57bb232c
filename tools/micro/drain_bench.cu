// Microbenchmark: deterministic-gradient drain variants over an 8.4M-row fixed-point
// accumulator (config-1 hash grid: 16 levels x 2^19 rows x 2 features).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/drain_bench tools/micro/drain_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void drain_bitmap(long long n_words, uint32_t* touched, long long* acc, float* grad) {
  const int lane = threadIdx.x & 31;
  for (long long wi = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; wi < n_words;
       wi += (static_cast<long long>(gridDim.x) * blockDim.x) >> 5) {
    const uint32_t bits = touched[wi];
    if (!bits) continue;
    __syncwarp();
    if (lane == 0) touched[wi] = 0;
    if (!((bits >> lane) & 1u)) continue;
    const size_t row = static_cast<size_t>(wi) * 32 + lane;
    const longlong2 a = reinterpret_cast<const longlong2*>(acc)[row];
    reinterpret_cast<longlong2*>(acc)[row] = make_longlong2(0, 0);
    float2 g = reinterpret_cast<float2*>(grad)[row];
    g.x += static_cast<float>(static_cast<double>(a.x) * 1.4210854715202004e-14);
    g.y += static_cast<float>(static_cast<double>(a.y) * 1.4210854715202004e-14);
    reinterpret_cast<float2*>(grad)[row] = g;
  }
}

__global__ void drain_sweep(long long rows, long long* acc, float* grad) {
  for (long long row = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; row < rows;
       row += static_cast<long long>(gridDim.x) * blockDim.x) {
    const longlong2 a = reinterpret_cast<const longlong2*>(acc)[row];
    if ((a.x | a.y) == 0) continue;
    reinterpret_cast<longlong2*>(acc)[row] = make_longlong2(0, 0);
    float2 g = reinterpret_cast<float2*>(grad)[row];
    g.x += static_cast<float>(static_cast<double>(a.x) * 1.4210854715202004e-14);
    g.y += static_cast<float>(static_cast<double>(a.y) * 1.4210854715202004e-14);
    reinterpret_cast<float2*>(grad)[row] = g;
  }
}

__global__ void fill(long long rows, long long* acc, uint32_t* touched, int every) {
  for (long long row = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; row < rows;
       row += static_cast<long long>(gridDim.x) * blockDim.x) {
    const bool t = (row * 2654435761ull >> 7) % every == 0;
    acc[2 * row] = t ? 12345 : 0;
    acc[2 * row + 1] = t ? -777 : 0;
    if (t) atomicOr(touched + (row >> 5), 1u << (row & 31));
  }
}

int main() {
  const long long rows = 16LL << 19, words = rows / 32;
  long long* acc;
  float* grad;
  uint32_t* touched;
  cudaMalloc(&acc, rows * 16);
  cudaMalloc(&grad, rows * 8);
  cudaMalloc(&touched, words * 4);
  cudaMemset(grad, 0, rows * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int every : {1, 2, 8, 64}) {
    for (int v = 0; v < 4; ++v) {
      cudaMemset(touched, 0, words * 4);
      fill<<<148 * 16, 256>>>(rows, acc, touched, every);
      cudaDeviceSynchronize();
      cudaEventRecord(e0);
      if (v == 0) drain_bitmap<<<(words + 7) / 8, 256>>>(words, touched, acc, grad);
      if (v == 1) drain_bitmap<<<148 * 16, 256>>>(words, touched, acc, grad);
      if (v == 2) drain_sweep<<<(rows + 255) / 256, 256>>>(rows, acc, grad);
      if (v == 3) drain_sweep<<<148 * 16, 256>>>(rows, acc, grad);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("touched 1/%d variant %d: %.1f us\n", every, v, ms * 1e3);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
