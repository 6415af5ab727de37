// FP64 tensor-core (DMMA) and FP64 FMA issue peaks on one B200, measured:
// every warp runs independent mma.sync.m8n8k4.f64 (or DFMA) chains from
// registers only.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 dmma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
  double acc[8][2];
  for (int q = 0; q < 8; ++q) acc[q][0] = acc[q][1] = 0.0;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                   : "+d"(acc[q][0]), "+d"(acc[q][1]) : "d"(a), "d"(b));
  }
  double s = 0.0;
  for (int q = 0; q < 8; ++q) s += acc[q][0] + acc[q][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double acc[8];
  for (int q = 0; q < 8; ++q) acc[q] = q;
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = fma(acc[q], a, b);
  }
  double s = 0.0;
  for (int q = 0; q < 8; ++q) s += acc[q];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int warps = 4; warps <= 16; warps *= 2) {
    const dim3 grid(sms * 2), block(32 * warps);
    dmma_loop<<<grid, block>>>(d, 100);
    cudaEventRecord(e0);
    dmma_loop<<<grid, block>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * grid.x * warps;
    std::printf("{\"kernel\": \"dmma m8n8k4\", \"warps_per_cta\": %d, \"tflops\": %.2f}\n", warps,
                flops / (ms * 1e-3) / 1e12);
    dfma_loop<<<grid, block>>>(d, 100);
    cudaEventRecord(e0);
    dfma_loop<<<grid, block>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double f2 = 2.0 * 8.0 * iters * grid.x * block.x;
    std::printf("{\"kernel\": \"dfma\", \"warps_per_cta\": %d, \"tflops\": %.2f}\n", warps, f2 / (ms * 1e-3) / 1e12);
  }
  return 0;
}
