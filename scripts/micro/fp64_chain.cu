// Microbenchmark: latency of a dependent FP64 add chain (DMUL + DADD per
// step, as the exact-order kernels use), with operands from registers or
// from shared memory.  One warp; prints cycles per step.
#include <cstdio>

__global__ void chain_reg(double* out, int steps, double w, double e) {
  double acc = 0.0;
  long long t0 = clock64();
  for (int i = 0; i < steps; ++i) acc += (w + i) * e;
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = acc, out[1] = double(t1 - t0) / steps;
}

__global__ void chain_smem(double* out, int steps) {
  __shared__ double s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = 1.0 + i * 1e-3;
  __syncthreads();
  double acc = 0.0;
  long long t0 = clock64();
  for (int i = 0; i < steps; ++i) {
    const double w = s[(i * 7) & 1023], e = s[(i * 13 + threadIdx.x) & 1023];
    if (w != 0.0) acc += w * e;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = acc, out[1] = double(t1 - t0) / steps;
}

__global__ void indep_smem(double* out, int steps) {  // 8 independent chains per thread
  __shared__ double s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = 1.0 + i * 1e-3;
  __syncthreads();
  double a[8] = {0};
  long long t0 = clock64();
  for (int i = 0; i < steps; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] += s[(i * 7 + k) & 1023] * s[(i * 13 + k + threadIdx.x) & 1023];
  }
  long long t1 = clock64();
  double acc = 0;
  for (int k = 0; k < 8; ++k) acc += a[k];
  if (threadIdx.x == 0) out[0] = acc, out[1] = double(t1 - t0) / steps;
}

int main() {
  double* d;
  cudaMalloc(&d, 16);
  double h[2];
  for (int threads : {32, 576}) {
    chain_reg<<<1, threads>>>(d, 100000, 1.0, 1e-9);
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("threads %d  reg chain:   %.1f cycles/step\n", threads, h[1]);
    chain_smem<<<1, threads>>>(d, 100000);
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("threads %d  smem chain:  %.1f cycles/step\n", threads, h[1]);
    indep_smem<<<1, threads>>>(d, 20000);
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("threads %d  8 indep chains: %.1f cycles/step (8 steps each)\n", threads, h[1]);
  }
  return 0;
}
