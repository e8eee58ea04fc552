// Probe: FP64 throughput of mma.sync.m8n8k4.f64 (DMMA) vs DFMA on this GPU.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/dmma_probe.cu -o /tmp/dmma_probe
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dmma(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[4][2] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(c[j][0]), "+d"(c[j][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dfma(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) c[j] = fma(a, b, c[j]);
  }
  double s = 0;
  for (int j = 0; j < 8; ++j) s += c[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 148 * 8 * 1024 * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    for (int warps : {4, 8, 16, 32}) {
      const int blocks = 148 * 4, threads = warps * 32 / 4;
      cudaEventRecord(e0);
      k_dmma<<<blocks, threads>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double fl_mma = 2.0 * 256 * 4 * (double)iters * blocks * (threads / 32);
      cudaEventRecord(e0);
      k_dfma<<<blocks, threads>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms2;
      cudaEventElapsedTime(&ms2, e0, e1);
      const double fl_fma = 2.0 * 8 * (double)iters * blocks * threads;
      if (rep) printf("warps/SM %2d: DMMA %.1f TFLOP/s   DFMA %.1f TFLOP/s\n", warps, fl_mma / ms * 1e-9, fl_fma / ms2 * 1e-9);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
