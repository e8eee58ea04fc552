// Dependent-chain latency probe for the fp64 / shuffle operations on the
// H2 PES iteration's critical path (DADD, DMUL, DFMA, SHFL of a double,
// sqrt, division, sincos).  One warp, clock64 around 256 dependent ops.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false lat_probe.cu
#include <cstdio>

constexpr int N = 256;

template <int K>
__global__ void probe(double x0, double* out, long long* cyc) {
  double x = x0 + threadIdx.x * 1e-3, y = 1.0000001;
  __syncwarp();
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) {
    if (K == 0) x = x + y;
    if (K == 1) x = x * y;
    if (K == 2) x = fma(x, y, 1e-9);
    if (K == 3) x = __shfl_xor_sync(0xffffffffu, x, 1);
    if (K == 4) x = sqrt(x) + 0.5;
    if (K == 5) x = 1.0 / x + 0.5;
    if (K == 6) {
      double s, c;
      sincos(x, &s, &c);
      x = s + c;
    }
    if (K == 7) x = __dsqrt_rn(x) + 0.5;
    if (K == 8) x = rsqrt(x) + 0.5;
    if (K == 9) x = __drcp_rn(x) + 0.5;
    if (K == 10) x = __shfl_sync(0xffffffffu, x, 0);
    if (K == 11) {
      float f = __shfl_xor_sync(0xffffffffu, (float)x, 1);
      x = f;
    }
    if (K == 12) x = x / (x + 1.0);
    if (K == 13) x = exp(-x) + 0.5;
    if (K == 14) x = erf(x) + 0.5;
    if (K == 15) x = 0.5 * sqrt(3.14159 / x) * erf(sqrt(x)) + 0.5;
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 32 * sizeof(double));
  cudaMallocManaged(&cyc, sizeof(long long));
  const char* names[] = {"DADD", "DMUL", "DFMA", "SHFL.f64 xor", "sqrt+add", "1/x+add", "sincos+add",
                         "__dsqrt_rn+add", "rsqrt+add", "__drcp_rn+add", "SHFL.f64 bcast", "SHFL.f32",
                         "x/(x+1)", "exp(-x)+add", "erf+add", "boys_f0-like"};
#define RUN(K)                                         \
  for (int rep = 0; rep < 2; ++rep) {                  \
    probe<K><<<1, 32>>>(1.3, out, cyc);                \
    cudaDeviceSynchronize();                           \
  }                                                    \
  printf("%-16s %7.1f cycles/op\n", names[K], (double)*cyc / N);
  RUN(0) RUN(1) RUN(2) RUN(3) RUN(4) RUN(5) RUN(6) RUN(7) RUN(8) RUN(9) RUN(10) RUN(11) RUN(12) RUN(13) RUN(14) RUN(15)
  // 16 warps on one SM: throughput-limited cost of the same chains
  double* out2;
  cudaMalloc(&out2, 512 * sizeof(double));
#define RUN512(K)                                      \
  for (int rep = 0; rep < 2; ++rep) {                  \
    probe<K><<<1, 512>>>(1.3, out2, cyc);              \
    cudaDeviceSynchronize();                           \
  }                                                    \
  printf("%-16s %7.1f cycles/op (512 threads)\n", names[K], (double)*cyc / N);
  RUN512(2) RUN512(5) RUN512(4) RUN512(13) RUN512(14) RUN512(15)
  return 0;
}
