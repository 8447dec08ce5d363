// Dependent-chain latency (clocks per op, one warp) of the FP64 operations a
// Jacobi rotation is built from: DFMA, division, sqrt, rsqrt, and one
// shuffle-add level of a warp reduction; plus __syncthreads at 640 threads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_latency.bin tools/fp64_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 4096;

__global__ void lat(double seed, double* out, long long* cyc) {
  double x = seed + threadIdx.x * 1e-3;
  long long t0, t1;
  // dfma
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = fma(x, 0.999999, 1e-7);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  // div
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = 1.0 / (x + 1.0);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = t1 - t0;
  // sqrt
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = sqrt(x + 1.0);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[2] = t1 - t0;
  // rsqrt
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = rsqrt(x + 1.0);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = t1 - t0;
  // shuffle + add (one reduction level)
  t0 = clock64();
  for (int i = 0; i < N; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = t1 - t0;
  out[threadIdx.x] = x;
}

__global__ void syncs(long long* cyc) {
  __shared__ int s;
  long long t0 = clock64();
  for (int i = 0; i < N; ++i) {
    if (threadIdx.x == 0) s = i;
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[5] = t1 - t0 + s * 0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaMallocManaged(&cyc, 8 * sizeof(long long));
  lat<<<1, 32>>>(0.5, out, cyc);
  syncs<<<1, 640>>>(cyc);
  cudaDeviceSynchronize();
  const char* names[] = {"dfma", "div", "sqrt", "rsqrt", "shfl+dadd", "syncthreads(640)"};
  for (int i = 0; i < 6; ++i) printf("%-18s %7.1f clk/op\n", names[i], (double)cyc[i] / N);
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
