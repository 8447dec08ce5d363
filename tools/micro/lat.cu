// Dependent-chain latencies of the FP64 / shuffle / shared-memory / barrier
// operations the one-CTA small kernels are built from (clock64, one warp;
// the barrier with 5 and 20 warps). nvcc -arch=sm_100a -o lat lat.cu
#include <cstdio>

__global__ void lat(double* out, double seed, int n) {
  __shared__ double sm[1024];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double x = seed + threadIdx.x * 1e-9;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 1.0 + i * 1e-12;
  __syncthreads();
  long long t0, t1;
  double r = 0.0;
#define CHAIN(name, expr)                                                       \
  t0 = clock64();                                                               \
  for (int i = 0; i < n; ++i) { expr; }                                         \
  t1 = clock64();                                                               \
  if (threadIdx.x == 0) printf("%-10s %6.1f cycles\n", name, (double)(t1 - t0) / n); \
  r += x;
  if (warp == 0) {
    CHAIN("dfma", x = fma(x, 1.0000001, 1e-9))
    CHAIN("dadd", x = x + 1e-9)
    CHAIN("ddiv", x = 1.0 / (x + 1.0))
    CHAIN("dsqrt", x = sqrt(x + 1.0))
    CHAIN("drsqrt", x = rsqrt(x + 1.0))
    CHAIN("shfl64", x = __shfl_xor_sync(0xffffffffu, x, 1) + 1e-9)
    CHAIN("lds64", x = sm[((int)(x * 1e-3) & 7) + lane] + x * 1e-20)
  }
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  t1 = clock64();
  if (threadIdx.x == 0) printf("bar(%d warps) %6.1f cycles\n", blockDim.x / 32, (double)(t1 - t0) / n);
  if (threadIdx.x == 0) out[0] = r;
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// DMMA m8n8k4: dependent-chain latency (one chain) and issue interval with
// NC independent chains per warp, W warps per SM sub-partition
template <int NC>
__global__ void dmma_lat(double* out, int n) {
  double c[NC][2];
  for (int k = 0; k < NC; ++k) c[k][0] = c[k][1] = threadIdx.x * 1e-9;
  const double a = 1.0000001, b = 0.9999999;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < NC; ++k) dmma(c[k][0], c[k][1], a, b);
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0)
    printf("dmma NC=%2d warps=%2d: %6.1f cycles per DMMA per warp (%6.1f per chain step)\n", NC,
           blockDim.x / 32, (double)(t1 - t0) / (n * NC), (double)(t1 - t0) / n);
  double s = 0;
  for (int k = 0; k < NC; ++k) s += c[k][0] + c[k][1];
  out[threadIdx.x] = s;
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  lat<<<1, 32>>>(d, 0.5, 1000);
  cudaDeviceSynchronize();
  lat<<<1, 160>>>(d, 0.5, 1000);
  cudaDeviceSynchronize();
  lat<<<1, 640>>>(d, 0.5, 1000);
  cudaDeviceSynchronize();
  double* o;
  cudaMalloc(&o, 1024 * 8);
  for (int w : {1, 4, 8, 16}) {
    dmma_lat<1><<<1, 32 * w>>>(o, 1000);
    cudaDeviceSynchronize();
    dmma_lat<3><<<1, 32 * w>>>(o, 1000);
    cudaDeviceSynchronize();
    dmma_lat<6><<<1, 32 * w>>>(o, 1000);
    cudaDeviceSynchronize();
    dmma_lat<12><<<1, 32 * w>>>(o, 1000);
    cudaDeviceSynchronize();
  }
  return 0;
}
