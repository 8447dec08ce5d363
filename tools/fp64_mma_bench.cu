// Throughput probe for the FP64 tensor-core shapes on sm_100a: m8n8k4,
// m16n8k4, m16n8k8, m16n8k16 (mma.sync), and plain DFMA, each with ILP
// independent accumulator chains per warp. Prints TFLOP/s per variant.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_mma_bench fp64_mma_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

template <int ILP>
__global__ void k884(double* out, double seed) {
  double acc[ILP][2];
  for (int i = 0; i < ILP; ++i) acc[i][0] = acc[i][1] = 0.0;
  double a = seed + threadIdx.x, b = seed * 0.5;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i)
      asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
          : "+d"(acc[i][0]), "+d"(acc[i][1])
          : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < ILP; ++i) s += acc[i][0] + acc[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int ILP>
__global__ void k1684(double* out, double seed) {
  double acc[ILP][4];
  for (int i = 0; i < ILP; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.0;
  double a0 = seed + threadIdx.x, a1 = seed * 2, b = seed * 0.5;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i)
      asm("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
          "{%0,%1,%2,%3};\n"
          : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3])
          : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < ILP; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int ILP>
__global__ void k1688(double* out, double seed) {
  double acc[ILP][4];
  for (int i = 0; i < ILP; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.0;
  double a0 = seed + threadIdx.x, a1 = seed * 2, a2 = seed * 3, a3 = seed * 4, b0 = seed * 0.5,
         b1 = seed * 0.25;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i)
      asm("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
          "{%8,%9}, {%0,%1,%2,%3};\n"
          : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3])
          : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
  }
  double s = 0;
  for (int i = 0; i < ILP; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int ILP>
__global__ void k16816(double* out, double seed) {
  double acc[ILP][4];
  for (int i = 0; i < ILP; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.0;
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = seed * (i + 1) + threadIdx.x;
  for (int i = 0; i < 4; ++i) b[i] = seed * 0.5 * (i + 1);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i)
      asm("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
          "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
          : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3])
          : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]),
            "d"(a[7]), "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
  for (int i = 0; i < ILP; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int ILP>
__global__ void kdfma(double* out, double seed) {
  double acc[ILP];
  for (int i = 0; i < ILP; ++i) acc[i] = seed * i;
  const double a = seed + threadIdx.x, b = 0.999999;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] = fma(acc[i], b, a);
  }
  double s = 0;
  for (int i = 0; i < ILP; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <class K>
void run(const char* name, K kern, double flop_per_warp_iter, int warps_per_block, double* d,
         int blocks_per_sm = 2) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * blocks_per_sm;
  kern<<<blocks, 32 * warps_per_block>>>(d, 1.0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) kern<<<blocks, 32 * warps_per_block>>>(d, 1.0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 5.0 * blocks * warps_per_block * (double)ITERS * flop_per_warp_iter;
  printf("%-28s warps/blk=%2d blk/SM=%d  %8.2f TFLOP/s\n", name, warps_per_block, blocks_per_sm,
         flops / (ms * 1e-3) / 1e12);
}

int main() {
  double* d;
  cudaMalloc(&d, 1 << 24);
  for (int w : {4, 8, 16}) {
    run("m8n8k4 ilp4", k884<4>, 4 * 512.0, w, d);
    run("m8n8k4 ilp8", k884<8>, 8 * 512.0, w, d);
    run("m16n8k4 ilp4", k1684<4>, 4 * 1024.0, w, d);
    run("m16n8k8 ilp4", k1688<4>, 4 * 2048.0, w, d);
    run("m16n8k16 ilp4", k16816<4>, 4 * 4096.0, w, d);
    run("dfma ilp8", kdfma<8>, 8 * 64.0, w, d);
  }
  // one warp per SM sub-partition (4 warps per SM) vs two
  run("m8n8k4 ilp1 1w/SMSP", k884<1>, 1 * 512.0, 4, d, 1);
  run("m8n8k4 ilp2 1w/SMSP", k884<2>, 2 * 512.0, 4, d, 1);
  run("m8n8k4 ilp3 1w/SMSP", k884<3>, 3 * 512.0, 4, d, 1);
  run("m8n8k4 ilp4 1w/SMSP", k884<4>, 4 * 512.0, 4, d, 1);
  run("m8n8k4 ilp6 1w/SMSP", k884<6>, 6 * 512.0, 4, d, 1);
  run("m8n8k4 ilp1 2w/SMSP", k884<1>, 1 * 512.0, 8, d, 1);
  run("m8n8k4 ilp2 2w/SMSP", k884<2>, 2 * 512.0, 8, d, 1);
  run("m8n8k4 ilp3 2w/SMSP", k884<3>, 3 * 512.0, 8, d, 1);
  run("m16n8k4 ilp1 1w/SMSP", k1684<1>, 1 * 1024.0, 4, d, 1);
  run("m16n8k4 ilp2 1w/SMSP", k1684<2>, 2 * 1024.0, 4, d, 1);
  run("m16n8k8 ilp1 1w/SMSP", k1688<1>, 1 * 2048.0, 4, d, 1);
  run("m16n8k8 ilp2 1w/SMSP", k1688<2>, 2 * 2048.0, 4, d, 1);
  run("m16n8k16 ilp1 1w/SMSP", k16816<1>, 1 * 4096.0, 4, d, 1);
  run("m16n8k16 ilp2 1w/SMSP", k16816<2>, 2 * 4096.0, 4, d, 1);
  run("m16n8k16 ilp1 2w/SMSP", k16816<1>, 1 * 4096.0, 8, d, 1);
  run("m8n8k4 ilp8 1w/SMSP", k884<8>, 8 * 512.0, 4, d, 1);
  run("m8n8k4 ilp12 1w/SMSP", k884<12>, 12 * 512.0, 4, d, 1);
  run("m8n8k4 ilp4 2w/SMSP", k884<4>, 4 * 512.0, 8, d, 1);
  run("m16n8k8 ilp4 1w/SMSP", k1688<4>, 4 * 2048.0, 4, d, 1);
  run("m16n8k16 ilp4 1w/SMSP", k16816<4>, 4 * 4096.0, 4, d, 1);
  run("dfma ilp8 1w/SMSP", kdfma<8>, 8 * 64.0, 4, d, 1);
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
