// Checks the assumed register-fragment layouts of the FP64 mma.sync shapes
// m16n8k8 and m16n8k16 on sm_100a against a host matmul.
//   g = lane >> 2, t = lane & 3
//   A (16 x K, row): a[i] = A[g + 8 (i & 1)][t + 4 (i >> 1)]
//   B (K x 8, col):  b[i] = B[t + 4 i][g]
//   C (16 x 8):      c[0..1] = C[g][2t .. 2t+1], c[2..3] = C[g + 8][2t .. 2t+1]
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_layout_check.bin tools/mma_layout_check.cu
#include <cmath>
#include <cstdio>
#include <cuda_runtime.h>

template <int K>
__global__ void kern(const double* A, const double* B, double* C) {
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double a[K / 2], b[K / 4], c[4] = {0, 0, 0, 0};
  for (int i = 0; i < K / 2; ++i) a[i] = A[(g + 8 * (i & 1)) * K + t + 4 * (i >> 1)];
  for (int i = 0; i < K / 4; ++i) b[i] = B[(t + 4 * i) * 8 + g];
  if constexpr (K == 8) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};\n"
        : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
        : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
  } else {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
        "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
        : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
        : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]),
          "d"(a[7]), "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  C[g * 8 + 2 * t] = c[0];
  C[g * 8 + 2 * t + 1] = c[1];
  C[(g + 8) * 8 + 2 * t] = c[2];
  C[(g + 8) * 8 + 2 * t + 1] = c[3];
}

template <int K>
int check() {
  double hA[16 * K], hB[K * 8], hC[128], ref[128];
  for (int i = 0; i < 16 * K; ++i) hA[i] = std::sin(1.0 + i);
  for (int i = 0; i < K * 8; ++i) hB[i] = std::cos(2.0 + 3 * i);
  for (int m = 0; m < 16; ++m)
    for (int n = 0; n < 8; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += hA[m * K + k] * hB[k * 8 + n];
      ref[m * 8 + n] = s;
    }
  double *dA, *dB, *dC;
  cudaMalloc(&dA, sizeof hA);
  cudaMalloc(&dB, sizeof hB);
  cudaMalloc(&dC, sizeof hC);
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  kern<K><<<1, 32>>>(dA, dB, dC);
  cudaMemcpy(hC, dC, sizeof hC, cudaMemcpyDeviceToHost);
  double err = 0;
  for (int i = 0; i < 128; ++i) err = std::fmax(err, std::fabs(hC[i] - ref[i]));
  printf("m16n8k%d max |err| = %.3e %s\n", K, err, err < 1e-12 ? "OK" : "MISMATCH");
  return err < 1e-12 ? 0 : 1;
}

int main() {
  int bad = check<8>() + check<16>();
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return bad;
}
