// Microbenchmark: legacy warp-level mma.sync TF32 (m16n8k8) and BF16 (m16n8k16) throughput on B200.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void tf32_kernel(float* out, int iters) {
  unsigned a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 + 5, b1 = a0 + 7;
  float c[4][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+f"(c[u][0]), "+f"(c[u][1]), "+f"(c[u][2]), "+f"(c[u][3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
  }
  float s = 0; for (int u = 0; u < 4; ++u) for (int v = 0; v < 4; ++v) s += c[u][v];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void bf16_kernel(float* out, int iters) {
  unsigned a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 + 5, b1 = a0 + 7;
  float c[4][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+f"(c[u][0]), "+f"(c[u][1]), "+f"(c[u][2]), "+f"(c[u][3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
  }
  float s = 0; for (int u = 0; u < 4; ++u) for (int v = 0; v < 4; ++v) s += c[u][v];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int blocks = 148 * 8, threads = 256, iters = 4000;
  float* out; cudaMalloc(&out, blocks * threads * sizeof(float));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); tf32_kernel<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 16 * 8 * 8 * (blocks * threads / 32.0) * iters * 4;
    printf("mma.sync TF32 m16n8k8: %.1f TFLOP/s\n", fl / ms / 1e9);
    cudaEventRecord(e0); bf16_kernel<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 16 * 8 * 16 * (blocks * threads / 32.0) * iters * 4;
    printf("mma.sync BF16 m16n8k16: %.1f TFLOP/s\n", fl / ms / 1e9);
  }
  return 0;
}
