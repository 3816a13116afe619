// Microbenchmark: legacy warp-level mma.sync throughput on sm_100a (TF32
// m16n8k8 and BF16 m16n8k16, FP32 accumulate), register operands only.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_sync_bench tools/mma_sync_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <bool kTf32>
__global__ void mma_loop(float* out, int iters) {
  uint32_t a0 = threadIdx.x, a1 = a0 * 3u, a2 = a0 * 5u, a3 = a0 * 7u, b0 = a0 * 11u, b1 = a0 * 13u;
  float d[4][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {   // 4 independent accumulators
      if (kTf32)
        asm volatile(
            "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
            "{%0,%1,%2,%3};"
            : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3])
            : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      else
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
            "{%0,%1,%2,%3};"
            : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3])
            : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
  }
  float s = 0.f;
  for (int j = 0; j < 4; ++j) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, sizeof(float) * sms * 8 * 1024);
  const int iters = 4096;
  for (int tf = 1; tf >= 0; --tf) {
    for (int warps : {4, 8, 16}) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      const int grid = sms * 2;
      float best = 1e9;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        if (tf) mma_loop<true><<<grid, 32 * warps>>>(out, iters);
        else mma_loop<false><<<grid, 32 * warps>>>(out, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      const double flop_per = tf ? 2.0 * 16 * 8 * 8 : 2.0 * 16 * 8 * 16;
      const double flops = double(grid) * warps * iters * 4 * flop_per;
      printf("%s mma.sync, %2d warps/CTA x 2 CTAs/SM: %7.1f TFLOP/s\n", tf ? "TF32" : "BF16", warps,
             flops / (best * 1e-3) / 1e12);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
