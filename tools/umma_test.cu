// Standalone check of a hand-written tcgen05 GEMM building block (kind::tf32,
// cta_group::1, M=128, N=32, K=144, SWIZZLE_NONE K-major operands, 3xTF32
// split for FP32-level accuracy) against a CPU double-precision reference.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_test tools/umma_test.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int M = 128, N = 32, K = 144;
constexpr int KC = K / 4;                 // 16-byte K chunks per row
constexpr int SBO = KC * 128;             // bytes between 8-row groups
constexpr int LBO = 128;                  // bytes between K chunks

__device__ __forceinline__ uint32_t sa(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
// byte offset of element (row, k) in the K-major interleaved canonical layout
__device__ __forceinline__ int kmaj_off(int row, int k) {
  return (row >> 3) * SBO + (k >> 2) * LBO + (row & 7) * 16 + (k & 3) * 4;
}
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
  uint64_t d = 0;
  d |= uint64_t((addr >> 4) & 0x3FFF);
  d |= uint64_t((LBO >> 4) & 0x3FFF) << 16;
  d |= uint64_t((SBO >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;                 // version 1 (sm100)
  return d;                               // base offset 0, lbo mode 0, SWIZZLE_NONE
}
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4)        // D format F32
       | (2u << 7)        // A format TF32
       | (2u << 10)       // B format TF32
       | (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);   // K-major A and B
}

__global__ void umma_gemm(const float* a, const float* b, float* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* a_hi = smem;
  uint8_t* a_lo = a_hi + M * K * 4;
  uint8_t* b_hi = a_lo + M * K * 4;
  uint8_t* b_lo = b_hi + N * K * 4;
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < M * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    const float v = a[i], h = tf32_rna(v);
    *reinterpret_cast<float*>(a_hi + kmaj_off(r, k)) = h;
    *reinterpret_cast<float*>(a_lo + kmaj_off(r, k)) = tf32_rna(v - h);
  }
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    const float v = b[i], h = tf32_rna(v);
    *reinterpret_cast<float*>(b_hi + kmaj_off(r, k)) = h;
    *reinterpret_cast<float*>(b_lo + kmaj_off(r, k)) = tf32_rna(v - h);
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(sa(&tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // st.shared -> async proxy
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;
  if (tid == 0) {
    const uint32_t idesc = idesc_tf32(M, N);
    for (int j = 0; j < K / 8; ++j) {      // 8 tf32 = 32 bytes of K per instruction
      const uint32_t off = j * 2 * LBO;
      const uint64_t ah = smem_desc(sa(a_hi) + off), al = smem_desc(sa(a_lo) + off);
      const uint64_t bh = smem_desc(sa(b_hi) + off), bl = smem_desc(sa(b_lo) + off);
      const uint64_t pa[3] = {ah, ah, al}, pb[3] = {bh, bl, bh};
      for (int t = 0; t < 3; ++t) {
        const uint32_t acc = (j > 0 || t > 0) ? 1u : 0u;
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
            "l"(pa[t]), "l"(pb[t]), "r"(idesc), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     sa(&bar))
                 : "memory");
  }
  asm volatile(
      "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}\n" ::"r"(
          sa(&bar))
      : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t v[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
        "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
        "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
        "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(tmem + (uint32_t(warp * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  const int row = warp * 32 + lane;
  for (int n = 0; n < N; ++n) out[row * N + n] = __uint_as_float(v[n]);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

int main() {
  float *a, *b, *o;
  cudaMallocManaged(&a, M * K * 4);
  cudaMallocManaged(&b, N * K * 4);
  cudaMallocManaged(&o, M * N * 4);
  srand(1);
  for (int i = 0; i < M * K; ++i) a[i] = float(rand()) / RAND_MAX * 2.f - 1.f;
  for (int i = 0; i < N * K; ++i) b[i] = float(rand()) / RAND_MAX * 0.2f - 0.1f;
  const size_t smem = size_t(2 * M * K * 4 + 2 * N * K * 4);
  cudaFuncSetAttribute(umma_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  umma_gemm<<<1, 128, smem>>>(a, b, o);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  double max_err = 0.0, max_ref = 0.0, max_f32 = 0.0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double ref = 0.0;
      float f32 = 0.f;
      for (int k = 0; k < K; ++k) {
        ref += double(a[m * K + k]) * double(b[n * K + k]);
        f32 = fmaf(a[m * K + k], b[n * K + k], f32);
      }
      max_err = fmax(max_err, fabs(o[m * N + n] - ref));
      max_f32 = fmax(max_f32, fabs(double(f32) - ref));
      max_ref = fmax(max_ref, fabs(ref));
    }
  printf("3xTF32 tcgen05: max |err| %.3e (fp32 FMA chain %.3e), max |ref| %.3f, sample %f vs ...\n",
         max_err, max_f32, max_ref, o[0]);
  return (e == cudaSuccess && max_err < 1e-4) ? 0 : 1;
}
