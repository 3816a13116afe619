// Shared device helpers: TMA bulk copies + mbarriers (sm_90+/sm_100a PTX),
// numpy-order FP64 arithmetic, warp reductions.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/eca_b200.h"

#define ECA_DEV __device__ __forceinline__

// NVTX ranges around the C-ABI entry points (header-only NVTX3: a no-op
// unless a tool such as nsys / ncu --nvtx is attached); one domain "eca".
#include <nvtx3/nvToolsExt.h>
struct EcaRange {
  explicit EcaRange(const char* name) {
    static nvtxDomainHandle_t dom = nvtxDomainCreateA("eca");
    nvtxEventAttributes_t a = {};
    a.version = NVTX_VERSION;
    a.size = NVTX_EVENT_ATTRIB_STRUCT_SIZE;
    a.messageType = NVTX_MESSAGE_TYPE_ASCII;
    a.message.ascii = name;
    nvtxDomainRangePushEx(dom_ = dom, &a);
  }
  ~EcaRange() { nvtxDomainRangePop(dom_); }
  nvtxDomainHandle_t dom_;
};
#define ECA_RANGE(name) EcaRange eca_range_(name)

// ECA_CHECKED builds (tools/checked.sh): device-side bounds checks at the
// kernels' computed indices; a violation traps (the launch fails with an
// error) instead of corrupting memory silently.  compute-sanitizer is not
// available on the GPU pool, so this plus tests/test_gpu_guard.py (canary
// zones, launch-shape determinism) stands in for memcheck / racecheck.
#ifdef ECA_CHECKED
#define ECA_CHECK(cond)        \
  do {                         \
    if (!(cond)) __trap();     \
  } while (0)
#else
#define ECA_CHECK(cond) \
  do {                  \
  } while (0)
#endif

namespace eca {

// ---------------------------------------------------------------- smem / TMA
ECA_DEV uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

ECA_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}

ECA_DEV void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

ECA_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}

ECA_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "ECA_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra ECA_WAIT;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

// One-shot L2 policy: frame rows are streamed exactly once.
ECA_DEV uint64_t l2_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// TMA 1-D bulk copy global -> shared, completion counted on `bar` (bytes % 16 == 0,
// both addresses 16-byte aligned).
ECA_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}

// ------------------------------------------------ numpy-order FP64 (no FMA)
ECA_DEV double add_rn(double a, double b) { return __dadd_rn(a, b); }
ECA_DEV double sub_rn(double a, double b) { return __dsub_rn(a, b); }
ECA_DEV double mul_rn(double a, double b) { return __dmul_rn(a, b); }
ECA_DEV double div_rn(double a, double b) { return __ddiv_rn(a, b); }

// ------------------------------------------------------------ warp helpers
constexpr unsigned kFull = 0xffffffffu;

ECA_DEV float warp_max(float v) {
#pragma unroll
  for (int d = 16; d; d >>= 1) v = fmaxf(v, __shfl_xor_sync(kFull, v, d));
  return v;
}

// max over the warp of a NON-NEGATIVE float: one REDUX on the bit patterns
// (IEEE order of non-negative floats is their unsigned-integer order)
ECA_DEV float warp_max_nonneg(float v) {
  return __uint_as_float(__reduce_max_sync(kFull, __float_as_uint(v)));
}

ECA_DEV double warp_sum(double v) {
#pragma unroll
  for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(kFull, v, d);
  return v;
}

ECA_DEV int warp_sum(int v) {
#pragma unroll
  for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(kFull, v, d);
  return v;
}

// (score, x) argmax with the reference's tie-breaks: left halves keep the
// smallest x among equal scores, right halves the largest (handcrafted.py:129-131).
struct Best {
  double s;
  int x;
};

ECA_DEV bool better(double s, int x, double bs, int bx, bool prefer_low_x) {
  if (s > bs) return true;
  if (s < bs) return false;
  return prefer_low_x ? (x < bx) : (x > bx);
}

ECA_DEV Best warp_best(Best b, bool prefer_low_x) {
#pragma unroll
  for (int d = 16; d; d >>= 1) {
    const double os = __shfl_xor_sync(kFull, b.s, d);
    const int ox = __shfl_xor_sync(kFull, b.x, d);
    if (better(os, ox, b.s, b.x, prefer_low_x)) {
      b.s = os;
      b.x = ox;
    }
  }
  return b;
}

}  // namespace eca
