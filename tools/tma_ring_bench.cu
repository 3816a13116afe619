// Microbenchmark: per-warp 1-D TMA (cp.async.bulk) rings streaming a large
// buffer into shared memory, as bounds_kernel does.  Reports GB/s per
// (copy bytes, copies per item, stages, warps per CTA).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_ring_bench tools/tma_ring_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// strip mode (item_bytes < 0): item = (frame * 16 + strip) * 2 + half of a 1080p frame
// pool; 3 copies of 2944 B (rows y-1..y+1, row stride 5760 B), like bounds_kernel
__constant__ int c_rows[16] = {25, 40, 65, 103, 160, 241, 346, 473, 607, 734, 839, 920, 977, 1015, 1040, 1055};

__global__ void ring(const uint8_t* src, int64_t item_bytes, int copies, int n_items, int ns,
                     int stage_bytes, int dynamic, int* ticket, unsigned long long* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, warps = blockDim.x >> 5;
  uint8_t* mine = smem + size_t(wib) * (ns * stage_bytes + 128);
  uint64_t* bars = reinterpret_cast<uint64_t*>(mine + ns * stage_bytes);
  int* q = reinterpret_cast<int*>(bars + 8);
  const int gw = blockIdx.x * warps + wib, nw = gridDim.x * warps;
  const int64_t cbytes = item_bytes / copies;
  auto issue = [&](int it, int s) {
    if (item_bytes < 0) {
      const int half = it & 1, fs = it >> 1, frame = fs / 16, strip = fs - frame * 16;
      const uint8_t* row0 = src + int64_t(frame) * (1080 * 5760) + int64_t(c_rows[strip] - 1) * 5760 +
                            half * 2880;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bars[s])),
                   "r"(uint32_t(3 * 2896)) : "memory");
      for (int r = 0; r < 3; ++r)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
                "r"(sa(mine + s * stage_bytes + r * 2944)),
            "l"(row0 + r * 5760), "r"(2896u), "r"(sa(&bars[s]))
            : "memory");
      return;
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bars[s])),
                 "r"(uint32_t(item_bytes)) : "memory");
    for (int c = 0; c < copies; ++c)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
              "r"(sa(mine + s * stage_bytes + c * cbytes)),
          "l"(src + int64_t(it) * item_bytes + c * cbytes), "r"(uint32_t(cbytes)), "r"(sa(&bars[s]))
          : "memory");
  };
  if (lane == 0) {
    for (int s = 0; s < ns; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bars[s])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < ns; ++s) {
      const int it = dynamic ? atomicAdd(ticket, 1) : gw + s * nw;
      q[s] = it;
      if (it < n_items) issue(it, s);
    }
  }
  __syncwarp();
  unsigned long long acc = 0;
  int stage = 0;
  uint32_t phase = 0;
  for (;;) {
    const int it = q[stage];
    if (it >= n_items) break;
    asm volatile(
        "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W;\n}\n" ::
            "r"(sa(&bars[stage])),
        "r"(phase) : "memory");
    acc += mine[stage * stage_bytes + lane * 4];
    __syncwarp();
    if (lane == 0) {
      const int nx = dynamic ? atomicAdd(ticket, 1) : it + ns * nw;
      q[stage] = nx;
      if (nx < n_items) issue(nx, stage);
    }
    __syncwarp();
    if (++stage == ns) {
      stage = 0;
      phase ^= 1u;
    }
  }
  if (acc == 0xdeadbeef) *sink = acc;
}

int host_mode(int sms) {
  // 1-D bulk copies whose SOURCE is mapped pinned host memory (zero-copy over PCIe)
  const int64_t total = int64_t(256) << 20;
  uint8_t* h = nullptr;
  if (cudaHostAlloc(&h, total, cudaHostAllocMapped) != cudaSuccess) { printf("hostalloc failed\n"); return 1; }
  memset(h, 1, total);
  uint8_t* d = nullptr;
  cudaHostGetDevicePointer(&d, h, 0);
  int* ticket; cudaMalloc(&ticket, 4);
  unsigned long long* sink; cudaMalloc(&sink, 8);
  for (int item : {2304, 8832, 32768}) {
    for (int ns : {1, 2, 4}) {
      const int warps = 2, n_items = int(total / item), stage = (item + 127) / 128 * 128;
      const size_t smem = size_t(warps) * (ns * stage + 128);
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ring, 32 * warps, smem);
      if (per_sm < 1) continue;
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      float best = 1e9;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        ring<<<sms * per_sm, 32 * warps, smem>>>(d, item, 1, n_items, ns, stage, 0, ticket, sink);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
      }
      printf("HOST-mapped source: item %6d B stages %d (%2d warps/SM): %6.1f GB/s  (%s)\n", item, ns,
             per_sm * warps, double(n_items) * item / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
  }
  cudaFreeHost(h);
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 1) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    return host_mode(sms);
  }
  const int64_t total = int64_t(2048) * 1080 * 5760;   // 2048 1080p frames (12.7 GB)
  uint8_t* buf;
  if (cudaMalloc(&buf, total + (1 << 20)) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMemset(buf, 1, total);
  int* ticket;
  cudaMalloc(&ticket, 4);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  struct Cfg { int item, copies, ns, warps, dyn; };
  const Cfg cfgs[] = {
      {-1, 3, 1, 2, 0}, {-1, 3, 1, 2, 1}, {-1, 3, 2, 2, 0}, {-1, 3, 2, 1, 0}, {-1, 3, 3, 1, 0},
      {-1, 3, 1, 1, 0}, {8832, 3, 1, 2, 0}, {8832, 3, 2, 2, 0}, {17664, 3, 1, 2, 0},
      {17664, 3, 2, 1, 0}, {35328, 3, 1, 1, 0}};
  for (const Cfg& c : cfgs) {
    const bool strip = c.item < 0;
    // 256 frames x 16 strips x 2 halves per launch (the bench step), or the
    // same 70.8 MB as contiguous items
    const int n_items = strip ? 256 * 16 * 2 : int(70778880 / c.item);
    const int64_t moved = strip ? int64_t(n_items) * 3 * 2896 : int64_t(n_items) * c.item;
    const int stage = strip ? 3 * 2944 : (c.item + 127) / 128 * 128;
    const size_t smem = size_t(c.warps) * (c.ns * stage + 128);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ring, 32 * c.warps, smem);
    if (per_sm < 1) { printf("skip\n"); continue; }
    const int grid = sms * per_sm;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e9;
    for (int rep = 0; rep < 8; ++rep) {
      cudaMemset(ticket, 0, 4);
      // rotate over the pool so every launch reads DRAM (1.6 GB per slot)
      const uint8_t* base = buf + int64_t(rep % 8) * 256 * 1080 * 5760;
      cudaEventRecord(a);
      ring<<<grid, 32 * c.warps, smem>>>(base, c.item, c.copies, n_items, c.ns, stage, c.dyn, ticket,
                                         sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("item %6d B  copies %d  stages %d  warps/CTA %d  CTAs/SM %2d (%2d warps)  %s  %7.1f GB/s\n",
           c.item, c.copies, c.ns, c.warps, per_sm, per_sm * c.warps, c.dyn ? "dyn " : "stat",
           double(moved) / (best * 1e-3) / 1e9);
  }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
