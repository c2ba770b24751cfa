// CTA-pair (cta_group::2) probe for the tensor search engine: what would pairing two SMs on one
// 256-query x 224-row tile buy?
//
// The search kernel (csrc/search_tc.cu) is power-capped: its MMA shape issued back to back with no
// memory traffic holds ~1.67 of 1.965 GHz (tc_peak_kernel).  In cta_group::2 mode each SM's tensor
// core reads its own 128 A rows but only HALF of the B tile from its shared memory (the halves are
// exchanged inside the TPC), and only half of every B tile has to come from L2.  Both cut energy per
// MAC, which under a power cap is clock.  This tool
//   1. checks the 2-CTA semantics the kernel would rely on (M = 256 split over the pair by rows,
//      B split by rows (N halves), D lanes = own A rows, all N columns) against a host dot product;
//   2. times the issue loop in both modes on every SM, alternating, under the same power cap.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/tc_pair_probe tools/tc_pair_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int kM = 128;          // A rows per CTA == TMEM lanes
constexpr int kN = 224;          // B rows per tile
constexpr int kKB = 128;         // bytes of K per row per stage (256 e2m1 dimensions)
constexpr uint32_t kABytes = kM * kKB;
constexpr uint32_t kSfCol = 480;
constexpr int kThreads = 192;
constexpr int kDepth = 4;

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  const long long t0 = clock64();
  while (!mbar_try_wait(bar, parity))
    if (clock64() - t0 > 4000000000ll) __trap();
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {  // K-major SWIZZLE_128B, 128-byte rows
  const uint64_t lo = (uint64_t(addr & 0x3FFFFu) >> 4) | (uint64_t(1) << 16);
  const uint64_t hi = uint64_t(1024 >> 4) | (uint64_t(1) << 14) | (uint64_t(2) << 29);
  return lo | (hi << 32);
}
template <int kM_, int kN_>
__host__ __device__ constexpr uint32_t idesc_fp4() {
  return (1u << 7) | (1u << 10) | (uint32_t(kN_ >> 3) << 17) | (1u << 23) | (uint32_t(kM_ >> 4) << 24);
}
template <int kCtas>
__device__ __forceinline__ void mma_fp4(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t sfa, uint32_t sfb,
                                        uint32_t acc) {
  if constexpr (kCtas == 1)
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %6, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%4], [%5], p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(sfa), "r"(sfb), "r"(acc)
        : "memory");
  else
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %6, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%4], [%5], p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(sfa), "r"(sfb), "r"(acc)
        : "memory");
}
template <int kCtas>
__device__ __forceinline__ void commit(uint32_t bar) {
  if constexpr (kCtas == 1)
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
  else
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void st32_fill(uint32_t taddr, uint32_t w) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, "
      "%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1};" ::"r"(taddr),
      "r"(w)
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void ld32(uint32_t taddr, int (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// kCtas = 1: the search kernel's shape (M128 N224, A 16 KB + B 28 KB per stage in this CTA)
// kCtas = 2: M256 N224 over a CTA pair (A 16 KB + B 14 KB per stage in each CTA)
// groups > 0: timing loop (4 MMAs per commit, kDepth commits in flight, operands = whatever smem holds)
// groups == 0: functional check: operands from a_img / b_img, one stage, accumulator written to d_out
template <int kCtas>
__global__ void __launch_bounds__(kThreads, 1)
pair_kernel(uint32_t groups, const uint8_t* __restrict__ a_img, const uint8_t* __restrict__ b_img, float* __restrict__ d_out) {
  constexpr uint32_t kBRows = kN / kCtas;
  constexpr uint32_t kBBytes = kBRows * kKB;
  constexpr uint32_t kStage = kABytes + kBBytes;
  extern __shared__ unsigned char smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  unsigned char* gen = smem_raw + (base - raw);
  const uint32_t bar0 = base + kStage;
  volatile uint32_t* tmem_slot = reinterpret_cast<volatile uint32_t*>(gen + kStage + 8 * kDepth);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = kCtas == 2 ? cluster_ctarank() : 0;
  const uint32_t pair = kCtas == 2 ? blockIdx.x / 2 : blockIdx.x;

  if (groups == 0) {  // this CTA's A rows [rank*128, +128) and B rows [rank*kBRows, +kBRows), already swizzled
    const uint4* asrc = reinterpret_cast<const uint4*>(a_img + (size_t(pair) * kCtas + rank) * kABytes);
    const uint4* bsrc = reinterpret_cast<const uint4*>(b_img + size_t(pair) * kN * kKB + size_t(rank) * kBBytes);
    for (uint32_t i = threadIdx.x; i < kABytes / 16; i += blockDim.x) reinterpret_cast<uint4*>(gen)[i] = asrc[i];
    for (uint32_t i = threadIdx.x; i < kBBytes / 16; i += blockDim.x) reinterpret_cast<uint4*>(gen + kABytes)[i] = bsrc[i];
  } else {
    for (uint32_t i = threadIdx.x; i < kStage / 16; i += blockDim.x)
      reinterpret_cast<uint4*>(gen)[i] = make_uint4(0x2A2A2A2Au, 0xA2A2A2A2u, 0x22AA22AAu, 0xAAAA2222u);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    for (int s = 0; s < kDepth; ++s) mbar_init(bar0 + 8u * s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    if constexpr (kCtas == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(const_cast<uint32_t*>(tmem_slot))),
                   "r"(512u)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(const_cast<uint32_t*>(tmem_slot))),
                   "r"(512u)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
  }
  fence_before();
  __syncthreads();
  if constexpr (kCtas == 2) cluster_sync();
  fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (warp >= 2) st32_fill(tmem_base + (uint32_t((warp & 3) * 32) << 16) + kSfCol, 0x7F7F7F7Fu);
  fence_before();
  __syncthreads();
  if constexpr (kCtas == 2) cluster_sync();
  fence_after();

  constexpr uint32_t idesc = idesc_fp4<kM * kCtas, kN>();
  if (rank == 0 && warp == 1 && lane == 0) {
    const uint64_t adesc = smem_desc(base);
    const uint64_t bdesc = smem_desc(base + kABytes);
    if (groups == 0) {
#pragma unroll
      for (uint32_t k = 0; k < kKB / 32; ++k)
        mma_fp4<kCtas>(tmem_base, adesc + 2 * k, bdesc + 2 * k, idesc, tmem_base + kSfCol, tmem_base + kSfCol + 16, k != 0u);
      commit<kCtas>(bar0);
      mbar_wait(bar0, 0);
    } else {
      for (uint32_t g = 0; g < groups; ++g) {
        const uint32_t slot = g % kDepth;
        if (g >= kDepth) mbar_wait(bar0 + 8u * slot, ((g / kDepth) - 1u) & 1u);
        const uint32_t d = tmem_base + (g & 1u) * kN;
#pragma unroll
        for (uint32_t k = 0; k < kKB / 32; ++k)
          mma_fp4<kCtas>(d, adesc + 2 * k, bdesc + 2 * k, idesc, tmem_base + kSfCol, tmem_base + kSfCol + 16, 1u);
        commit<kCtas>(bar0 + 8u * slot);
      }
      for (uint32_t g = groups > kDepth ? groups - kDepth : 0; g < groups; ++g)
        mbar_wait(bar0 + 8u * (g % kDepth), (g / kDepth) & 1u);
    }
  }
  __syncwarp();
  fence_before();
  __syncthreads();
  if constexpr (kCtas == 2) cluster_sync();
  fence_after();
  if (groups == 0 && warp >= 2) {  // lanes = own A rows, columns = all kN B rows
    const int quarter = warp & 3;
    const uint32_t qrow = quarter * 32 + lane;
    float* dst = d_out + (size_t(pair) * kCtas * kM + rank * kM + qrow) * kN;
    for (int c = 0; c < kN; c += 32) {
      int v[32];
      ld32(tmem_base + (uint32_t(quarter * 32) << 16) + c, v);
      for (int j = 0; j < 32; ++j) dst[c + j] = __int_as_float(v[j]);
    }
  }
  fence_before();
  __syncthreads();
  if constexpr (kCtas == 2) cluster_sync();
  if (warp == 1) {
    fence_after();
    if constexpr (kCtas == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512u) : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512u) : "memory");
  }
}

template <int kCtas>
static void launch(int n_ctas, uint32_t groups, const uint8_t* a, const uint8_t* b, float* d, cudaStream_t s) {
  constexpr uint32_t kStage = kABytes + (kN / kCtas) * kKB;
  constexpr uint32_t smem = kStage + 1024 + 256;
  CK(cudaFuncSetAttribute(pair_kernel<kCtas>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n_ctas);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kCtas;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, pair_kernel<kCtas>, groups, a, b, d));
}

// host image of `rows` x 256 +-1 values in the kernel's layout: 128 bytes per row, 16-byte units XOR-swizzled by row & 7
static void make_image(const std::vector<int8_t>& v, int rows, std::vector<uint8_t>& img) {
  img.assign(size_t(rows) * kKB, 0);
  for (int r = 0; r < rows; ++r)
    for (int d = 0; d < 256; ++d) {
      const uint8_t nib = v[size_t(r) * 256 + d] > 0 ? 0x2 : 0xA;
      const int byte = d / 2, unit = byte / 16, in_unit = byte % 16;
      uint8_t& dst = img[size_t(r) * kKB + ((unit ^ (r & 7)) << 4) + in_unit];
      dst |= (d & 1) ? nib << 4 : nib;
    }
}

template <int kCtas>
static bool functional(int n_pairs) {
  const int a_rows = kM * kCtas;
  std::vector<int8_t> a(size_t(n_pairs) * a_rows * 256), b(size_t(n_pairs) * kN * 256);
  uint32_t s = 12345u + kCtas;
  for (auto& x : a) x = ((s = s * 1664525u + 1013904223u) >> 16) & 1 ? 1 : -1;
  for (auto& x : b) x = ((s = s * 1664525u + 1013904223u) >> 16) & 1 ? 1 : -1;
  std::vector<uint8_t> ai, bi, tmp;
  for (int p = 0; p < n_pairs; ++p) {
    // A: per CTA a 128-row block whose swizzle phase restarts at its own row 0
    for (int c = 0; c < kCtas; ++c) {
      std::vector<int8_t> blk(a.begin() + (size_t(p) * a_rows + c * kM) * 256, a.begin() + (size_t(p) * a_rows + (c + 1) * kM) * 256);
      make_image(blk, kM, tmp);
      ai.insert(ai.end(), tmp.begin(), tmp.end());
    }
    // B: 224 rows; each CTA's half starts at row rank * 112 (a multiple of 8: same swizzle phase)
    std::vector<int8_t> blk(b.begin() + size_t(p) * kN * 256, b.begin() + size_t(p + 1) * kN * 256);
    make_image(blk, kN, tmp);
    bi.insert(bi.end(), tmp.begin(), tmp.end());
  }
  uint8_t *da, *db;
  float* dd;
  CK(cudaMalloc(&da, ai.size()));
  CK(cudaMalloc(&db, bi.size()));
  CK(cudaMalloc(&dd, size_t(n_pairs) * a_rows * kN * 4));
  CK(cudaMemcpy(da, ai.data(), ai.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(db, bi.data(), bi.size(), cudaMemcpyHostToDevice));
  CK(cudaMemset(dd, 0xFF, size_t(n_pairs) * a_rows * kN * 4));
  launch<kCtas>(n_pairs * kCtas, 0, da, db, dd, 0);
  CK(cudaDeviceSynchronize());
  std::vector<float> out(size_t(n_pairs) * a_rows * kN);
  CK(cudaMemcpy(out.data(), dd, out.size() * 4, cudaMemcpyDeviceToHost));
  size_t bad = 0;
  for (int p = 0; p < n_pairs; ++p)
    for (int r = 0; r < a_rows; ++r)
      for (int c = 0; c < kN; ++c) {
        int dot = 0;
        for (int d = 0; d < 256; ++d) dot += a[(size_t(p) * a_rows + r) * 256 + d] * b[(size_t(p) * kN + c) * 256 + d];
        const float got = out[(size_t(p) * a_rows + r) * kN + c];
        if (got != float(dot)) {
          if (bad < 5) printf("  mismatch pair %d row %d col %d: got %g want %d\n", p, r, c, got, dot);
          ++bad;
        }
      }
  printf("functional cta_group::%d (M%d N%d): %zu mismatches of %zu\n", kCtas, kM * kCtas, kN, bad, out.size());
  cudaFree(da);
  cudaFree(db);
  cudaFree(dd);
  return bad == 0;
}

template <int kCtas>
static double timed(int n_sms, double seconds, float* out_ms) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  uint32_t groups = 1u << 14;
  float ms = 0;
  for (int pass = 0; pass < 3; ++pass) {
    CK(cudaEventRecord(e0));
    launch<kCtas>(n_sms, groups, nullptr, nullptr, nullptr, 0);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (pass == 0) {
      double want = seconds * 1e3 / (ms > 1e-3f ? ms : 1e-3f) * groups;
      groups = uint32_t(want < 4.0e9 ? want : 4.0e9);
      if (groups < 1024) groups = 1024;
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *out_ms = ms;
  // per group: 4 MMAs of (M x N x 64); a pair issues M = 256 from one CTA, so n_sms / kCtas issuers
  const double ops_group = 2.0 * (kM * kCtas) * kN * 256.0;
  return ops_group * groups * (n_sms / kCtas) / (ms * 1e-3);
}

int main(int argc, char** argv) {
  const double seconds = argc > 1 ? atof(argv[1]) : 0.5;
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  const int n_sms = prop.multiProcessorCount;
  printf("%s, %d SMs\n", prop.name, n_sms);
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(n_sms);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kABytes + (kN / 2) * kKB + 1280;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n_clusters = 0;
    CK(cudaFuncSetAttribute(pair_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(cfg.dynamicSmemBytes)));
    CK(cudaOccupancyMaxActiveClusters(&n_clusters, pair_kernel<2>, &cfg));
    printf("co-resident 2-CTA clusters (1 CTA per SM by launch bounds): %d\n", n_clusters);
  }
  bool ok = functional<1>(3);
  ok = functional<2>(3) && ok;
  if (!ok) return 2;
  for (int rep = 0; rep < 3; ++rep) {
    float ms1, ms2;
    const double r1 = timed<1>(n_sms, seconds, &ms1);
    const double r2 = timed<2>(n_sms / 2 * 2, seconds, &ms2);
    printf("rep %d: cta_group::1 %.3f POP/s (%.1f ms)   cta_group::2 %.3f POP/s (%.1f ms)   ratio %.4f\n", rep, r1 * 1e-15,
           ms1, r2 * 1e-15, ms2, r2 / r1);
  }
  return 0;
}
