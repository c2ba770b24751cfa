// Measured ceiling for the encode kernel's access pattern: random whole-row gathers
// out of an L2-resident codebook-sized table by every SM at once.
//
// encode_kernel (csrc/encode.cu) reads, per peak, one position row of D/8 bytes chosen by the peak's m/z bin:
// the 32 lanes of a warp fetch consecutive 16-byte slabs (LDG.128), 8 rows in flight per warp.  This tool does
// exactly that and nothing else (XOR-folds what it loads so the loads cannot be dropped): table of n_rows x
// row_bytes, one warp per "spectrum", `batch` independent rows in flight, rows drawn by a per-warp LCG
// (uniform over the table, like bins over the codebook).  Reported: GB/s of gathered bytes = the number the
// encode kernel's gather rate (n_bins x D/8 bytes per spectrum / kernel time) can be quoted against.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/l2_gather_bench tools/l2_gather_bench.cu
//   tools/l2_gather_bench            # sweeps D in {2048, 8192, 16384} x warps/CTA x rows in flight
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

template <int kBatch>
__global__ void gather_kernel(const uint4* __restrict__ table, uint32_t n_rows, uint32_t row_u4, uint32_t rows_per_warp,
                              uint4* __restrict__ sink) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  uint32_t state = warp * 2654435761u + 12345u;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (uint32_t r = 0; r < rows_per_warp; r += kBatch) {
    uint32_t row[kBatch];
#pragma unroll
    for (int b = 0; b < kBatch; ++b) {
      state = state * 1664525u + 1013904223u;
      row[b] = static_cast<uint32_t>((uint64_t(state) * n_rows) >> 32);
    }
    for (uint32_t u = lane; u < row_u4; u += 32) {
      uint4 v[kBatch];
#pragma unroll
      for (int b = 0; b < kBatch; ++b) v[b] = __ldg(table + size_t(row[b]) * row_u4 + u);
#pragma unroll
      for (int b = 0; b < kBatch; ++b) {
        acc.x ^= v[b].x;
        acc.y ^= v[b].y;
        acc.z ^= v[b].z;
        acc.w ^= v[b].w;
      }
    }
  }
  if (acc.x == 0x12345678u && acc.y == 0x9abcdef0u) sink[warp] = acc;  // never true in practice; keeps the loads alive
}


// ---- the same gather staged through shared memory by bulk copies (cp.async.bulk + mbarrier) ----------------
// One warp per "spectrum"; per group of 8 entries lanes 0..7 each issue ONE 512-byte bulk copy of a half row
// into the warp's ring of kRing groups (4 KB each), completion on one mbarrier per group; the warp then reads
// the landed half rows with LDS.128 (lane = 16-byte slab) and XOR-folds them.  kLevel adds one LDS.128 per
// entry from an 18 KB table (the encoder's level rows).  No registers are held by loads in flight, so the
// bytes in flight per SM are set by the ring size, not by occupancy.
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_LOOP:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_LOOP;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

template <int kRing, int kLevel>
__global__ void gather_tma_kernel(const uint4* __restrict__ table, uint32_t n_rows, uint32_t row_u4, uint32_t groups_per_warp,
                                  uint4* __restrict__ sink) {
  extern __shared__ __align__(128) unsigned char smem[];
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5, warps = blockDim.x >> 5;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  // layout: [level table 18 KB][per warp: kRing x 4 KB ring][per warp: kRing barriers]
  uint4* s_lvl = reinterpret_cast<uint4*>(smem);
  unsigned char* ring = smem + 18432 + size_t(wib) * kRing * 4096;
  const uint32_t ring_a = smem_u32(ring);
  const uint32_t bar_a = smem_u32(smem + 18432 + size_t(warps) * kRing * 4096 + size_t(wib) * kRing * 8);
  for (uint32_t i = threadIdx.x; i < 18432 / 16; i += blockDim.x) s_lvl[i] = make_uint4(i, i * 3, i * 5, i * 7);
  if (lane == 0)
    for (int g = 0; g < kRing; ++g) mbar_init(bar_a + 8u * g, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  uint32_t state = warp * 2654435761u + 12345u + lane * 40503u;  // lanes 0..7 draw the 8 rows of a group
  const uint32_t halves = row_u4 / 32;                          // 512-byte half rows per row
  auto issue = [&](uint32_t g) {
    const uint32_t slot = g % kRing;
    if (lane == 0) mbar_expect_tx(bar_a + 8u * slot, 8 * 512);
    __syncwarp();
    if (lane < 8) {
      state = state * 1664525u + 1013904223u;
      const uint32_t row = static_cast<uint32_t>((uint64_t(state) * n_rows) >> 32);
      const uint32_t half = (state >> 7) % halves;
      bulk_g2s(ring_a + slot * 4096 + lane * 512, table + size_t(row) * row_u4 + half * 32, 512, bar_a + 8u * slot);
    }
  };
  for (uint32_t g = 0; g < kRing && g < groups_per_warp; ++g) issue(g);
  uint4 acc = make_uint4(0, 0, 0, 0);
  uint32_t lv = lane * 7u;
  for (uint32_t g = 0; g < groups_per_warp; ++g) {
    const uint32_t slot = g % kRing;
    mbar_wait(bar_a + 8u * slot, (g / kRing) & 1u);
    const uint4* src = reinterpret_cast<const uint4*>(ring + slot * 4096) + lane;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint4 v = src[j * 32];
      if (kLevel) {
        lv = lv * 1664525u + 1013904223u;
        const uint4 l = s_lvl[((lv >> 20) % 17u) * 64 + lane];  // warp-uniform level would be the real pattern; lanes differ here only by table row
        v.x ^= l.x;
        v.y ^= l.y;
        v.z ^= l.z;
        v.w ^= l.w;
      }
      acc.x ^= v.x;
      acc.y ^= v.y;
      acc.z ^= v.z;
      acc.w ^= v.w;
    }
    __syncwarp();
    if (g + kRing < groups_per_warp) issue(g + kRing);
  }
  if (acc.x == 0x12345678u && acc.y == 0x9abcdef0u) sink[warp] = acc;
}

template <int kRing, int kLevel>
static double run_tma(const uint4* d_table, uint32_t n_rows, uint32_t row_u4, int warps_per_cta, int ctas_per_sm, int sms,
                      uint4* d_sink, float* out_ms) {
  const uint32_t groups_per_warp = 2048;
  const int grid = sms * ctas_per_sm;
  const size_t smem = 18432 + size_t(warps_per_cta) * kRing * 4096 + size_t(warps_per_cta) * kRing * 8;
  if (smem * ctas_per_sm > 227 * 1024) return 0.0;
  cudaFuncSetAttribute(gather_tma_kernel<kRing, kLevel>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  gather_tma_kernel<kRing, kLevel><<<grid, warps_per_cta * 32, smem>>>(d_table, n_rows, row_u4, groups_per_warp, d_sink);
  cudaEventRecord(e0);
  gather_tma_kernel<kRing, kLevel><<<grid, warps_per_cta * 32, smem>>>(d_table, n_rows, row_u4, groups_per_warp, d_sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *out_ms = ms;
  if (cudaGetLastError() != cudaSuccess) return -1.0;
  const double bytes = double(grid) * warps_per_cta * groups_per_warp * 8 * 512.0;
  return bytes / (ms * 1e-3) / 1e9;
}

template <int kBatch>
static double run(const uint4* d_table, uint32_t n_rows, uint32_t row_u4, int warps_per_cta, int ctas_per_sm, int sms,
                  uint4* d_sink, float* out_ms) {
  const uint32_t rows_per_warp = 8192 / kBatch * kBatch;
  const int grid = sms * ctas_per_sm;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  gather_kernel<kBatch><<<grid, warps_per_cta * 32>>>(d_table, n_rows, row_u4, rows_per_warp, d_sink);  // warm (L2 fill)
  cudaEventRecord(e0);
  gather_kernel<kBatch><<<grid, warps_per_cta * 32>>>(d_table, n_rows, row_u4, rows_per_warp, d_sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *out_ms = ms;
  const double bytes = double(grid) * warps_per_cta * rows_per_warp * row_u4 * 16.0;
  return bytes / (ms * 1e-3) / 1e9;
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  int clock_khz = 0;
  cudaDeviceGetAttribute(&clock_khz, cudaDevAttrClockRate, 0);
  std::printf("device %s, %d SMs, L2 %.0f MB, nominal %.3f GHz\n", prop.name, prop.multiProcessorCount,
              prop.l2CacheSize / 1048576.0, clock_khz / 1e6);
  const uint32_t n_rows = 27980;  // dimension(PreprocessConfig{}) = f (preprocess.cpp:36-39)
  uint4* d_sink = nullptr;
  cudaMalloc(&d_sink, size_t(1) << 24);
  double best_all[3] = {0, 0, 0};
  const uint32_t dims[3] = {2048, 8192, 16384};
  for (int di = 0; di < 3; ++di) {
    const uint32_t row_u4 = dims[di] / 128;
    const size_t bytes = size_t(n_rows) * row_u4 * 16;
    std::vector<uint32_t> h(bytes / 4);
    uint32_t s = 1u + di;
    for (auto& w : h) w = (s = s * 1664525u + 1013904223u);
    uint4* d_table = nullptr;
    cudaMalloc(&d_table, bytes);
    cudaMemcpy(d_table, h.data(), bytes, cudaMemcpyHostToDevice);
    for (int warps : {4, 8, 16})
      for (int ctas : {1, 2, 4, 8}) {
        if (warps * ctas > 64) continue;
        float ms;
        double g4 = run<4>(d_table, n_rows, row_u4, warps, ctas, prop.multiProcessorCount, d_sink, &ms);
        double g8 = run<8>(d_table, n_rows, row_u4, warps, ctas, prop.multiProcessorCount, d_sink, &ms);
        double g16 = run<16>(d_table, n_rows, row_u4, warps, ctas, prop.multiProcessorCount, d_sink, &ms);
        std::printf("D=%5u table %6.2f MB  %2d warps/CTA x %d CTA/SM (%2d warps/SM): rows in flight 4: %8.1f  8: %8.1f  16: %8.1f GB/s\n",
                    dims[di], bytes / 1e6, warps, ctas, warps * ctas, g4, g8, g16);
        best_all[di] = g4 > best_all[di] ? g4 : best_all[di];
        best_all[di] = g8 > best_all[di] ? g8 : best_all[di];
        best_all[di] = g16 > best_all[di] ? g16 : best_all[di];
      }
    cudaFree(d_table);
  }

  // bulk-copy staged variant, D = 8192 only (half rows of 512 bytes)
  {
    const uint32_t row_u4 = 8192 / 128;
    const size_t bytes = size_t(n_rows) * row_u4 * 16;
    std::vector<uint32_t> h(bytes / 4);
    uint32_t s = 77u;
    for (auto& w : h) w = (s = s * 1664525u + 1013904223u);
    uint4* d_table = nullptr;
    cudaMalloc(&d_table, bytes);
    cudaMemcpy(d_table, h.data(), bytes, cudaMemcpyHostToDevice);
    for (int warps : {8, 12, 16, 24})
      for (int ctas : {1, 2}) {
        float ms;
        const double a2 = run_tma<2, 0>(d_table, n_rows, row_u4, warps, ctas, prop.multiProcessorCount, d_sink, &ms);
        const double a3 = run_tma<3, 0>(d_table, n_rows, row_u4, warps, ctas, prop.multiProcessorCount, d_sink, &ms);
        const double a4 = run_tma<4, 0>(d_table, n_rows, row_u4, warps, ctas, prop.multiProcessorCount, d_sink, &ms);
        const double l2 = run_tma<2, 1>(d_table, n_rows, row_u4, warps, ctas, prop.multiProcessorCount, d_sink, &ms);
        const double l3 = run_tma<3, 1>(d_table, n_rows, row_u4, warps, ctas, prop.multiProcessorCount, d_sink, &ms);
        const double l4 = run_tma<4, 1>(d_table, n_rows, row_u4, warps, ctas, prop.multiProcessorCount, d_sink, &ms);
        std::printf("TMA-staged D=8192 %2d warps/CTA x %d CTA/SM: ring 2/3/4 groups of 8 half rows: %8.1f %8.1f %8.1f GB/s;  + level LDS: %8.1f %8.1f %8.1f GB/s\n",
                    warps, ctas, a2, a3, a4, l2, l3, l4);
      }
    cudaFree(d_table);
  }
  for (int di = 0; di < 3; ++di)
    std::printf("BEST D=%u: %.1f GB/s of gathered rows (%.1f B/clk at the nominal clock)\n", dims[di], best_all[di],
                best_all[di] * 1e9 / (clock_khz * 1e3));
  const cudaError_t e = cudaDeviceSynchronize();
  std::printf("status: %s\n", cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
