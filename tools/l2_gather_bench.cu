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
  for (int di = 0; di < 3; ++di)
    std::printf("BEST D=%u: %.1f GB/s of gathered rows (%.1f B/clk at the nominal clock)\n", dims[di], best_all[di],
                best_all[di] * 1e9 / (clock_khz * 1e3));
  const cudaError_t e = cudaDeviceSynchronize();
  std::printf("status: %s\n", cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
