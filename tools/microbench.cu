// Pipe-rate microbenchmarks that decide the search kernel's inner loop on sm_100a:
//   POPC rate, LOP3 rate, whether they overlap, and the legacy b1 tensor path (mma.sync
//   m16n8k256 and.popc).  Prints per-SM-per-clock throughputs.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

#define ITERS 4096

__global__ void k_popc(uint32_t* out, uint32_t seed) {
  uint32_t a[8];
  for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x * 8 + i;
  uint32_t acc[8] = {0};
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { acc[i] += __popc(a[i]); a[i] ^= acc[i]; }
  }
  uint32_t s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_popc_only(uint32_t* out, uint32_t seed) {  // dependent chain per slot: popc(popc()) keeps only POPC in the loop
  uint32_t a[8];
  for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x * 8 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = __popc(a[i]) | 0x10000u * 0 + a[i] * 0 + __popc(a[i] + it);
  }
  uint32_t s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_lop3(uint32_t* out, uint32_t seed) {
  uint32_t a[8], b = seed * 3 + threadIdx.x, c = seed * 7;
  for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x * 8 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = (a[i] & b) | (a[i] & c) | (b & c) ^ it;
  }
  uint32_t s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// xor + popc + add: the plain Hamming inner loop (per 32-bit word: 1 LOP, 1 POPC, 1 IADD)
__global__ void k_hamming(uint32_t* out, uint32_t seed) {
  uint32_t r[8], q[8], acc[8] = {0};
  for (int i = 0; i < 8; ++i) { r[i] = seed + threadIdx.x * 8 + i; q[i] = seed * 5 + i; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { acc[i] += __popc(r[i] ^ q[i]); r[i] += 0x9e3779b9u; }
  }
  uint32_t s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// 3:2 carry-save version: per 3 words 3 XOR + 2 CSA LOP3 + 2 POPC + 2 IADD
__global__ void k_hamming_csa3(uint32_t* out, uint32_t seed) {
  uint32_t r[9], q[9], a1[3] = {0}, a2[3] = {0};
  for (int i = 0; i < 9; ++i) { r[i] = seed + threadIdx.x * 9 + i; q[i] = seed * 5 + i; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int g = 0; g < 3; ++g) {
      uint32_t x = r[3 * g] ^ q[3 * g], y = r[3 * g + 1] ^ q[3 * g + 1], z = r[3 * g + 2] ^ q[3 * g + 2];
      a1[g] += __popc(x ^ y ^ z);
      a2[g] += __popc((x & y) | (x & z) | (y & z));
      r[3 * g] += 0x9e3779b9u; r[3 * g + 1] += 0x7f4a7c15u; r[3 * g + 2] += 0x85ebca6bu;
    }
  }
  uint32_t s = 0;
  for (int g = 0; g < 3; ++g) s += a1[g] + 2 * a2[g];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// 7:3 carry-save: per 7 words 7 XOR + 8 LOP3 + 3 POPC + 3 IADD
__global__ void k_hamming_csa7(uint32_t* out, uint32_t seed) {
  uint32_t r[7], q[7], a1 = 0, a2 = 0, a4 = 0;
  for (int i = 0; i < 7; ++i) { r[i] = seed + threadIdx.x * 7 + i; q[i] = seed * 5 + i; }
  for (int it = 0; it < ITERS; ++it) {
    uint32_t x[7];
#pragma unroll
    for (int i = 0; i < 7; ++i) { x[i] = r[i] ^ q[i]; r[i] += 0x9e3779b9u * (i + 1); }
    uint32_t s1 = x[0] ^ x[1] ^ x[2], c1 = (x[0] & x[1]) | (x[0] & x[2]) | (x[1] & x[2]);
    uint32_t s2 = x[3] ^ x[4] ^ x[5], c2 = (x[3] & x[4]) | (x[3] & x[5]) | (x[4] & x[5]);
    uint32_t ones = s1 ^ s2 ^ x[6], c3 = (s1 & s2) | (s1 & x[6]) | (s2 & x[6]);
    uint32_t twos = c1 ^ c2 ^ c3, fours = (c1 & c2) | (c1 & c3) | (c2 & c3);
    a1 += __popc(ones); a2 += __popc(twos); a4 += __popc(fours);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a1 + 2 * a2 + 4 * a4;
}

// legacy binary tensor path: mma.sync.m16n8k256 b1 and.popc, 4 independent accumulators
__global__ void k_mma_b1(int* out, uint32_t seed) {
  uint32_t a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = seed + threadIdx.x * 4 + i;
  b[0] = seed * 3 + threadIdx.x; b[1] = seed * 5 + threadIdx.x;
  int c[4][4] = {};
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc "
                   "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+r"(c[j][0]), "+r"(c[j][1]), "+r"(c[j][2]), "+r"(c[j][3])
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  int s = 0;
  for (int j = 0; j < 4; ++j) for (int i = 0; i < 4; ++i) s += c[j][i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// int8 legacy mma.sync m16n8k32 s8
__global__ void k_mma_s8(int* out, uint32_t seed) {
  uint32_t a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = seed + threadIdx.x * 4 + i;
  b[0] = seed * 3 + threadIdx.x; b[1] = seed * 5 + threadIdx.x;
  int c[4][4] = {};
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 "
                   "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+r"(c[j][0]), "+r"(c[j][1]), "+r"(c[j][2]), "+r"(c[j][3])
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  int s = 0;
  for (int j = 0; j < 4; ++j) for (int i = 0; i < 4; ++i) s += c[j][i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename K, typename T>
static void run(const char* name, K kernel, T* out, double ops_per_thread_iter, int sms, double clk_ghz,
                const char* unit) {
  const int threads = 256, blocks = sms * 8;
  kernel<<<blocks, threads>>>(out, 1);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) kernel<<<blocks, threads>>>(out, r + 2);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double total = 5.0 * blocks * threads * double(ITERS) * ops_per_thread_iter;
  const double per_s = total / (ms * 1e-3);
  printf("%-18s %8.3f ms  %10.2f G%s/s  %8.2f %s/clk/SM (at %.3f GHz)  err=%s\n", name, ms, per_s * 1e-9,
         unit, per_s / (sms * clk_ghz * 1e9), unit, clk_ghz, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  const double ghz = p.clockRate * 1e-6;
  printf("device %s, %d SMs, clockRate %.3f GHz (nominal max; actual clock may differ)\n", p.name, sms, ghz);
  uint32_t* out;
  cudaMalloc(&out, size_t(sms) * 8 * 256 * 4);
  run("popc+xor+add", k_popc, out, 8, sms, ghz, "popc");
  run("lop3", k_lop3, out, 8, sms, ghz, "lop3");
  run("hamming plain", k_hamming, out, 8, sms, ghz, "word");
  run("hamming csa3", k_hamming_csa3, out, 9, sms, ghz, "word");
  run("hamming csa7", k_hamming_csa7, out, 7, sms, ghz, "word");
  run("mma.b1 and.popc", k_mma_b1, (int*)out, 4.0 * 16 * 8 * 256 / 32, sms, ghz, "bitmac");
  run("mma.s8 k32", k_mma_s8, (int*)out, 4.0 * 16 * 8 * 32 / 32, sms, ghz, "mac");
  return 0;
}
