// IMAD-family / IADD3 issue-rate microbenchmark for sm_100a.
// Each kernel runs many independent dependency chains per thread at full occupancy, so the
// measured rate is the pipe throughput, not latency. Rates are reported per SM per clock
// (warp-instructions x 32 / cycles / SMs), with cycles from clock64() on each SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CHAINS 8
#define ITERS 4096

__device__ __forceinline__ void imad_lo(uint32_t& x, uint32_t a, uint32_t b) {
  asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x) : "r"(a), "r"(b));
}
__device__ __forceinline__ void imad_hi(uint32_t& x, uint32_t a, uint32_t b) {
  asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(x) : "r"(a), "r"(b));
}
// one 4-pair carry-chained row: acc[0..7] += a*{b0..b3} at even offsets; 4 IMAD.WIDE.U32 (P carry)
__device__ __forceinline__ void imad_row4(uint32_t* acc, uint32_t a, const uint32_t* b) {
  asm volatile("mad.lo.cc.u32 %0, %8, %9, %0;\n\tmadc.hi.cc.u32 %1, %8, %9, %1;\n\t"
               "madc.lo.cc.u32 %2, %8, %10, %2;\n\tmadc.hi.cc.u32 %3, %8, %10, %3;\n\t"
               "madc.lo.cc.u32 %4, %8, %11, %4;\n\tmadc.hi.cc.u32 %5, %8, %11, %5;\n\t"
               "madc.lo.cc.u32 %6, %8, %12, %6;\n\tmadc.hi.u32 %7, %8, %12, %7;"
               : "+r"(acc[0]), "+r"(acc[1]), "+r"(acc[2]), "+r"(acc[3]), "+r"(acc[4]), "+r"(acc[5]), "+r"(acc[6]), "+r"(acc[7])
               : "r"(a), "r"(b[0]), "r"(b[1]), "r"(b[2]), "r"(b[3]));
}
// carry-chained pair: mad.lo.cc + madc.hi.cc (fuses to IMAD.WIDE.U32 with P carry) + madc
__device__ __forceinline__ void imad_wide_cc(uint32_t& lo, uint32_t& hi, uint32_t& c, uint32_t a, uint32_t b) {
  asm volatile("mad.lo.cc.u32 %0, %3, %4, %0;\n\tmadc.hi.cc.u32 %1, %3, %4, %1;\n\taddc.u32 %2, %2, 0;"
               : "+r"(lo), "+r"(hi), "+r"(c) : "r"(a), "r"(b));
}
__device__ __forceinline__ void iadd3(uint32_t& x, uint32_t a, uint32_t b) {
  asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %0, %0, %2;" : "+r"(x) : "r"(a), "r"(b));
}
__device__ __forceinline__ void lop3(uint32_t& x, uint32_t a, uint32_t b) {
  asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x) : "r"(a), "r"(b));
}
__device__ __forceinline__ void addcc(uint32_t& x, uint32_t& y, uint32_t a, uint32_t b) {
  asm volatile("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, %1, %3;" : "+r"(x), "+r"(y) : "r"(a), "r"(b));
}

__device__ __forceinline__ void dfma(double& x, double a, double b) {
  asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x) : "d"(a), "d"(b));
}

// FP64 FMA rate (B200 keeps a full FP64 pipe; context for DESIGN.md §9 — not used by the kernels)
__global__ void bench_dfma(uint32_t* out, uint32_t seed, long long* cyc) {
  double x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = 1.0 + 1e-9 * (threadIdx.x + c);
  const double a = 0.999999 + 1e-12 * seed, b = 1e-7 * threadIdx.x;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) dfma(x[c], a, b);
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 12345.0) out[0] = 1;
  if (threadIdx.x == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}

template <int MODE>
__global__ void bench(uint32_t* out, uint32_t seed, long long* cyc) {
  uint32_t x[CHAINS], y[CHAINS], z[CHAINS];
  double fx[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) fx[c] = 1.0 + 1e-9 * (threadIdx.x + c);
  const double fa = 0.999999 + 1e-12 * seed, fb = 1e-7 * threadIdx.x;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) { x[c] = seed + threadIdx.x * 7 + c; y[c] = x[c] ^ 0x5bd1e995u; z[c] = c; }
  uint32_t a = seed * 3 + 1 + threadIdx.x * 2, b = (seed ^ 0x9e3779b9u) + threadIdx.x;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      if (MODE == 0) imad_lo(x[c], a, b);
      if (MODE == 1) imad_hi(x[c], a, b);
      if (MODE == 2 && (c & 3) == 0) { uint32_t bb[4] = {y[c], y[c+1], y[c+2], y[c+3]}; imad_row4(&x[c & 0], x[(c + 4) & 7] ^ a, bb); }
      if (MODE == 3) imad_wide_cc(x[c], y[c], z[c], a, b);
      if (MODE == 4) iadd3(x[c], a, b);
      if (MODE == 5) lop3(x[c], a, b);
      if (MODE == 6) { if ((c & 3) == 0) { uint32_t bb[4] = {y[c], y[c+1], y[c+2], y[c+3]}; imad_row4(&x[c & 0], x[(c + 4) & 7] ^ a, bb); } lop3(z[c], a, b); }   // fma + alu co-issue
      if (MODE == 7) addcc(x[c], y[c], a, b);
      if (MODE == 8) { imad_lo(x[c], a, b); lop3(z[c], a, b); }
      // FP64 next to IMAD.WIDE: does the fp64 pipe run concurrently with the fma-heavy products?
      if (MODE == 9) { if ((c & 3) == 0) { uint32_t bb[4] = {y[c], y[c+1], y[c+2], y[c+3]}; imad_row4(&x[c & 0], x[(c + 4) & 7] ^ a, bb); } dfma(fx[c], fa, fb); }
      if (MODE == 10) { if ((c & 3) == 0) { uint32_t bb[4] = {y[c], y[c+1], y[c+2], y[c+3]}; imad_row4(&x[c & 0], x[(c + 4) & 7] ^ a, bb); } if (c & 1) dfma(fx[c], fa, fb); }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s ^= x[c] ^ y[c] ^ z[c] ^ (uint32_t)(fx[c] * 7.0);
  if (s == 0x12345678u) out[0] = s;
  if (threadIdx.x == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}

template <int MODE>
void run(const char* name, int instr_per_chain_step, int nsm, int threads, int blocks_per_sm) {
  uint32_t* out; long long* cyc; cudaMalloc(&out, 4); cudaMalloc(&cyc, 8);
  int grid = nsm * blocks_per_sm;
  bench<MODE><<<grid, threads>>>(out, 1, cyc);  // warm
  cudaMemset(cyc, 0, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  bench<MODE><<<grid, threads>>>(out, 1, cyc);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  // warp-iterations executed per SM sub-partition (4 SMSPs per SM); one iteration = CHAINS chain steps
  double warp_iters_smsp = (double)grid * threads / 32 * ITERS / nsm / 4;
  double cyc_per_warp_iter = (double)c / warp_iters_smsp;
  double per_sm_clk = instr_per_chain_step * CHAINS * 32.0 * 4 / cyc_per_warp_iter;  // named op, thread-ops/SM/clk
  printf("{\"mode\": \"%s\", \"cyc_per_warp_iter_smsp\": %.3f, \"named_op_thread_per_sm_per_clk\": %.2f, \"ms\": %.3f, \"cycles\": %lld, \"implied_mhz\": %.0f}\n",
         name, cyc_per_warp_iter, per_sm_clk, ms, c, c / (ms * 1e3));
  cudaFree(out); cudaFree(cyc);
}

int main() {
  int dev = 0, nsm = 0, clk = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  printf("{\"device\": \"%s\", \"sms\": %d, \"clock_khz\": %d, \"cc\": \"%d.%d\", \"regs_per_sm\": %d}\n",
         p.name, nsm, clk, p.major, p.minor, p.regsPerMultiprocessor);
  // instructions per chain step in SASS are checked with cuobjdump (tools/sass_count.py)
  run<0>("IMAD", 1, nsm, 256, 4);
  run<1>("IMAD.HI", 1, nsm, 256, 4);
  run<2>("IMAD.WIDE.U32(.X) carry rows", 1, nsm, 256, 4);
  run<3>("IMAD.WIDE.cc+IADD3.X", 1, nsm, 256, 4);
  run<4>("IADD3(2 adds)", 1, nsm, 256, 4);
  run<5>("LOP3", 1, nsm, 256, 4);
  run<6>("IMAD.WIDE rows + LOP3", 1, nsm, 256, 4);
  run<7>("IADD3+IADD3.X pairs", 2, nsm, 256, 4);
  run<8>("IMAD+LOP3", 1, nsm, 256, 4);
  run<9>("IMAD.WIDE rows + DFMA (1:1)", 1, nsm, 256, 4);
  run<10>("IMAD.WIDE rows + DFMA (2:1)", 1, nsm, 256, 4);
  {
    uint32_t* out; long long* cyc; cudaMalloc(&out, 4); cudaMalloc(&cyc, 8);
    const int grid = nsm * 4, threads = 256;
    bench_dfma<<<grid, threads>>>(out, 1, cyc);
    cudaMemset(cyc, 0, 8);
    bench_dfma<<<grid, threads>>>(out, 1, cyc);
    cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double warp_iters_smsp = (double)grid * threads / 32 * ITERS / nsm / 4;
    const double cpi = (double)c / warp_iters_smsp;
    printf("{\"mode\": \"DFMA (fp64 pipe)\", \"cyc_per_warp_iter_smsp\": %.3f, \"named_op_thread_per_sm_per_clk\": %.2f}\n",
           cpi, CHAINS * 32.0 * 4 / cpi);
  }
  return 0;
}
