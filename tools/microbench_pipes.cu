// microbench_pipes.cu -- measured issue rates of the integer / FP64 pipes on the
// box's B200 (per SM per clock), to ground the IMAD roofline used by bench.py
// and to choose the limb-product formulation.  Build + run on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1410_1599_b200/csrc \
//        tools/microbench_pipes.cu -o /tmp/mb && /tmp/mb
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include "mp_arith.cuh"

constexpr int ITERS = 4096;
constexpr int CH = 8;  // independent chains per thread

template <int OP>
__global__ void kern(uint32_t seed, uint32_t* out, long long* cyc) {
  uint32_t x[CH], y = seed * 2654435761u + threadIdx.x, z = seed ^ 0x9e3779b9u;
  uint64_t w[CH];
  const uint64_t zz = ((uint64_t)z << 32) | (seed * 977u);
  uint32_t v[CH];
  double d[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) { x[c] = y + c; w[c] = x[c]; v[c] = x[c] ^ 5u; d[c] = 1.0 + c * 1e-3; }
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (OP == 0) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(y), "r"(z));
      if (OP == 1) asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(y), "r"(z));
      // loop-carried multiplier (the low word of the running value): nothing to hoist
      if (OP == 2)
        asm volatile("{.reg .u32 t; cvt.u32.u64 t, %0; mad.wide.u32 %0, t, %1, %2;}" : "+l"(w[c]) : "r"(y), "l"(zz));
      if (OP == 3) asm volatile("add.u32 %0, %0, %1; add.u32 %0, %0, %2;" : "+r"(x[c]) : "r"(y), "r"(z));
      if (OP == 4) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(y), "r"(z));
      if (OP == 5) asm volatile("shf.l.wrap.b32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(y), "r"(z));
      if (OP == 6) asm volatile("fma.rn.f64 %0, %0, %0, %0;" : "+d"(d[c]));
      if (OP == 7) {  // 1 IMAD + 1 LOP3 interleaved (co-issue test)
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(y), "r"(z));
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(v[c]) : "r"(y), "r"(z));
      }
      if (OP == 8) {  // carry chain pair as the limb product emits (mad.lo.cc / madc.hi)
        asm volatile("mad.lo.cc.u32 %0, %0, %1, %2; madc.hi.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(y), "r"(z));
      }
    }
  }
  long long t1 = clock64();
  uint32_t acc = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) acc ^= x[c] ^ v[c] ^ (uint32_t)w[c] ^ (uint32_t)(w[c] >> 32) ^ (uint32_t)(uint64_t)d[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// full L-limb product throughput with the library's mul_full (IMAD-eq = 2 L^2)
template <int L>
__global__ void kmul(uint32_t seed, uint32_t* out, long long* cyc) {
  uint32_t a[L], b[L], r[2 * L];
#pragma unroll
  for (int i = 0; i < L; ++i) { a[i] = seed * (i + 7) + threadIdx.x; b[i] = seed ^ (i * 977 + threadIdx.x); }
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < 256; ++it) {
    mpg::mul_full<L>(a, b, r);
#pragma unroll
    for (int i = 0; i < L; ++i) a[i] ^= r[i + L / 2];
  }
  long long t1 = clock64();
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < L; ++i) acc ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// one MP madd (mp_mul + mp_add) per iteration: full primitive cost
template <int L>
__global__ void kmadd(uint32_t seed, uint32_t* out, long long* cyc) {
  mpg::MP<L> a, b, acc, t;
#pragma unroll
  for (int i = 0; i < L; ++i) { a.m[i] = seed * (i + 7) + threadIdx.x; b.m[i] = seed ^ (i * 977 + threadIdx.x); }
  a.m[L - 1] |= 0x80000000u; b.m[L - 1] |= 0x80000000u;
  a.e = 0; b.e = 1; a.s = threadIdx.x & 1; b.s = 0;
  mpg::mp_zero(acc);
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < 128; ++it) {
    mpg::mp_mul<L>(a, b, 0, t);
    mpg::MP<L> r;
    mpg::mp_add<L>(acc, t, 0u, 0, r);
    acc = r;
    b.m[0] ^= acc.m[0];
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.m[0] ^ acc.e;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// mp_mul alone (short product + rounding) and mp_add alone, L limbs
template <int L>
__global__ void kmulonly(uint32_t seed, uint32_t* out, long long* cyc) {
  mpg::MP<L> a, b, t;
#pragma unroll
  for (int i = 0; i < L; ++i) { a.m[i] = seed * (i + 7) + threadIdx.x; b.m[i] = seed ^ (i * 977 + threadIdx.x); }
  a.m[L - 1] |= 0x80000000u; b.m[L - 1] |= 0x80000000u;
  a.e = 0; b.e = 1; a.s = threadIdx.x & 1; b.s = 0;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < 128; ++it) {
    mpg::mp_mul<L>(a, b, 0, t);
    b.m[0] ^= t.m[1];
    b.m[L - 1] |= 0x80000000u;
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = b.m[0] ^ t.e;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int L>
__global__ void kaddonly(uint32_t seed, uint32_t* out, long long* cyc) {
  mpg::MP<L> acc, t;
#pragma unroll
  for (int i = 0; i < L; ++i) { acc.m[i] = seed * (i + 7) + threadIdx.x; t.m[i] = seed ^ (i * 977 + threadIdx.x); }
  acc.m[L - 1] |= 0x80000000u; t.m[L - 1] |= 0x80000000u;
  acc.e = 3; t.e = 1; acc.s = 0; t.s = threadIdx.x & 1;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < 128; ++it) {
    mpg::mp_add<L>(acc, t, 0u, 0, acc);
    t.m[0] ^= acc.m[0];
    t.s ^= acc.m[1] & 1u;
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.m[0] ^ acc.e;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <class K>
double run(K k, const char* name, double ops_per_thread_iter, int iters, int threads, int blocks_per_sm) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int blocks = sms * blocks_per_sm;
  uint32_t* out; long long* cyc;
  cudaMalloc(&out, sizeof(uint32_t) * blocks * threads);
  cudaMalloc(&cyc, sizeof(long long) * blocks);
  k<<<blocks, threads>>>(1u, out, cyc);  // warm
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<blocks, threads>>>(2u, out, cyc);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
  std::vector<long long> c(blocks);
  cudaMemcpy(c.data(), cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
  std::sort(c.begin(), c.end());
  double med = (double)c[blocks / 2];
  // per-SM rate: blocks_per_sm blocks co-resident, each threads * iters * ops
  double per_clk_sm = blocks_per_sm * (double)threads * iters * ops_per_thread_iter / med;
  double total = (double)blocks * threads * iters * ops_per_thread_iter;
  printf("{\"op\": \"%s\", \"ops_per_clk_per_sm\": %.2f, \"ops_per_s\": %.4e, \"ms\": %.3f, \"med_cycles\": %.0f, \"err\": \"%s\"}\n",
         name, per_clk_sm, total / (ms * 1e-3), ms, med, cudaGetErrorString(err));
  cudaFree(out); cudaFree(cyc);
  return per_clk_sm;
}

int main() {
  const int T = 256, B = 4;
  run(kern<0>, "IMAD (mad.lo.u32)", CH, ITERS, T, B);
  run(kern<1>, "IMAD.HI (mad.hi.u32)", CH, ITERS, T, B);
  run(kern<2>, "IMAD.WIDE.U32 (mad.wide.u32, loop-carried; 1 op = 1 instruction = 2 IMAD-eq)", CH, ITERS, T, B);
  run(kern<3>, "IADD (2 add.u32 -> IADD3?)", 2 * CH, ITERS, T, B);
  run(kern<4>, "LOP3", CH, ITERS, T, B);
  run(kern<5>, "SHF", CH, ITERS, T, B);
  run(kern<6>, "DFMA", CH, ITERS, T, B);
  run(kern<7>, "IMAD+LOP3 pairs (count IMAD)", CH, ITERS, T, B);
  run(kern<8>, "mad.lo.cc+madc.hi pairs (count IMAD-eq=2)", 2 * CH, ITERS, T, B);
  run(kmul<4>, "mul_full<4> (IMAD-eq 2L^2)", 2 * 4 * 4, 256, T, B);
  run(kmul<8>, "mul_full<8> (IMAD-eq 2L^2)", 2 * 8 * 8, 256, T, B);
  run(kmul<16>, "mul_full<16> (IMAD-eq 2L^2)", 2 * 16 * 16, 256, T, 2);
  run(kmul<32>, "mul_full<32> (IMAD-eq 2L^2)", 2 * 32 * 32, 256, 128, 2);
  run(kmadd<8>, "mp_mul+mp_add L=8 (IMAD-eq 2L^2)", 2 * 8 * 8, 128, T, B);
  run(kmulonly<8>, "mp_mul only L=8 (IMAD-eq 2L^2)", 2 * 8 * 8, 128, T, B);
  run(kaddonly<8>, "mp_add only L=8 (count 1 op = 128 'IMAD-eq')", 2 * 8 * 8, 128, T, B);
  run(kmadd<32>, "mp_mul+mp_add L=32 (IMAD-eq 2L^2)", 2 * 32 * 32, 128, 128, 2);
  return 0;
}
