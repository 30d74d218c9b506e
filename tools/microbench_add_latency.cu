// Latency of a dependent chain of MP operations in ONE thread (the exact back
// substitution's and the LU panel's critical path), vs the throughput kernels' use.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -Ipaper_1410_1599_b200/csrc tools/microbench_add_latency.cu -o /tmp/mb_add && /tmp/mb_add
#include <cstdio>
#include <cuda_runtime.h>

#include "mp_arith.cuh"

using namespace mpg;

template <int L>
__global__ void chain_add(const uint32_t* t_rec, int n, uint32_t* out, long long* cycles) {
  MP<L> acc, t;
  load_rec<L>(t_rec, acc);
  const long long c0 = clock64();
  for (int s = 0; s < n; ++s) {
    load_rec<L>(t_rec + (1 + (s & 63)) * rec_stride(L), t);
    mp_add<L>(acc, t, 1u, 0, acc);
  }
  const long long c1 = clock64();
  store_rec<L>(out, acc);
  *cycles = c1 - c0;
}

template <int L>
__global__ void chain_madd(const uint32_t* t_rec, int n, uint32_t* out, long long* cycles) {
  MP<L> acc, a, b, p;
  load_rec<L>(t_rec, acc);
  const long long c0 = clock64();
  for (int s = 0; s < n; ++s) {
    load_rec<L>(t_rec + (1 + (s & 63)) * rec_stride(L), a);
    load_rec<L>(t_rec + (1 + ((s + 7) & 63)) * rec_stride(L), b);
    mp_mul<L>(a, b, 0, p);
    mp_add<L>(acc, p, 1u, 0, acc);
  }
  const long long c1 = clock64();
  store_rec<L>(out, acc);
  *cycles = c1 - c0;
}

template <int L>
void run() {
  constexpr int S = rec_stride(L);
  uint32_t h[65 * S] = {};
  unsigned long long x = 0x9E3779B97F4A7C15ull;
  for (int e = 0; e < 65; ++e) {
    for (int k = 0; k < L; ++k) {
      x ^= x << 13; x ^= x >> 7; x ^= x << 17;
      h[e * S + k] = (uint32_t)x;
    }
    h[e * S + L - 1] |= 0x80000000u;
    h[e * S + L] = (uint32_t)(int)((x >> 40) % 5) - 2;  // exponents -2 .. 2
    h[e * S + L + 1] = (uint32_t)(x >> 63);
  }
  uint32_t *d, *o;
  long long* c;
  cudaMalloc(&d, sizeof h);
  cudaMalloc(&o, 4 * S);
  cudaMalloc(&c, 8);
  cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice);
  const int n = 20000;
  long long cy = 0;
  chain_add<L><<<1, 1>>>(d, n, o, c);
  chain_add<L><<<1, 1>>>(d, n, o, c);
  cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
  std::printf("L=%2d dependent mp_add : %7.1f cycles / op\n", L, (double)cy / n);
  chain_madd<L><<<1, 1>>>(d, n, o, c);
  chain_madd<L><<<1, 1>>>(d, n, o, c);
  cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
  std::printf("L=%2d dependent mul+add: %7.1f cycles / op\n", L, (double)cy / n);
  cudaFree(d);
  cudaFree(o);
  cudaFree(c);
}

int main() {
  run<4>();
  run<8>();
  run<16>();
  return 0;
}
