// tc_probe.cu -- validates the tcgen05 (kind::i8) building blocks used by the
// tensor-core MP product: TMEM alloc, K-major SWIZZLE_NONE smem descriptors, the
// unsigned-int8 MMA, commit -> mbarrier, tcgen05.ld.  Computes byte convolutions
//   D[j][t] = sum_s B_j[s] * A[t - s]      (j < 128, t < N, s < K bytes)
// i.e. the exact limb-product columns of 128 MP mantissas B_j by one mantissa A,
// and compares with a CPU reference.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/tc_probe.cu -o /tmp/tcp && /tmp/tcp
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#ifndef KB
#define KB 32  // mantissa bytes (L = KB/4 limbs)
#endif
#ifndef MM
#define MM 128
#endif
#ifndef LANE_OFF
#define LANE_OFF 0  // TMEM lane offset of the MMA's D (probe: 16 = upper half of each quadrant)
#endif
constexpr int M = MM;
constexpr int K = KB;          // MMA K extent in bytes (multiple of 32)
constexpr int N = 2 * KB;      // conv columns computed (2K-1 needed)
constexpr int SBO = (K / 16) * 128;  // bytes between 8-row groups (K-major, no swizzle)
constexpr int LBO = 128;             // bytes between the 16-byte K chunks

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// canonical K-major SWIZZLE_NONE offset of byte (row r, k) for a tile with K bytes per row
__host__ __device__ __forceinline__ int kmaj_off(int r, int k) {
  return (r >> 3) * SBO + (k >> 4) * LBO + (r & 7) * 16 + (k & 15);
}
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((LBO >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((SBO >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version = 1 (Blackwell)
  // base_offset 0, lbo_mode 0, layout_type 0 = SWIZZLE_NONE
  return d;
}
__host__ __device__ constexpr uint32_t idesc_u8(int m, int n) {
  // c_format S32 = 2 @ [4,6); a/b format u8 = 0; K-major a/b = 0; n>>3 @ [17,23); m>>4 @ [24,29)
  return (2u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__global__ void __launch_bounds__(128) probe(const uint8_t* __restrict__ bmat /*128 x K*/,
                                             const uint8_t* __restrict__ a /*K*/, uint32_t* out /*128 x N*/,
                                             uint32_t* err) {
  extern __shared__ __align__(1024) uint8_t dsm[];
  uint8_t* sA = dsm;            // A-operand: rows j = B_j bytes (M x K)
  uint8_t* sB = dsm + M * K;    // B-operand: Toeplitz rows t (N x K)
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < M * K; e += 128) sA[kmaj_off(e / K, e % K)] = bmat[e];
  for (int e = tid; e < N * K; e += 128) {
    const int t = e / K, s = e % K;
    const int x = t - s;
    sB[kmaj_off(t, s)] = (x >= 0 && x < K) ? a[x] : 0;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(N < 32 ? 32 : N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&mbar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = idesc_u8(M, N);
    for (int kc = 0; kc < K / 32; ++kc) {
      const uint64_t da = smem_desc(smem_u32(sA) + kc * 2 * LBO);
      const uint64_t db = smem_desc(smem_u32(sB) + kc * 2 * LBO);
      const uint32_t acc = kc > 0;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tbase + ((uint32_t)LANE_OFF << 16)),
          "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        smem_u32(&mbar)));
  }
  // wait for the MMA (bounded spin)
  {
    uint32_t done = 0;
    for (int it = 0; it < 1000000 && !done; ++it) {
      asm volatile(
          "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
          "selp.u32 %0, 1, 0, P1;\n\t}"
          : "=r"(done)
          : "r"(smem_u32(&mbar)), "r"(0));
    }
    if (!done) atomicOr(err, 1u);
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  // each warp reads its 32 lanes; 16 columns per tcgen05.ld
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t v[16];
    const uint32_t taddr = tbase + ((uint32_t)(warp * 32) << 16) + c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int q = 0; q < 16; ++q) out[(warp * 32 + lane) * N + c0 + q] = v[q];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(N < 32 ? 32 : N));
}

int main() {
  std::vector<uint8_t> hb(128 * K), ha(K);
  uint64_t s = 12345;
  auto rnd = [&] { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return (uint8_t)(s >> 24); };
  for (auto& x : hb) x = rnd();
  for (auto& x : ha) x = rnd();
  uint8_t *db, *da;
  uint32_t *dout, *derr;
  cudaMalloc(&db, M * K);
  cudaMalloc(&da, K);
  cudaMalloc(&dout, 4 * 128 * N);
  cudaMalloc(&derr, 4);
  cudaMemset(derr, 0, 4);
  cudaMemset(dout, 0xFF, 4 * 128 * N);
  cudaMemcpy(db, hb.data(), M * K, cudaMemcpyHostToDevice);
  cudaMemcpy(da, ha.data(), K, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, M * K + N * K);
  probe<<<1, 128, M * K + N * K>>>(db, da, dout, derr);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<uint32_t> out(128 * N);
  uint32_t herr = 0;
  cudaMemcpy(out.data(), dout, 4 * 128 * N, cudaMemcpyDeviceToHost);
  cudaMemcpy(&herr, derr, 4, cudaMemcpyDeviceToHost);
  long bad = 0;
  if (M == 64) {  // locate each row of D among the 128 TMEM lanes (probe reads lanes 0..127)
    for (int j = 0; j < 64; ++j) {
      int found = -1;
      for (int lane = 0; lane < 128 && found < 0; ++lane) {
        bool ok = true;
        for (int t = 0; t < N && ok; ++t) {
          uint32_t ref = 0;
          for (int k = 0; k < K; ++k)
            if (t - k >= 0 && t - k < K) ref += (uint32_t)hb[j * K + k] * ha[t - k];
          ok = out[lane * N + t] == ref;
        }
        if (ok) found = lane;
      }
      if (j < 4 || j > 60 || found < 0) printf("row %d -> lane %d\n", j, found);
      if (found < 0) ++bad;
    }
    printf("{\"M\": 64, \"rows_not_found\": %ld, \"cuda\": \"%s\"}\n", bad, cudaGetErrorString(e));
    return bad ? 1 : 0;
  }
  for (int j = 0; j < M; ++j)
    for (int t = 0; t < N; ++t) {
      uint32_t ref = 0;
      for (int k = 0; k < K; ++k)
        if (t - k >= 0 && t - k < K) ref += (uint32_t)hb[j * K + k] * ha[t - k];
      if (out[j * N + t] != ref) {
        if (bad < 5) printf("mismatch j=%d t=%d got %u want %u\n", j, t, out[j * N + t], ref);
        ++bad;
      }
    }
  printf("{\"probe\": \"tcgen05 kind::i8 byte convolution\", \"K\": %d, \"N\": %d, \"cuda\": \"%s\", \"timeout_flag\": %u, "
         "\"mismatches\": %ld}\n", K, N, cudaGetErrorString(e), herr, bad);
  return bad ? 1 : 0;
}
