// tc_probe.cu -- A/B of the K2 score contraction at the GQA-4 1-bit geometry
// (C3/C4: 8 query rows per KV head, d = 128, 32-token blocks with per-block
// per-channel key scales): legacy mma.sync (what K2 ships) against a tcgen05
// variant (A = expanded codes in TMEM, B = the per-block Q*s hi/lo in shared
// memory, accumulators in TMEM, one elected thread issuing the MMAs).
//
// Both variants compute, for every 32-token block b and query row j,
//   S[b][t][j] = sum_c code[b][t][c] * Q[j][c] * s[b][c],  s = (hi - lo) / 2
// from the same HBM inputs (1-bit key codes 512 B + key params 512 B per
// block), with the same B-operand precision (f16 hi + lo of Q*s, ~22 bits),
// and differ only in how the contraction is issued:
//   M (mma.sync): per warp and block, B fragments via shared memory, 2 m-tiles
//     x 8 k-steps x (hi, lo) = 32 HMMA.16816 -- K2's score phase (attend_mma.cu).
//   T (tcgen05): per CTA of 4 warps and 4 blocks (one per warp, tokens on the
//     M = 128 TMEM lanes), every thread expands its token's 128 code bits into
//     64 f16x2 registers and stores them to TMEM (tcgen05.st 32x32b.x64); the
//     warp builds its block's 16 B rows (8 hi + 8 lo) of a block-diagonal
//     N = 64 operand in the canonical K-major layout; one thread issues 8
//     tcgen05.mma (M128 N64 K16, A from TMEM) per 4 blocks; the epilogue reads
//     its block's 16 accumulator columns back (tcgen05.ld 32x32b.x16).
//     Two stages (TMEM A/D and shared B), so block i's MMAs overlap block
//     i+1's expansion and block i-1's epilogue.
// The block-diagonal N wastes 3/4 of the tensor work (the scale s varies
// along the contraction index and changes every block); it is the price of
// M = 128 rows.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/tc_probe.cu -o tools/tc_probe
//   tools/tc_probe [nblocks]     (prints one JSON line per variant + the check)
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      std::exit(1);                                                                  \
    }                                                                                \
  } while (0)

constexpr int NR = 8;  // query rows per KV head (GQA-4 x {output, speculative})

// ---- shared helpers ------------------------------------------------------------------------
__device__ __forceinline__ uint32_t pack_f16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ void split2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  hi = pack_f16x2(x0, x1);
  __half2 h = *reinterpret_cast<__half2*>(&hi);
  float2 hf = __half22float2(h);
  lo = pack_f16x2(x0 - hf.x, x1 - hf.y);
}
// (hi, lo) of the product of two hi + lo f16x2 pairs (K2's mul_hilo)
__device__ __forceinline__ void mul_hilo(uint32_t ah, uint32_t al, uint32_t bh, uint32_t bl, uint32_t& hi,
                                         uint32_t& lo) {
  asm("{\n\t.reg .b32 nh, e;\n\t"
      "mul.rn.f16x2 %0, %2, %4;\n\t"
      "neg.f16x2 nh, %0;\n\t"
      "fma.rn.f16x2 e, %2, %4, nh;\n\t"
      "fma.rn.f16x2 e, %2, %5, e;\n\t"
      "fma.rn.f16x2 %1, %3, %4, e;\n\t}"
      : "=r"(hi), "=r"(lo)
      : "r"(ah), "r"(al), "r"(bh), "r"(bl));
}
__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ float s_of(uint32_t w) {  // (lo | hi << 16) bf16 -> (hi - lo) / 2
  return (__uint_as_float(w & 0xFFFF0000u) - __uint_as_float(w << 16)) * 0.5f;
}

struct Args {
  const uint32_t* codes;   // [nb][32 tokens][4 words]: word tq, bit ks (+8 sh, +16 half) -> ch 32tq+8sh+ks+16half
  const uint32_t* params;  // [nb][128 channels] bf16 (lo | hi << 16)
  const float* q;          // [NR][128]
  float* check;            // [nverify][32][NR] scores of the first blocks
  float* sink;             // per-thread checksums
  int nb, nverify;
};

// ---- variant M: K2's score phase on mma.sync ------------------------------------------------
// lane (kks = lane & 7, ktk = lane >> 3) owns channels 32ktk + kks + 8m (m = 0..3) for the
// B build; the fragment lane (gq, tq) reads rows gq, K pairs (2tq, 2tq+1), (2tq+8, 2tq+9).
__global__ void __launch_bounds__(256, 2) k_mma(Args a) {
  __shared__ __align__(16) uint4 bk_all[8][8][4 * NR + 4];
  __shared__ __align__(16) uint4 qh_s[NR][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gq = lane >> 2, tq = lane & 3;
  const int kks = lane & 7, ktk = lane >> 3;
  uint4(*bk)[4 * NR + 4] = bk_all[warp];
  if (warp == 0) {  // Q * 2^-kks as f16 hi/lo pairs b0 = (m0, m2), b1 = (m1, m3)
    for (int j = 0; j < NR; ++j) {
      float qv[4];
      for (int m = 0; m < 4; ++m) qv[m] = a.q[j * 128 + 32 * ktk + kks + 8 * m] * exp2f(-(float)kks);
      uint4 h;
      split2(qv[0], qv[2], h.x, h.z);
      split2(qv[1], qv[3], h.y, h.w);
      qh_s[j][lane] = h;
    }
  }
  __syncthreads();
  float chk = 0.f;
  const int wstride = gridDim.x * 8;
  // inputs of the next block are loaded one iteration ahead (registers)
  uint32_t np[4], nk[2][2];
  auto fetch = [&](int b) {
#pragma unroll
    for (int m = 0; m < 4; ++m) np[m] = b < a.nb ? __ldg(a.params + (size_t)b * 128 + 32 * ktk + kks + 8 * m) : 0u;
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int hf = 0; hf < 2; ++hf)
        nk[mt][hf] = b < a.nb ? __ldg(a.codes + ((size_t)b * 32 + 16 * mt + gq + 8 * hf) * 4 + tq) : 0u;
  };
  fetch(blockIdx.x * 8 + warp);
  for (int b = blockIdx.x * 8 + warp; b < a.nb; b += wstride) {
    float s4[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) s4[m] = s_of(np[m]);
    uint32_t kw[2][2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) kw[mt][hf] = nk[mt][hf];
    fetch(b + wstride);
    uint32_t sh0, sl0, sh1, sl1;
    split2(s4[0], s4[2], sh0, sl0);
    split2(s4[1], s4[3], sh1, sl1);
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      const uint4 qh = qh_s[j][lane];
      uint4 frag;
      mul_hilo(qh.x, qh.z, sh0, sl0, frag.x, frag.z);
      mul_hilo(qh.y, qh.w, sh1, sl1, frag.y, frag.w);
      bk[kks][4 * j + (ktk ^ ((kks >> 1) & 3))] = frag;
    }
    __syncwarp();
    float dk[2][4], dl[2][4];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int i = 0; i < 4; ++i) dk[mt][i] = dl[mt][i] = 0.f;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const uint4 bb = bk[ks][4 * gq + (tq ^ ((ks >> 1) & 3))];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const uint32_t msk = (1u << ks) | (1u << (16 + ks));
        const uint32_t a0 = kw[mt][0] & msk, a2 = (kw[mt][0] >> 8) & msk;
        const uint32_t a1 = kw[mt][1] & msk, a3 = (kw[mt][1] >> 8) & msk;
        mma16816(dk[mt], a0, a1, a2, a3, bb.x, bb.y);
        mma16816(dl[mt], a0, a1, a2, a3, bb.z, bb.w);
      }
    }
    __syncwarp();
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int hf = 0; hf < 2; ++hf)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const float sc = (dk[mt][2 * hf + e] + dl[mt][2 * hf + e]) * 16777216.f;
          chk += sc;
          if (b < a.nverify) a.check[((size_t)b * 32 + 16 * mt + gq + 8 * hf) * NR + 2 * tq + e] = sc;
        }
  }
  a.sink[blockIdx.x * blockDim.x + threadIdx.x] = chk;
}

// ---- variant T: tcgen05 ----------------------------------------------------------------------
constexpr int kLBO = 8 * 128 + 16;   // bytes between K-adjacent core matrices (padded: conflict-free stores)
constexpr int kBBytes = 16 * kLBO;   // one stage's B: 16 K chunks x 8 N groups x 128 B (+ pad)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {  // K-major, no swizzle, SBO = 128, LBO = kLBO
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((kLBO >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((128 >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm_100)
  return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}
// kind::f16 instruction descriptor: D f32, A/B f16, K-major both, N = 64, M = 128
constexpr uint32_t kIdesc = (1u << 4) | (0u << 7) | (0u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);

template <int S>  // S = pipeline stages (TMEM A/D + shared B); 128 S TMEM columns per CTA
__global__ void __launch_bounds__(128, 4 / S) k_tc(Args a) {
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* bsm = smem;                                          // [S][kBBytes]
  uint4* qt = reinterpret_cast<uint4*>(smem + S * kBBytes);           // [NR][16 q][2] (hi, lo) x 4 cc
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S * kBBytes + NR * 16 * 2 * 16);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)), "n"(128 * S));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // Q table: K pair cc = 16tq + 8sh + ks holds channels (32tq + 8sh + ks, +16), scaled by 2^-ks
  for (int i = threadIdx.x; i < NR * 64; i += 128) {
    const int j = i >> 6, cc = i & 63, tq = cc >> 4, sh = (cc >> 3) & 1, ks = cc & 7;
    const int ch = 32 * tq + 8 * sh + ks;
    const float sc = exp2f(-(float)ks);
    uint32_t h, l;
    split2(a.q[j * 128 + ch] * sc, a.q[j * 128 + ch + 16] * sc, h, l);
    reinterpret_cast<uint32_t*>(qt)[(j * 16 + (cc >> 2)) * 8 + (cc & 3)] = h;
    reinterpret_cast<uint32_t*>(qt)[(j * 16 + (cc >> 2)) * 8 + 4 + (cc & 3)] = l;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = *tslot;
  const uint32_t tlane = (uint32_t)(32 * warp) << 16;
  // B-build role: rows 4 rgrp .. 4 rgrp + 3, 16-byte K chunk q = 4tq + 2sh + kg (pairs cc = 4q .. 4q+3)
  const int rgrp = lane >> 4, q = ((lane >> 2) & 3) * 4 + ((lane >> 1) & 1) * 2 + (lane & 1);
  const int ch0 = 32 * ((lane >> 2) & 3) + 8 * ((lane >> 1) & 1) + 4 * (lane & 1);  // channel of (cc = 4q, half 0)
  float chk = 0.f;
  const int ntile = (a.nb + 3) / 4;
  int it = 0;
  int prev_b = -1;
// epilogue of a finished tile: its 16 accumulator columns of this warp's block
  auto epilogue = [&](int pst, int pit, int pb) {
    mbar_wait(&bar[pst], (pit / S) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    uint32_t v[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
        "[%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(tbase + tlane + 64 * S + 64 * pst + 16 * warp));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      const float sc = (__uint_as_float(v[j]) + __uint_as_float(v[8 + j])) * 16777216.f;
      chk += sc;
      if (pb >= 0 && pb < a.nverify) a.check[((size_t)pb * 32 + lane) * NR + j] = sc;
    }
  };
  uint4 nw4, np0, np1;  // the next tile's inputs, loaded one iteration ahead
  auto fetch = [&](int tile) {
    const int b = tile * 4 + warp;
    nw4 = np0 = np1 = make_uint4(0u, 0u, 0u, 0u);
    if (b < a.nb) {
      nw4 = __ldg(reinterpret_cast<const uint4*>(a.codes + ((size_t)b * 32 + lane) * 4));
      np0 = __ldg(reinterpret_cast<const uint4*>(a.params + (size_t)b * 128 + ch0));
      np1 = __ldg(reinterpret_cast<const uint4*>(a.params + (size_t)b * 128 + ch0 + 16));
    }
  };
  fetch(blockIdx.x);
  for (int tile = blockIdx.x; tile < ntile + 0; tile += gridDim.x, ++it) {
    const int st = S == 1 ? 0 : it & 1;
    const int b = tile * 4 + warp;
    const bool live = b < a.nb;
    const uint4 w4 = nw4, p0 = np0, p1 = np1;
    fetch(tile + gridDim.x);
    // (1) A: this thread's token -> 64 f16x2 code registers -> TMEM lanes 32w + t, columns 64 st ..
    {
      const uint32_t ww[4] = {w4.x, w4.y, w4.z, w4.w};
      uint32_t r[64];
#pragma unroll
      for (int tq = 0; tq < 4; ++tq)
#pragma unroll
        for (int sh = 0; sh < 2; ++sh)
#pragma unroll
          for (int ks = 0; ks < 8; ++ks)
            r[16 * tq + 8 * sh + ks] = (ww[tq] >> (8 * sh)) & ((1u << ks) | (1u << (16 + ks)));
      const uint32_t ta = tbase + tlane + 64 * st;
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x64.b32 [%0], {"
          "%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
          "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,"
          "%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,"
          "%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63,%64};" ::"r"(ta),
          "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
          "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
          "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
          "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]), "r"(r[32]),
          "r"(r[33]), "r"(r[34]), "r"(r[35]), "r"(r[36]), "r"(r[37]), "r"(r[38]), "r"(r[39]), "r"(r[40]),
          "r"(r[41]), "r"(r[42]), "r"(r[43]), "r"(r[44]), "r"(r[45]), "r"(r[46]), "r"(r[47]), "r"(r[48]),
          "r"(r[49]), "r"(r[50]), "r"(r[51]), "r"(r[52]), "r"(r[53]), "r"(r[54]), "r"(r[55]), "r"(r[56]),
          "r"(r[57]), "r"(r[58]), "r"(r[59]), "r"(r[60]), "r"(r[61]), "r"(r[62]), "r"(r[63])
          : "memory");
    }
    // (2) B: block b's 8 hi + 8 lo N rows (n = 16 warp + {j, 8 + j}) into the K-major core matrices
    {
      uint32_t sh2[4], sl2[4];
      if (live) {
        split2(s_of(p0.x), s_of(p1.x), sh2[0], sl2[0]);
        split2(s_of(p0.y), s_of(p1.y), sh2[1], sl2[1]);
        split2(s_of(p0.z), s_of(p1.z), sh2[2], sl2[2]);
        split2(s_of(p0.w), s_of(p1.w), sh2[3], sl2[3]);
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) sh2[i] = sl2[i] = 0u;
      }
      unsigned char* bs = bsm + st * kBBytes + q * kLBO;
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int j = 4 * rgrp + jj;
        const uint4 qh = qt[(j * 16 + q) * 2], ql = qt[(j * 16 + q) * 2 + 1];
        uint4 oh, ol;
        mul_hilo(qh.x, ql.x, sh2[0], sl2[0], oh.x, ol.x);
        mul_hilo(qh.y, ql.y, sh2[1], sl2[1], oh.y, ol.y);
        mul_hilo(qh.z, ql.z, sh2[2], sl2[2], oh.z, ol.z);
        mul_hilo(qh.w, ql.w, sh2[3], sl2[3], oh.w, ol.w);
        *reinterpret_cast<uint4*>(bs + (2 * warp) * 128 + j * 16) = oh;      // N group 2w: hi rows
        *reinterpret_cast<uint4*>(bs + (2 * warp + 1) * 128 + j * 16) = ol;  // N group 2w+1: lo rows
      }
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    // (3) one thread issues the 8 K-steps of this tile
    if (threadIdx.x == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t bbase = smem_u32(bsm + st * kBBytes);
      const uint32_t dcol = tbase + 64 * S + 64 * st, acol = tbase + 64 * st;
      const uint32_t mask0 = 0u;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint64_t bd = sdesc(bbase + 2 * k * kLBO);
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, {%5, %5, %5, %5}, p;\n\t}"
            ::"r"(dcol), "r"(acol + 8 * k), "l"(bd), "r"(kIdesc), "r"(k), "r"(mask0)
            : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(&bar[st]))
                   : "memory");
    }
    // (4) the previous tile's epilogue overlaps this tile's MMAs
    if (S == 1) {
      epilogue(0, it, b);
    } else if (it > 0) {
      epilogue(st ^ 1, it - 1, prev_b);
    }
    prev_b = b;
  }
  if (S == 2 && it > 0) epilogue((it - 1) & 1, it - 1, prev_b);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(128 * S));
  a.sink[blockIdx.x * blockDim.x + threadIdx.x] = chk;
}

// ---- host --------------------------------------------------------------------------------------
static uint16_t f2bf(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  return (uint16_t)((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
}
static float bf2f(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float x;
  std::memcpy(&x, &u, 4);
  return x;
}

int main(int argc, char** argv) {
  const int nb = argc > 1 ? std::atoi(argv[1]) : 262144;  // C3: 8 seqs x 8 KV heads x 4096 blocks
  const int nverify = 64;
  std::vector<uint32_t> codes((size_t)nb * 128), params((size_t)nb * 128);
  std::vector<float> q(NR * 128);
  uint64_t x = 88172645463325252ull;
  auto rnd = [&]() {
    x ^= x << 13;
    x ^= x >> 7;
    x ^= x << 17;
    return x;
  };
  for (auto& c : codes) c = (uint32_t)rnd();
  for (size_t i = 0; i < params.size(); ++i) {
    const float lo = -0.5f - (rnd() % 1000) / 500.f, hi = 0.5f + (rnd() % 1000) / 500.f;
    params[i] = (uint32_t)f2bf(lo) | ((uint32_t)f2bf(hi) << 16);
  }
  for (auto& v : q) v = ((int)(rnd() % 2001) - 1000) / 250.f;
  uint32_t *dc, *dp;
  float *dq, *dchk, *dsink;
  CK(cudaMalloc(&dc, codes.size() * 4));
  CK(cudaMalloc(&dp, params.size() * 4));
  CK(cudaMalloc(&dq, q.size() * 4));
  CK(cudaMalloc(&dchk, (size_t)nverify * 32 * NR * 4));
  CK(cudaMalloc(&dsink, 1 << 24));
  CK(cudaMemcpy(dc, codes.data(), codes.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dp, params.data(), params.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dq, q.data(), q.size() * 4, cudaMemcpyHostToDevice));
  // CPU reference for the first nverify blocks
  std::vector<double> ref((size_t)nverify * 32 * NR);
  double refmax = 0;
  for (int b = 0; b < nverify; ++b)
    for (int t = 0; t < 32; ++t)
      for (int j = 0; j < NR; ++j) {
        double s = 0;
        for (int c = 0; c < 128; ++c) {
          const int tq = c >> 5, r = c & 31, half = r >> 4, sh = (r >> 3) & 1, ks = r & 7;
          const uint32_t w = codes[((size_t)b * 32 + t) * 4 + tq];
          const int bit = (w >> (8 * sh + 16 * half + ks)) & 1;
          const uint32_t p = params[(size_t)b * 128 + c];
          const double sc = ((double)bf2f(p >> 16) - (double)bf2f(p & 0xFFFF)) * 0.5;
          s += bit * (double)q[j * 128 + c] * sc;
        }
        ref[((size_t)b * 32 + t) * NR + j] = s;
        refmax = std::fmax(refmax, std::fabs(s));
      }
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  Args a{dc, dp, dq, dchk, dsink, nb, nverify};
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto tc_smem = [](int S) { return (size_t)S * kBBytes + NR * 16 * 2 * 16 + 64; };
  CK(cudaFuncSetAttribute(k_tc<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tc_smem(1)));
  CK(cudaFuncSetAttribute(k_tc<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tc_smem(2)));
  const char* names[3] = {"mma.sync (K2 score phase), 16 warps/SM",
                          "tcgen05 (TMEM A, block-diagonal N=64), 2 stages, 2 CTAs x 4 warps/SM",
                          "tcgen05 (TMEM A, block-diagonal N=64), 1 stage, 4 CTAs x 4 warps/SM"};
  for (int variant = 0; variant < 3; ++variant) {
    auto launch = [&]() {
      if (variant == 0) k_mma<<<sms * 2, 256>>>(a);
      else if (variant == 1) k_tc<2><<<sms * 2, 128, tc_smem(2)>>>(a);
      else k_tc<1><<<sms * 4, 128, tc_smem(1)>>>(a);
    };
    CK(cudaMemset(dchk, 0, (size_t)nverify * 32 * NR * 4));
    launch();
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<float> got((size_t)nverify * 32 * NR);
    CK(cudaMemcpy(got.data(), dchk, got.size() * 4, cudaMemcpyDeviceToHost));
    double maxerr = 0;
    for (size_t i = 0; i < got.size(); ++i) maxerr = std::fmax(maxerr, std::fabs(got[i] - ref[i]));
    for (int w = 0; w < 3; ++w) launch();
    CK(cudaEventRecord(e0));
    const int reps = 10;
    for (int r = 0; r < reps; ++r) launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    ms /= reps;
    const double bytes = (double)nb * 1024.0;
    std::printf(
        "{\"variant\": \"%s\", \"blocks\": %d, \"ms\": %.4f, \"clk_per_block_per_sm_at_1965\": %.1f, "
        "\"input_gbs\": %.1f, \"max_abs_err_vs_fp64\": %.3e, \"ref_max\": %.3e}\n",
        names[variant], nb, ms,
        ms * 1e-3 * 1.965e9 * sms / nb, bytes / (ms * 1e-3) / 1e9, maxerr, refmax);
  }
  return 0;
}
