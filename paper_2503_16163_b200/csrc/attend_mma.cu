// attend_mma.cu -- K2 fast path: fused dequantize + score + softmax + P.V over
// the packed 1/2-bit tier on tensor cores (mma.sync m16n8k16, f16 in, fp32
// accumulate), for d=128, g=32, up to 8 query rows per kv head.
//
// Reference semantics: engine.py:51-63 + kvcache.py:222-243 (see
// attend_generic.cu).  Algebra (per g-token block, per kv head):
//   K~[t,c] = z_c + s_c*code[t,c]          (per-channel key groups)
//   S2[t,j] = sum_c Q[j,c]*K~[t,c]          Q = q * d^-0.5 * log2(e)
//           = C_j + sum_c code[t,c] * (Q[j,c]*s_c),   C_j = sum_c Q[j,c]*z_c
//   V~[t,c] = z_{t,grp(c)} + s_{t,grp(c)}*code[t,c]   (per-token value groups)
//   O[c,j]  = sum_t P[j,t]*z_{t,grp} + sum_t code[t,c] * (P[j,t]*s_{t,grp})
// Both sums over codes are MMAs whose A operand is the packed codes and whose
// B operand is a per-block fp32 product (Q*s, P*s).
//
// Code expansion: one AND moves a 2-bit (1-bit) code pair from a packed word
// into the low mantissa bits of an f16x2 register, i.e. an f16 subnormal
// code * 2^(p-24).  p depends only on the MMA K index (channel for scores,
// token for P.V) -- never on M -- so the 2^-p is folded into B, and 2^24 into
// the fp32 epilogue.  B = x * 2^-p * 2^-E is split into f16 hi + lo (two MMAs,
// ~22 significant bits); E is a per-(seq, head) exponent from the quantizer's
// range maxima that keeps max|B| <= 2^14.  Zero-points never touch the MMA:
// C_j and sum_t P*z are fp32 side sums.
//
// MMA shapes.  Scores: M = 16 tokens, N = 8 query rows (padded), K = 16
// channels.  P.V: M = 16 channels, K = 16 tokens; when rows*4 <= 8 (MHA: 2
// rows) the N = 8 columns hold (value group, row) pairs so that one B
// fragment serves all four value groups and no lane idles in its
// construction ("packed groups", PG); otherwise N = rows and each group has
// its own B fragment.
//
// Work split: grid (nsplit + 1, H, batch), 8 warps per CTA.  A CTA streams a
// contiguous range of 32-token blocks of one (seq, kv head); each warp owns
// every 8th block and keeps its own online-softmax state; the CTA merges its
// warps and writes one (m, l, O) partial.  Per block a warp reads 3072 B
// (2-bit) / 2048 B (1-bit): codes straight into registers (coalesced,
// prefetched one block ahead), group params via cp.async into a shared-memory
// double buffer.  The last split runs the exact segment (pinned slots,
// residual window, in-step rows) with the generic CTA body.
#include <algorithm>

#include "exact_segment.cuh"

namespace spc {
namespace {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;

__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_f16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// x0 -> low half, x1 -> high half; hi + lo carries ~22 significant bits
__device__ __forceinline__ void split2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  hi = pack_f16x2(x0, x1);
  __half2 h = *reinterpret_cast<__half2*>(&hi);
  float2 hf = __half22float2(h);
  lo = pack_f16x2(x0 - hf.x, x1 - hf.y);
}

__device__ __forceinline__ float pow2i(int e) {  // 2^e, e in [-126, 127]
  return __int_as_float((127 + e) << 23);
}

__device__ __forceinline__ int ceil_log2(float x) {  // x > 0
  int e = ilogbf(x);
  return (x > ldexpf(1.f, e)) ? e + 1 : e;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ float warp_max_g(float v) {  // over lanes sharing lane&3
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 4));
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 8));
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 16));
  return v;
}
__device__ __forceinline__ float warp_sum_g(float v) {
  v += __shfl_xor_sync(0xffffffffu, v, 4);
  v += __shfl_xor_sync(0xffffffffu, v, 8);
  v += __shfl_xor_sync(0xffffffffu, v, 16);
  return v;
}
__device__ __forceinline__ float warp_sum_all(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// key-param word of channel c in the swizzled shared copy (conflict-free reads
// of channels {32t + ks + 8m} by lane (ks, t))
__device__ __forceinline__ int kpar_swz(int c) { return c ^ ((c >> 5) << 3); }

template <int NR>
struct WarpSmem {
  uint32_t kpar[2][128];   // key (lo|hi) per channel, swizzled, double buffer
  uint32_t vpar[2][128];   // value (lo|hi) per (token, group)
  uint4 bk[8][32];         // key B fragments {b0hi, b1hi, b0lo, b1lo}, [ks][lane ^ ks]
  float P[NR][33];         // probabilities of the block, [row][token]
};

template <int NR>
struct MergeSmem {
  float o[kWarps][NR][128];
  float m[kWarps][NR];
  float l[kWarps][NR];
};

template <int NR>
constexpr size_t fast_smem_bytes() {
  return sizeof(WarpSmem<NR>) * kWarps > sizeof(MergeSmem<NR>) ? sizeof(WarpSmem<NR>) * kWarps
                                                                 : sizeof(MergeSmem<NR>);
}

template <int BITS, int NR>
__global__ void __launch_bounds__(kThreads, 2) k_attend_fast(AttnArgs a) {
  constexpr bool PG = (NR * 4 <= 8);    // value MMA columns = (group, row) pairs
  constexpr int KW = BITS * 2;          // key-code words per lane per m-tile (2 tokens x BITS words)
  constexpr int VW = BITS * 4;          // value-code words per lane per block
  const Geo& G = a.G;
  const LayerBufs& B = a.B;
  const int split = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  if (split == a.nsplit) {  // exact segment: first 128 threads
    if (threadIdx.x < kCH) generic_cta(a, split, h, b, reinterpret_cast<float*>(smem_raw));
    return;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  WarpSmem<NR>& ws = reinterpret_cast<WarpSmem<NR>*>(smem_raw)[warp];

  const int nb_total = a.f / 32;
  const int blk0 = split * a.blocks_per_split;
  const int blk1 = min(nb_total, blk0 + a.blocks_per_split);
  const float cs = BITS == 1 ? 0.5f : (1.f / 3.f);

  // ---- per-lane query slice for the cooperative key-B construction ----------------
  // lane (ks = lane&7, tk = lane>>3) owns channels 32tk + ks + 8m, m = 0..3
  const int kks = lane & 7, ktk = lane >> 3;
  float Qr[NR][4];
  float qabs = 0.f;
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    const int r = j / G.G, g2 = j - r * G.G;
    const __nv_bfloat16* qp = a.q + (((size_t)b * a.rows + r) * G.Hq + h * G.G + g2) * 128;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      Qr[j][m] = __bfloat162float(qp[32 * ktk + kks + 8 * m]) * a.sm_scale_log2;
      qabs = fmaxf(qabs, fabsf(Qr[j][m]));
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) qabs = fmaxf(qabs, __shfl_xor_sync(0xffffffffu, qabs, o));
  const float rk = __uint_as_float(B.rmax[((size_t)b * G.H + h) * 2 + 0]) * cs;
  const float rv = __uint_as_float(B.rmax[((size_t)b * G.H + h) * 2 + 1]) * cs;
  const int Ek = (qabs * rk > 0.f) ? ceil_log2(qabs * rk) - 14 : 0;
  const int Ev = (rv > 0.f) ? ceil_log2(rv) - 14 : 0;
  // key-side K-index scale of this lane's channels: 2^(-sp - Ek)
  const int sp = BITS == 2 ? 2 * (kks & 3) : kks;
  const float kk_scale = pow2i(-sp - Ek);
  const float k_out = pow2i(24 + Ek);  // D * k_out = sum_c code * Q * s
  const float v_out = pow2i(24 + Ev);

  // zero the unused rows of the key-B fragments once
  for (int i = lane; i < 8 * 32; i += 32) {
    int ks = i >> 5, l = i & 31;
    if ((l >> 2) >= NR) ws.bk[ks][l ^ ks] = make_uint4(0, 0, 0, 0);
  }

  // ---- per-warp running state -------------------------------------------------------
  // score rows owned by this lane: 2tq, 2tq+1
  float m_run[2] = {-CUDART_INF_F, -CUDART_INF_F};
  float l_run[2] = {0.f, 0.f};
  float dv[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) dv[i][0] = dv[i][1] = dv[i][2] = dv[i][3] = 0.f;
  // value zero-point side sums: PG: role (grp, j) = (gq / NR, gq % NR); else j = gq, per grp
  float zacc[PG ? 1 : 4];
#pragma unroll
  for (int i = 0; i < (PG ? 1 : 4); ++i) zacc[i] = 0.f;

  const size_t bi0 = blk_index(G, b, h, 0);
  const uint32_t* kc_base = B.kcodes + bi0 * (size_t)G.bwords;
  const uint32_t* vc_base = B.vcodes + bi0 * (size_t)G.bwords;
  const uint32_t* kp_base = B.kparams + bi0 * 128;
  const uint32_t* vp_base = B.vparams + bi0 * 128;
  const uint32_t* bm_base = B.bitmap + ((size_t)b * G.U + (G.scope ? h : 0)) * (G.L / 32);
  const int agg_j0 = a.agg_row * G.G;

  // code registers (current + prefetched)
  uint32_t kw[2][KW], vw[VW], nkw[2][KW], nvw[VW], bm = 0, nbm = 0;

  auto load_codes = [&](int blk, uint32_t (&k_)[2][KW], uint32_t (&v_)[VW], uint32_t& bm_) {
    const uint32_t* kc = kc_base + (size_t)blk * G.bwords;
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
      for (int half = 0; half < 2; ++half) {  // token T0 (half 0) / T1 (half 1)
        const int T = 16 * mt + gq + 8 * half;
        if (BITS == 2) {
          uint2 w = *reinterpret_cast<const uint2*>(kc + T * 8 + 2 * tq);
          k_[mt][2 * half] = w.x;
          k_[mt][2 * half + 1] = w.y;
        } else {
          k_[mt][half] = kc[T * 4 + tq];
        }
      }
    }
    const uint32_t* vc = vc_base + (size_t)blk * G.bwords + lane * VW;
#pragma unroll
    for (int i = 0; i < VW; i += 4) {
      uint4 w = *reinterpret_cast<const uint4*>(vc + i);
      v_[i] = w.x;
      v_[i + 1] = w.y;
      v_[i + 2] = w.z;
      v_[i + 3] = w.w;
    }
    bm_ = bm_base[blk];
  };
  auto load_params = [&](int blk, int buf) {
    const int q = lane;  // 16-byte chunk
    cp_async16(&ws.kpar[buf][4 * (q ^ ((q >> 3) << 1))], kp_base + (size_t)blk * 128 + 4 * q);
    cp_async16(&ws.vpar[buf][4 * q], vp_base + (size_t)blk * 128 + 4 * q);
    cp_async_commit();
  };

  int blk = blk0 + warp;
  int buf = 0;
  if (blk < blk1) {
    load_codes(blk, kw, vw, bm);
    load_params(blk, 0);
  }
  for (; blk < blk1; blk += kWarps, buf ^= 1) {
    const int nxt = blk + kWarps;
    if (nxt < blk1) {
      load_codes(nxt, nkw, nvw, nbm);
      load_params(nxt, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncwarp();

    // ---- key B fragments (cooperative) + zero-point constants C_j ---------------
    float Cp[NR];
    {
      float s4[4], z4[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const uint32_t w = ws.kpar[buf][kpar_swz(32 * ktk + kks + 8 * m)];
        const float lo = __uint_as_float(w << 16), hi = __uint_as_float(w & 0xFFFF0000u);
        s4[m] = (hi - lo) * cs * kk_scale;
        z4[m] = BITS == 1 ? fmaf(0.75f, lo, 0.25f * hi) : lo;
      }
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        float w0 = Qr[j][0] * s4[0], w1 = Qr[j][1] * s4[1], w2 = Qr[j][2] * s4[2], w3 = Qr[j][3] * s4[3];
        Cp[j] = fmaf(Qr[j][0], z4[0], fmaf(Qr[j][1], z4[1], fmaf(Qr[j][2], z4[2], Qr[j][3] * z4[3])));
        uint4 frag;
        if (BITS == 2) {  // b0 = (m0, m1), b1 = (m2, m3)
          split2(w0, w1, frag.x, frag.z);
          split2(w2, w3, frag.y, frag.w);
        } else {          // b0 = (m0, m2), b1 = (m1, m3)
          split2(w0, w2, frag.x, frag.z);
          split2(w1, w3, frag.y, frag.w);
        }
        ws.bk[kks][(4 * j + ktk) ^ kks] = frag;
      }
#pragma unroll
      for (int j = 0; j < NR; ++j) Cp[j] = warp_sum_all(Cp[j]);
    }
    __syncwarp();

    // ---- scores: D[token][row] over 8 k-steps, 2 m-tiles --------------------------
    float dk[2][4];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) dk[mt][0] = dk[mt][1] = dk[mt][2] = dk[mt][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const uint4 bb = ws.bk[ks][lane ^ ks];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        uint32_t a0, a1, a2, a3;
        if (BITS == 2) {
          const uint32_t msk = (3u << (2 * (ks & 3))) | (3u << (16 + 2 * (ks & 3)));
          const int sh = ks < 4 ? 0 : 8;
          a0 = (kw[mt][0] >> sh) & msk;  // T0, channels (32tq+ks, +8)
          a2 = (kw[mt][1] >> sh) & msk;  // T0, channels (32tq+16+ks, +24)
          a1 = (kw[mt][2] >> sh) & msk;  // T1
          a3 = (kw[mt][3] >> sh) & msk;
        } else {
          const uint32_t msk = (1u << ks) | (1u << (16 + ks));
          a0 = kw[mt][0] & msk;          // T0, channels (32tq+ks, +16)
          a2 = (kw[mt][0] >> 8) & msk;   // T0, channels (32tq+8+ks, +24)
          a1 = kw[mt][1] & msk;
          a3 = (kw[mt][1] >> 8) & msk;
        }
        mma16816(dk[mt], a0, a1, a2, a3, bb.x, bb.y);
        mma16816(dk[mt], a0, a1, a2, a3, bb.z, bb.w);
      }
    }

    // ---- epilogue: log2 scores, mask, spill, online softmax ----------------------
    // lane holds rows jr0 = 2tq, jr1 = 2tq+1 for tokens T = 16mt + gq (+8)
    const int jr0 = 2 * tq, jr1 = 2 * tq + 1;
    float c0 = 0.f, c1 = 0.f;
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      if (j == jr0) c0 = Cp[j];
      if (j == jr1) c1 = Cp[j];
    }
    float sc[2][4];
    const int pos0 = blk * 32;
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        const int T = 16 * mt + gq + 8 * hf;
        const bool msk = (bm >> T) & 1u;
        sc[mt][2 * hf] = msk ? -CUDART_INF_F : fmaf(dk[mt][2 * hf], k_out, c0);
        sc[mt][2 * hf + 1] = msk ? -CUDART_INF_F : fmaf(dk[mt][2 * hf + 1], k_out, c1);
        if (!msk) {
          if (jr0 < NR && jr0 >= agg_j0 && jr0 < agg_j0 + G.G)
            a.spill[((size_t)b * G.Hq + h * G.G + (jr0 - agg_j0)) * G.L + pos0 + T] = sc[mt][2 * hf];
          if (jr1 < NR && jr1 >= agg_j0 && jr1 < agg_j0 + G.G)
            a.spill[((size_t)b * G.Hq + h * G.G + (jr1 - agg_j0)) * G.L + pos0 + T] = sc[mt][2 * hf + 1];
        }
      }
    }
    float mx0 = fmaxf(fmaxf(sc[0][0], sc[0][2]), fmaxf(sc[1][0], sc[1][2]));
    float mx1 = fmaxf(fmaxf(sc[0][1], sc[0][3]), fmaxf(sc[1][1], sc[1][3]));
    mx0 = warp_max_g(mx0);
    mx1 = warp_max_g(mx1);
    const float mn0 = fmaxf(m_run[0], mx0), mn1 = fmaxf(m_run[1], mx1);
    const bool grow = (mn0 > m_run[0]) || (mn1 > m_run[1]);
    if (__any_sync(0xffffffffu, grow)) {
      const float al0 = m_run[0] == -CUDART_INF_F ? 0.f : exp2f(m_run[0] - mn0);
      const float al1 = m_run[1] == -CUDART_INF_F ? 0.f : exp2f(m_run[1] - mn1);
      l_run[0] *= al0;
      l_run[1] *= al1;
      // alpha for the value accumulator columns of this lane and its z role
      float ac0, ac1, az[PG ? 1 : 4];
      if (PG) {
        // columns n = 2tq, 2tq+1 -> row n % NR; rows 0..NR-1 live in lanes with tq = 0
        const float r0 = __shfl_sync(0xffffffffu, al0, 0), r1 = __shfl_sync(0xffffffffu, al1, 0);
        ac0 = NR == 1 ? r0 : r0;  // n = 2tq  -> row (2tq) % NR = 0 for NR in {1, 2}
        ac1 = NR == 1 ? r0 : r1;  // n = 2tq+1 -> row 0 (NR=1) or 1 (NR=2)
        az[0] = (NR == 1 || (gq & 1) == 0) ? r0 : r1;
      } else {
        ac0 = al0;
        ac1 = al1;
        // z role row j = gq lives in lane (tq = gq >> 1) component gq & 1
        const float x0 = __shfl_sync(0xffffffffu, al0, gq >> 1), x1 = __shfl_sync(0xffffffffu, al1, gq >> 1);
        const float ar = (gq & 1) ? x1 : x0;
#pragma unroll
        for (int i = 0; i < 4; ++i) az[i] = ar;
      }
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        dv[mt][0] *= ac0;
        dv[mt][1] *= ac1;
        dv[mt][2] *= ac0;
        dv[mt][3] *= ac1;
      }
#pragma unroll
      for (int i = 0; i < (PG ? 1 : 4); ++i) zacc[i] *= az[i];
      m_run[0] = mn0;
      m_run[1] = mn1;
    }
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        const int T = 16 * mt + gq + 8 * hf;
        const float p0 = exp2f(sc[mt][2 * hf] - m_run[0]);
        const float p1 = exp2f(sc[mt][2 * hf + 1] - m_run[1]);
        l_run[0] += p0;
        l_run[1] += p1;
        if (jr0 < NR) ws.P[jr0][T] = p0;
        if (jr1 < NR) ws.P[jr1][T] = p1;
      }
    }
    __syncwarp();

    // ---- value B fragments -------------------------------------------------------
    // lane role: PG: column n = gq -> (grp = gq / NR, row = gq % NR); else row = gq
    uint32_t vb[PG ? 1 : 4][2][4];  // [grp][ks] {b0hi, b1hi, b0lo, b1lo}
#pragma unroll
    for (int gi = 0; gi < (PG ? 1 : 4); ++gi) {
      const int grp = PG ? (gq / NR) : gi;
      const int row = PG ? (gq % NR) : gq;
      const bool live = PG ? (gq < 4 * NR) : (gq < NR);
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        float x[4];
#pragma unroll
        for (int slot = 0; slot < 4; ++slot) {
          const int khalf = slot >> 1;
          const int t = 16 * ks + 2 * tq + (slot & 1) + 8 * khalf;
          const int q = 2 * ks + khalf;
          const int sq = BITS == 2 ? 2 * q : q;
          float val = 0.f;
          if (live) {
            const uint32_t w = ws.vpar[buf][t * 4 + grp];
            const float lo = __uint_as_float(w << 16), hi = __uint_as_float(w & 0xFFFF0000u);
            const float p = ws.P[row < NR ? row : 0][t];
            const float z = BITS == 1 ? fmaf(0.75f, lo, 0.25f * hi) : lo;
            zacc[gi] = fmaf(p, z, zacc[gi]);
            val = p * ((hi - lo) * cs) * pow2i(-sq - Ev);
          }
          x[slot] = val;
        }
        split2(x[0], x[1], vb[gi][ks][0], vb[gi][ks][2]);
        split2(x[2], x[3], vb[gi][ks][1], vb[gi][ks][3]);
      }
    }

    // ---- P.V over 8 channel m-tiles x 2 token k-steps -----------------------------
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        uint32_t a0, a1, a2, a3;
        const int q0 = 2 * ks, q1 = 2 * ks + 1;
        if (BITS == 2) {
          const uint32_t W = vw[mt], W8 = W >> 8;
          const uint32_t m0 = (3u << (2 * q0)) | (3u << (16 + 2 * q0));
          const uint32_t m1 = (3u << (2 * q1)) | (3u << (16 + 2 * q1));
          a0 = W & m0;
          a1 = W8 & m0;
          a2 = W & m1;
          a3 = W8 & m1;
        } else {
          const uint32_t W = vw[mt >> 1] >> (8 * (mt & 1)), W4 = W >> 4;
          const uint32_t m0 = (1u << q0) | (1u << (16 + q0));
          const uint32_t m1 = (1u << q1) | (1u << (16 + q1));
          a0 = W & m0;
          a1 = W4 & m0;
          a2 = W & m1;
          a3 = W4 & m1;
        }
        const int gi = PG ? 0 : (mt >> 1);
        mma16816(dv[mt], a0, a1, a2, a3, vb[gi][ks][0], vb[gi][ks][1]);
        mma16816(dv[mt], a0, a1, a2, a3, vb[gi][ks][2], vb[gi][ks][3]);
      }
    }

    // rotate prefetched registers
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int i = 0; i < KW; ++i) kw[mt][i] = nkw[mt][i];
#pragma unroll
    for (int i = 0; i < VW; ++i) vw[i] = nvw[i];
    bm = nbm;
    __syncwarp();
  }

  // ---- warp results -> shared, CTA merge -> partial ----------------------------------
  l_run[0] = warp_sum_g(l_run[0]);
  l_run[1] = warp_sum_g(l_run[1]);
#pragma unroll
  for (int i = 0; i < (PG ? 1 : 4); ++i) {  // z sums over the 4 lanes of a row group
    zacc[i] += __shfl_xor_sync(0xffffffffu, zacc[i], 1);
    zacc[i] += __shfl_xor_sync(0xffffffffu, zacc[i], 2);
  }
  __syncthreads();
  MergeSmem<NR>& ms = *reinterpret_cast<MergeSmem<NR>*>(smem_raw);
  if (gq == 0) {
    if (2 * tq < NR) {
      ms.m[warp][2 * tq] = m_run[0];
      ms.l[warp][2 * tq] = l_run[0];
    }
    if (2 * tq + 1 < NR) {
      ms.m[warp][2 * tq + 1] = m_run[1];
      ms.l[warp][2 * tq + 1] = l_run[1];
    }
  }
  if (PG) {
    // lane columns n = 2tq + e; its D rows are channels 16mt + gq (+8); useful iff
    // group(n) = n / NR == mt >> 1.  The z sum of column n lives in lanes gq == n.
    const float zc0 = __shfl_sync(0xffffffffu, zacc[0], 4 * (2 * tq));
    const float zc1 = __shfl_sync(0xffffffffu, zacc[0], 4 * ((2 * tq + 1) & 7));
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int n = 2 * tq + e;
        if (n < 4 * NR && n / NR == (mt >> 1)) {
          const int j = n % NR;
          const float zc = e ? zc1 : zc0;
          ms.o[warp][j][16 * mt + gq] = fmaf(dv[mt][e], v_out, zc);
          ms.o[warp][j][16 * mt + gq + 8] = fmaf(dv[mt][2 + e], v_out, zc);
        }
      }
    }
  } else {
    // columns = rows 2tq, 2tq+1; z sum of (grp, row j) lives in lanes gq == j
#pragma unroll
    for (int gi = 0; gi < 4; ++gi) {
      const float z0 = __shfl_sync(0xffffffffu, zacc[gi], 4 * (2 * tq));
      const float z1 = __shfl_sync(0xffffffffu, zacc[gi], 4 * ((2 * tq + 1) & 7));
#pragma unroll
      for (int mt = 2 * gi; mt < 2 * gi + 2; ++mt) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int j = 2 * tq + e;
          if (j < NR) {
            const float zc = e ? z1 : z0;
            ms.o[warp][j][16 * mt + gq] = fmaf(dv[mt][e], v_out, zc);
            ms.o[warp][j][16 * mt + gq + 8] = fmaf(dv[mt][2 + e], v_out, zc);
          }
        }
      }
    }
  }
  __syncthreads();
  const int R = NR;
  const size_t base = (((size_t)b * G.H + h) * (a.nsplit + 1) + split) * R;
  for (int i = threadIdx.x; i < NR * 128; i += kThreads) {
    const int j = i >> 7, c = i & 127;
    float M = -CUDART_INF_F;
#pragma unroll
    for (int w = 0; w < kWarps; ++w)
      if (ms.l[w][j] > 0.f) M = fmaxf(M, ms.m[w][j]);
    float o = 0.f, L = 0.f;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      if (ms.l[w][j] > 0.f) {
        const float f = exp2f(ms.m[w][j] - M);
        o = fmaf(ms.o[w][j][c], f, o);
        L = fmaf(ms.l[w][j], f, L);
      }
    }
    a.part_o[(base + j) * 128 + c] = o;
    if (c == 0) {
      a.part_ml[(base + j) * 2 + 0] = M;
      a.part_ml[(base + j) * 2 + 1] = L;
    }
  }
}

template <int BITS, int NR>
void launch_fast_t(const AttnArgs& a, cudaStream_t st) {
  constexpr size_t smem = fast_smem_bytes<NR>();
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_attend_fast<BITS, NR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)std::max(smem, generic_smem_bytes(a.G, a.rows)));
    configured = true;
  }
  dim3 grid(a.nsplit + 1, a.G.H, a.G.batch);
  k_attend_fast<BITS, NR><<<grid, kThreads, std::max(smem, generic_smem_bytes(a.G, a.rows)), st>>>(a);
}

}  // namespace

int attend_fast_supported(const Geo& G, int rows) {
  const int R = rows * G.G;
  return G.fast && (R == 1 || R == 2 || R == 4 || R == 8) && G.L % 32 == 0;
}

// splits per (seq, head): enough CTAs for several full waves at 2 CTAs/SM
int launch_attend_fast(const AttnArgs& a0, cudaStream_t st) {
  AttnArgs a = a0;
  const Geo& G = a.G;
  const int nblk = a.f / 32;
  const int units = G.H * G.batch;
  int want = (6 * 2 * 148 + units - 1) / units;  // ~6 waves
  want = std::max(1, std::min(want, std::min(127, std::max(1, nblk / 8))));
  a.blocks_per_split = std::max(1, (nblk + want - 1) / want);
  a.nsplit = std::max(1, (nblk + a.blocks_per_split - 1) / a.blocks_per_split);
  const int R = a.rows * G.G;
  if (G.bits == 2) {
    if (R == 1) launch_fast_t<2, 1>(a, st);
    else if (R == 2) launch_fast_t<2, 2>(a, st);
    else if (R == 4) launch_fast_t<2, 4>(a, st);
    else launch_fast_t<2, 8>(a, st);
  } else {
    if (R == 1) launch_fast_t<1, 1>(a, st);
    else if (R == 2) launch_fast_t<1, 2>(a, st);
    else if (R == 4) launch_fast_t<1, 4>(a, st);
    else launch_fast_t<1, 8>(a, st);
  }
  launch_combine(a, st);
  return 2;
}

}  // namespace spc
