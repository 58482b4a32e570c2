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
// 8 query rows (GQA-4 x {output, speculative}; TSC): the score MMA is transposed, M = rows
// (hi plane on M rows 0-7, lo plane on 8-15), N = 8 tokens per n-tile, K = channels, with A =
// the per-block Q*s hi/lo built in registers and B = the expanded codes.  A lane then holds row
// gq's scores of tokens 8nt + 2tq + {0,1}, which are the P.V B-fragment positions: P stays in
// registers, and the hi + lo planes of a row sit in one lane.
//
// Work split: grid (nsplit + 1, H, batch), 8 warps per CTA.  A CTA streams a
// contiguous range of 32-token blocks of one (seq, kv head); each warp owns
// every 8th block and keeps its own online-softmax state; the CTA merges its
// warps and writes one (m, l, O) partial.  Per block a warp needs 3072 B
// (2-bit) / 2048 B (1-bit) -- key codes, value codes, key and value group
// params, four contiguous segments -- which one elected lane fetches with
// cp.async.bulk (TMA) into a 3-stage per-warp shared-memory ring tracked by
// mbarriers, so two blocks are always in flight while the third is computed.
// The last split is the exact segment (pinned slots, residual window, in-step
// rows; full-precision bf16 rows, fp32 CUDA-core dot products).
#include <algorithm>
#include <cstdlib>

#include "exact_segment.cuh"

namespace spc {
namespace {

#ifndef SPC_K2_WARPS
#define SPC_K2_WARPS 8
#endif
constexpr int kWarps = SPC_K2_WARPS;
constexpr int kThreads = kWarps * 32;
#ifndef SPC_K2_STAGES
#define SPC_K2_STAGES 3
#endif
#ifndef SPC_K2_MINB
#define SPC_K2_MINB 2
#endif
constexpr int kStages = SPC_K2_STAGES;  // TMA ring depth per warp
// 2-bit x 8 rows (GQA-4 dual-token at 2 bits) would need 130 KB per CTA with the
// 3-stage ring -- one CTA per SM; two stages bring it to 105 KB and two CTAs
template <int BITS, int NR>
constexpr int stages_of() { return (BITS == 2 && NR == 8) ? 2 : kStages; }
constexpr int kMinBlocks = SPC_K2_MINB; // resident CTAs per SM
#ifndef SPC_K2_LAZY
#define SPC_K2_LAZY 1
#endif
// Lazy online-softmax rescale (SPC_K2_LAZY): the running max m_run is only
// raised (warp reduction + accumulator rescale) when some score exceeds it by
// more than kSlack (log2 units); otherwise P = exp2(s - m_run) <= 2^kSlack is
// used as is.  (O, l) are scaled consistently, so the result is the same
// softmax; the per-block max reduction (3 dependent SHFL+FMNMX levels per
// row) disappears from the common path.
constexpr int kSlackLog2 = SPC_K2_LAZY ? 8 : 0;  // P <= 2^kSlackLog2
constexpr float kSlack = (float)kSlackLog2;
#ifndef SPC_K2_HKB
#define SPC_K2_HKB 1
#endif
// f16x2 key-B build for the shared-memory query rows (NR >= 4, SPC_K2_HKB): the
// query is split once per CTA into f16 hi + lo pairs (Qh) and the block's key
// scales once per block into f16 hi + lo pairs (shared by all rows); per row
// and channel pair B = Qh * sh is then formed with four f16x2 ops
//   hi = rn(Qhi*shi),  lo = rn(Qlo*shi + rn(Qhi*slo + (Qhi*shi - hi)))
// where Qhi*shi - hi is the exact rounding error (FMA), so hi + lo carries the
// same ~22 bits as the fp32 product split into hi + lo (split2), at 4 instead
// of 8 instructions per pair.  Q is pre-scaled by 2^-aq (max |Q| in [2^6, 2^7])
// and the scales by 2^aq, so both factors stay in the f16 normal range and
// max |B| <= 2^14 as before.
constexpr bool kHalfKeyB = SPC_K2_HKB != 0;
#ifndef SPC_K2_VCOOP
#define SPC_K2_VCOOP 1
#endif
// Cooperative value-parameter decode for the wide GQA rows (NR >= 4, SPC_K2_VCOOP):
// once per block the 32 lanes decode the 128 (token, group) value params into
// f16 hi + lo pairs of s' = s * 2^-(q+Ev) and z' = z * 2^-Ez in shared memory
// (each lane one (group, k-step, tq): four tokens).  The value B fragment of
// row j is then mul_hilo(P hi/lo, s' hi/lo) -- four f16x2 ops per token pair --
// instead of decoding every (token, group) param in all eight row lanes, and
// sum_t P * z runs on the tensor cores: one m16n8k16 with A rows 0-3 = z' hi of
// the four groups, rows 4-7 = z' lo, and B = the P hi / lo fragments.
constexpr bool kVCoop = SPC_K2_VCOOP != 0;
#ifndef SPC_K2_FOLD
#define SPC_K2_FOLD 16
#endif
#ifndef SPC_K2_FOLD_PG
#define SPC_K2_FOLD_PG 16
#endif
#ifndef SPC_K2_FOLD_MIN
#define SPC_K2_FOLD_MIN 32
#endif
// Accumulator fold (SPC_K2_FOLD = F; 0 = off): every F blocks a warp adds its
// z sums (sum_t P z) into the value accumulator and restarts them.  mma.sync's
// fp32 accumulation truncates each k-step's sum to the accumulator's exponent,
// a bias toward zero of ~2^-24 |D| per MMA.  With unsigned codes the scale part
// sum_t P s code and the zero-point part sum_t P z each grow linearly over a
// warp's blocks while their sum (the output) is a random walk that largely
// cancels them, so the bias is amplified: measured at the C4 rank share (1 KV
// head, 128k, 8 splits = 64 blocks per warp) the fp32 output's per-head error
// was 2.6e-3 and fell as 1/(blocks per warp) with more splits
// (profiles/r2_35_fold.json).  Folding keeps both accumulators at the output's
// scale: 2.6e-3 -> 1.9e-4 there (F = 16), for ~50 instructions per F blocks per
// warp.  Only launches whose warps walk more than SPC_K2_FOLD_MIN blocks use
// the folding instantiation (C4 share: 64; C3: 23 at 5.5e-4 unfolded; C2: 18).
constexpr int kFold = SPC_K2_FOLD;
constexpr int kFoldPG = SPC_K2_FOLD_PG;  // the MHA (PG) rows' fold period
constexpr int kFoldMinBlocks = SPC_K2_FOLD_MIN;
#ifndef SPC_K2_CMMA
#define SPC_K2_CMMA 0
#endif
// Zero-point constants on the tensor cores (NR >= 4 rows, SPC_K2_CMMA):
// C_j = sum_c Q[j,c] z_c is one m16n8k16 per 16 channels with A = the CTA's
// f16 hi + lo query table (rows 0-7 hi, 8-15 lo) and B = the block's key
// zero-points z * 2^-Ezk as f16 hi + lo (columns 0, 1), instead of 32 FFMA and a
// 9-shuffle reduce-scatter per lane and block.  Off by default: the A/B on one
// box measured C3 K2 +1.7% against the FFMA form (the fragment loads and their
// address arithmetic cost more issue slots than the FFMA chain they replace).
constexpr bool kCMma = SPC_K2_CMMA != 0;
#ifndef SPC_K2_NOSPILL
#define SPC_K2_NOSPILL 0
#endif
// Measurement only (SPC_K2_NOSPILL=1 builds an A/B library whose aggregate is
// invalid): K2 without the speculative-row logit spill, to price the spill.
constexpr bool kNoSpill = SPC_K2_NOSPILL != 0;
#ifndef SPC_K2_EXACT_ORDER
#define SPC_K2_EXACT_ORDER 0
#endif
// CTA order of a launch: 0 = (split, head, seq) grid, each unit's exact CTA after
// its splits; 1 = 1-D grid with every unit's splits first and all exact CTAs at
// the end (the short exact CTAs backfill the last wave); 2 = exact CTAs first
constexpr int kExactOrder = SPC_K2_EXACT_ORDER;

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

__device__ __forceinline__ uint32_t h2u(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
__device__ __forceinline__ __half2 u2h(uint32_t u) { return *reinterpret_cast<__half2*>(&u); }
// (hi, lo) f16x2 of the product of two hi + lo f16x2 pairs (see kHalfKeyB)
__device__ __forceinline__ void mul_hilo(uint32_t ah, uint32_t al, uint32_t bh, uint32_t bl, uint32_t& hi,
                                         uint32_t& lo) {
  // hi = rn(ah*bh); lo = rn(al*bh + rn(ah*bl + (ah*bh - hi))) -- the first FMA is exact
  asm("{\n\t.reg .b32 nh, e;\n\t"
      "mul.rn.f16x2 %0, %2, %4;\n\t"
      "neg.f16x2 nh, %0;\n\t"
      "fma.rn.f16x2 e, %2, %4, nh;\n\t"
      "fma.rn.f16x2 e, %2, %5, e;\n\t"
      "fma.rn.f16x2 %1, %3, %4, e;\n\t}"
      : "=r"(hi), "=r"(lo)
      : "r"(ah), "r"(al), "r"(bh), "r"(bl));
}

__device__ __forceinline__ float fast_exp2(float x) {  // ex2.approx (|rel err| ~2^-22); -inf -> 0
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float pow2i(int e) {  // 2^e, e in [-126, 127]
  return __int_as_float((127 + e) << 23);
}

__device__ __forceinline__ int ceil_log2(float x) {  // x > 0
  int e = ilogbf(x);
  return (x > ldexpf(1.f, e)) ? e + 1 : e;
}

// ---- TMA bulk copies + mbarriers (per-warp ring) --------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
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
__device__ __forceinline__ void tma_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// shared-window addresses precomputed by the caller (the per-block issue path)
__device__ __forceinline__ void mbar_expect_tx_u32(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_u32(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

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

template <int BITS>
struct StageLayout {
  static constexpr int kc = 0;                 // key codes: 32 rows x 4*BITS words
  static constexpr int vc = 32 * 4 * BITS;     // value codes (fragment-native)
  static constexpr int kp = 2 * 32 * 4 * BITS; // key (lo|hi) per channel
  static constexpr int vp = kp + 128;          // value (lo|hi) per (token, group)
  static constexpr int words = vp + 128;
  static constexpr unsigned code_bytes = 32 * 4 * BITS * 4;
  static constexpr unsigned bytes = words * 4;
};

template <int BITS, int NR>
struct __align__(16) WarpSmem {
  // key B fragments {b0hi, b1hi, b0lo, b1lo} of lane (row j, t'), [ks][4j + (t' ^ ((ks>>1)&3))];
  // row stride = 4 mod 8 uint4 so a 128-bit store phase (ks = 0..7) hits 8 distinct bank slots
  static constexpr int kBkRow = 4 * NR + ((NR & 1) ? 0 : 4);
  uint4 bk[8][kBkRow];
  static constexpr int kS = stages_of<BITS, NR>();
  uint32_t stage[kS][StageLayout<BITS>::words];            // TMA ring
  // block probabilities: PG (<= 2 rows) [row][40]; otherwise [row & 1][token][row >> 1]
  // in 132-float planes, conflict-free for both the score-side stores (t = c+gq,
  // row = 2tq+e) and the value-side loads (row = gq, t = c+2tq)
  // PG rows use stride 40 (even: token pairs load as float2; banks 8*row + t)
  // VCOOP rows (NR >= 4): [row][36]: score-side stores conflict-free (banks 8tq + 4e + gq + ...),
  // value-side token pairs load as float2
  static constexpr bool kPRow = kVCoop && NR * 4 > 8;
  static constexpr int kPWords = NR * 4 <= 8 ? NR * 40 : kPRow ? NR * 36 : 2 * 132;
  float P[kPWords];
  __device__ static constexpr int pidx(int row, int t) {
    return NR * 4 <= 8 ? row * 40 + t : kPRow ? row * 36 + t : (row & 1) * 132 + t * 4 + (row >> 1);
  }
  float4 sz[64];                                          // value (s*2^-q, z) pairs, vparams order (szidx)
  uint64_t bar[kS];
  float zfold;  // the accumulator fold's z scale (kFold), read once per fold
  // float4 slot f of sz, low two bits XORed with the 8-slot row index (mod 4): the
  // decode stores (lane l -> 2l + h) and the PG loads (16 grp + 4 tq + 2 ks + h;
  // grp = gq >> 1 for 2 rows, gq & 3 for 1 row) hit 8 distinct 16-byte bank
  // groups per 8-lane phase (unswizzled: 2-way / 4-way conflicts)
  __device__ static constexpr int szidx(int f) { return f ^ ((f >> 3) & 3); }
};

template <int NR>
struct MergeSmem {
  float o[kWarps][NR][128];
  float m[kWarps][NR];
  float l[kWarps][NR];
  float f[kWarps][NR];  // exp2(m_w - M) per warp and row (0 for empty warps)
  float M[NR], L[NR];
};

// exact segment scratch (split == nsplit CTAs): a chunk of CH full-precision
// K and V rows is staged into shared memory with cp.async before any math
template <int NR>
struct ExactSmem {
  // rows per chunk (staged form: NR <= 4).  SPC_EXACT_CH2=192 stages a whole MHA
  // segment (64 pins + up to 95 residual + 2 in-step rows) in one chunk: faster
  // in the one-layer harness (C2 K2 -0.4%), slower in the 32-layer bench (-0.7%,
  // PCIe gather 47 -> 43 GB/s with the larger shared-memory footprint), so 128
#ifndef SPC_EXACT_CH2
#define SPC_EXACT_CH2 128
#endif
  static constexpr int CH = NR <= 2 ? SPC_EXACT_CH2 : 128;
  uint4 krow[CH][16];  // bf16 x 128 per row; reused for the warps' partial outputs at the end
  uint4 vrow[CH][16];
  float sc[NR][CH];
  float fac[NR], m[NR], l[NR], pm[NR], pl[NR];
  int slots[1024];     // occupied pin slots, slot order
  int spos[1024];      // their positions
  int npin;
  using Out = float[kWarps][NR][128];
  __device__ Out& o() { return *reinterpret_cast<Out*>(&krow[0][0]); }
};

// exact segment scratch, direct-load form
template <int NR>
struct ExactRowsSmem {
  static constexpr int CH = 512;
  float sc[NR][CH];
  float fac[NR], m[NR], l[NR], pm[NR], pl[NR];
  int slots[1024];
  int npin;
  float o[kWarps][NR][128];
};

template <int BITS, int NR>
constexpr size_t fast_smem_bytes() {
  size_t a = sizeof(WarpSmem<BITS, NR>) * kWarps + (NR > 2 ? NR * 16 * (36 + (kHalfKeyB ? 36 : 0)) + 16 : 0),
         b = sizeof(MergeSmem<NR>),
         c = NR == 8 ? sizeof(ExactRowsSmem<NR>) : sizeof(ExactSmem<NR>);
  return a > b ? (a > c ? a : c) : (b > c ? b : c);
}

// ---- exact segment: pinned slots + residual ring + in-step rows (bf16, exact) ----------
// One CTA per (seq, kv head), 8 warps, latency-oriented.  Rows come in chunks
// of CH: every K and V row of the chunk is staged into shared memory with
// 16-byte cp.async copies issued up front (one memory round trip per chunk),
// then a warp scores kRows rows per batch and finishes the NR x kRows per-lane
// partial dot products with one warp reduce-scatter (V-1 shuffles).  Online
// softmax across chunks; the pinned rows' own (max, sum) -- the pinned mass,
// engine.py:314-316 -- is tracked alongside.
template <int NR>
__device__ void exact_segment_fast(const AttnArgs& a, const int split, const int h, const int b,
                                   unsigned char* smem) {
  const Geo& G = a.G;
  const LayerBufs& B = a.B;
  ExactSmem<NR>& ex = *reinterpret_cast<ExactSmem<NR>*>(smem);
  static_assert(sizeof(typename ExactSmem<NR>::Out) <= sizeof(ex.krow), "partial outputs alias the staged key rows");
  constexpr int CH = ExactSmem<NR>::CH;
  constexpr int kRows = NR <= 2 ? 4 : 16 / NR;  // rows per warp batch
  constexpr int V = NR * kRows;                  // partial sums per lane per batch: 4, 8 or 16
  constexpr int LV = V == 4 ? 2 : V == 8 ? 3 : 4;
  static_assert(V == (1 << LV), "reduce-scatter needs a power-of-two value count");
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int unit = G.scope ? h : 0, hh = G.scope ? 0 : h;
  float Qr[NR][4];
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    const int r = j / G.G, g2 = j - r * G.G;
    const uint2 w = *reinterpret_cast<const uint2*>(a.q + (((size_t)b * a.rows + r) * G.Hq + h * G.G + g2) * 128 + 4 * lane);
    const __nv_bfloat162 q01 = *reinterpret_cast<const __nv_bfloat162*>(&w.x);
    const __nv_bfloat162 q23 = *reinterpret_cast<const __nv_bfloat162*>(&w.y);
    Qr[j][0] = __low2float(q01) * a.sm_scale_log2;
    Qr[j][1] = __high2float(q01) * a.sm_scale_log2;
    Qr[j][2] = __low2float(q23) * a.sm_scale_log2;
    Qr[j][3] = __high2float(q23) * a.sm_scale_log2;
  }
  const int32_t* pp = B.pin_pos + ((size_t)b * G.U + unit) * G.k;
  if (warp == 0) {  // ballot compaction of the occupied slots (and their positions), in slot order
    int cnt = 0;
    for (int s0 = 0; s0 < G.k; s0 += 32) {
      const int pos = s0 + lane < G.k ? pp[s0 + lane] : -1;
      const bool occ = pos >= 0;
      const unsigned m = __ballot_sync(0xffffffffu, occ);
      if (occ) {
        const int w = cnt + __popc(m & ((1u << lane) - 1u));
        ex.slots[w] = s0 + lane;
        ex.spos[w] = pos;
      }
      cnt += __popc(m);
    }
    if (lane == 0) ex.npin = cnt;
  }
  if (tid < NR) {
    ex.m[tid] = -CUDART_INF_F;
    ex.l[tid] = 0.f;
    ex.pm[tid] = -CUDART_INF_F;
    ex.pl[tid] = 0.f;
  }
  __syncthreads();
  const int npin = ex.npin, nres = a.n - a.f, total = npin + nres + a.rows;
  const int agg_j0 = a.agg_row * G.G;
  float acc[NR][4];
#pragma unroll
  for (int j = 0; j < NR; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;

  for (int c0 = 0; c0 < total; c0 += CH) {
    const int count = min(total, c0 + CH) - c0;
    // ---- stage the chunk: warp-sized groups of 32 x 16 B = one K row (lanes 0-15) + its V row
    for (int i = tid; i < count * 32; i += kThreads) {
      const int r = i >> 5, piece = i & 31, it = c0 + r;
      const __nv_bfloat16* base;
      if (it < npin) {
        const size_t o = ((((size_t)b * G.U + unit) * G.k + ex.slots[it]) * G.Hu + hh) * 128;
        base = (piece < 16 ? B.pool_k : B.pool_v) + o;
      } else if (it < npin + nres) {
        const int p = a.f + (it - npin);
        const size_t o = (((size_t)b * G.H + h) * G.ring + p % G.ring) * 128;
        base = (piece < 16 ? B.ring_k : B.ring_v) + o;
      } else {
        const size_t o = (((size_t)b * a.rows + (it - npin - nres)) * G.H + h) * 128;
        base = (piece < 16 ? a.k_new : a.v_new) + o;
      }
      cp_async16(piece < 16 ? &ex.krow[r][piece] : &ex.vrow[r][piece - 16],
                 reinterpret_cast<const uint4*>(base) + (piece & 15));
    }
    cp_async_wait_all();
    __syncthreads();
    // ---- scores: kRows rows per warp batch, one reduce-scatter
    for (int it0 = warp; it0 < count; it0 += kWarps * kRows) {
      float v[V];
#pragma unroll
      for (int u = 0; u < kRows; ++u) {
        const int it = min(it0 + u * kWarps, count - 1);  // rows past the chunk are discarded below
        const uint2 kw = reinterpret_cast<const uint2*>(ex.krow[it])[lane];
        const __nv_bfloat162 k01 = *reinterpret_cast<const __nv_bfloat162*>(&kw.x);
        const __nv_bfloat162 k23 = *reinterpret_cast<const __nv_bfloat162*>(&kw.y);
        const float k0 = __low2float(k01), k1 = __high2float(k01), k2 = __low2float(k23), k3 = __high2float(k23);
#pragma unroll
        for (int j = 0; j < NR; ++j)
          v[u * NR + j] = fmaf(Qr[j][0], k0, fmaf(Qr[j][1], k1, fmaf(Qr[j][2], k2, Qr[j][3] * k3)));
      }
      // reduce-scatter: after LV halving steps lane holds value idx = lane >> (5 - LV)
#pragma unroll
      for (int st2 = 0; st2 < LV; ++st2) {
        const int o = 16 >> st2, half = V >> (st2 + 1);
        const bool up = lane & o;
#pragma unroll
        for (int i2 = 0; i2 < half; ++i2) {
          const float keep = up ? v[i2 + half] : v[i2], send = up ? v[i2] : v[i2 + half];
          v[i2] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
#pragma unroll
      for (int o = 16 >> LV; o; o >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
      const int idx = lane >> (5 - LV), u = idx / NR, j = idx - u * NR;
      const int it = it0 + u * kWarps;
      if ((lane & ((1 << (5 - LV)) - 1)) == 0 && it < count) {
        const int g = c0 + it;  // row index over the whole segment
        const float sv = v[0];
        const bool m = (g == npin + nres + 1) && j < G.G;  // row 0 never sees the speculative column
        ex.sc[j][it] = m ? -CUDART_INF_F : sv;
        if (g < npin && j >= agg_j0 && j < agg_j0 + G.G)
          a.spill[((size_t)b * G.Hq + h * G.G + (j - agg_j0)) * G.L + ex.spos[g]] = sv;
      }
    }
    __syncthreads();
    if (warp < NR) {  // online softmax of row `warp` over the chunk + pinned-only stats
      const int j = warp;
      const int npc = max(0, min(count, npin - c0));  // pinned rows in this chunk
      float mx = -CUDART_INF_F, mxp = -CUDART_INF_F;
      for (int i = lane; i < count; i += 32) {
        const float x = ex.sc[j][i];
        mx = fmaxf(mx, x);
        if (i < npc) mxp = fmaxf(mxp, x);
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        mxp = fmaxf(mxp, __shfl_xor_sync(0xffffffffu, mxp, o));
      }
      const float mold = ex.m[j], mnew = fmaxf(mold, mx);
      const float pmold = ex.pm[j], pmnew = fmaxf(pmold, mxp);
      float sum = 0.f, psum = 0.f;
      for (int i = lane; i < count; i += 32) {
        const float x = ex.sc[j][i];
        const float p = mnew == -CUDART_INF_F ? 0.f : fast_exp2(x - mnew);
        if (i < npc) psum += pmnew == -CUDART_INF_F ? 0.f : fast_exp2(x - pmnew);
        ex.sc[j][i] = p;
        sum += p;
      }
      sum = warp_sum_all(sum);
      psum = warp_sum_all(psum);
      __syncwarp();
      if (lane == 0) {
        const float f = mold == -CUDART_INF_F ? 0.f : exp2f(mold - mnew);
        ex.fac[j] = f;
        ex.m[j] = mnew;
        ex.l[j] = ex.l[j] * f + sum;
        const float pf = pmold == -CUDART_INF_F ? 0.f : exp2f(pmold - pmnew);
        ex.pm[j] = pmnew;
        ex.pl[j] = ex.pl[j] * pf + psum;
      }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      const float f = ex.fac[j];
      acc[j][0] *= f;
      acc[j][1] *= f;
      acc[j][2] *= f;
      acc[j][3] *= f;
    }
    // ---- P.V from the staged value rows
    for (int it = warp; it < count; it += kWarps) {
      const uint2 vw = reinterpret_cast<const uint2*>(ex.vrow[it])[lane];
      const __nv_bfloat162 v01 = *reinterpret_cast<const __nv_bfloat162*>(&vw.x);
      const __nv_bfloat162 v23 = *reinterpret_cast<const __nv_bfloat162*>(&vw.y);
      const float x0 = __low2float(v01), x1 = __high2float(v01), x2 = __low2float(v23), x3 = __high2float(v23);
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        const float p = ex.sc[j][it];
        acc[j][0] = fmaf(p, x0, acc[j][0]);
        acc[j][1] = fmaf(p, x1, acc[j][1]);
        acc[j][2] = fmaf(p, x2, acc[j][2]);
        acc[j][3] = fmaf(p, x3, acc[j][3]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < NR; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) ex.o()[warp][j][4 * lane + i] = acc[j][i];
  __syncthreads();
  const size_t base = (((size_t)b * G.H + h) * (a.nsplit + 1) + split) * NR;
  for (int i = tid; i < NR * 128; i += kThreads) {
    const int j = i >> 7, c = i & 127;
    float o = 0.f;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) o += ex.o()[w][j][c];
    a.part_o[(base + j) * 128 + c] = o;
  }
  if (tid < NR) {
    a.part_ml[(base + tid) * 2 + 0] = ex.m[tid];
    a.part_ml[(base + tid) * 2 + 1] = ex.l[tid];
    const size_t pb = ((size_t)b * G.H + h) * NR + tid;
    a.pin_ml[pb * 2 + 0] = ex.pm[tid];
    a.pin_ml[pb * 2 + 1] = ex.pl[tid];
  }
}

// ---- exact segment, direct-load form (used for NR = 8, where overlapping the row loads
// with the 8-row dot products beats staging) ----------------------------------------
// One CTA per (seq, kv head), 8 warps, latency-oriented: a warp scores kRows
// rows per batch with every row's 8-byte key load issued before any math, and
// the NR x kRows per-lane partial dot products are finished by one warp
// reduce-scatter (V-1 shuffles for V values instead of 5 per value).  Rows are
// processed in chunks of CH with an online softmax; the pinned rows' own
// (max, sum) -- the pinned mass, engine.py:314-316 -- is tracked alongside, so
// pinned and residual rows share one chunk.
template <int NR>
__device__ void exact_segment_rows(const AttnArgs& a, const int split, const int h, const int b,
                                   unsigned char* smem) {
  const Geo& G = a.G;
  const LayerBufs& B = a.B;
  ExactRowsSmem<NR>& ex = *reinterpret_cast<ExactRowsSmem<NR>*>(smem);
  constexpr int CH = ExactRowsSmem<NR>::CH;
  constexpr int kRows = NR <= 2 ? 4 : 16 / NR;  // rows per warp batch (measured best; NR=8 spill-free)
  constexpr int V = NR * kRows;                  // partial sums per lane per batch: 4, 8 or 16
  constexpr int LV = V == 4 ? 2 : V == 8 ? 3 : 4;
  static_assert(V == (1 << LV), "reduce-scatter needs a power-of-two value count");
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int unit = G.scope ? h : 0, hh = G.scope ? 0 : h;
  float Qr[NR][4];
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    const int r = j / G.G, g2 = j - r * G.G;
    const uint2 w = *reinterpret_cast<const uint2*>(a.q + (((size_t)b * a.rows + r) * G.Hq + h * G.G + g2) * 128 + 4 * lane);
    const __nv_bfloat162 q01 = *reinterpret_cast<const __nv_bfloat162*>(&w.x);
    const __nv_bfloat162 q23 = *reinterpret_cast<const __nv_bfloat162*>(&w.y);
    Qr[j][0] = __low2float(q01) * a.sm_scale_log2;
    Qr[j][1] = __high2float(q01) * a.sm_scale_log2;
    Qr[j][2] = __low2float(q23) * a.sm_scale_log2;
    Qr[j][3] = __high2float(q23) * a.sm_scale_log2;
  }
  const int32_t* pp = B.pin_pos + ((size_t)b * G.U + unit) * G.k;
  if (warp == 0) {  // ballot compaction of the occupied slots, in slot order
    int cnt = 0;
    for (int s0 = 0; s0 < G.k; s0 += 32) {
      const bool occ = s0 + lane < G.k && pp[s0 + lane] >= 0;
      const unsigned m = __ballot_sync(0xffffffffu, occ);
      if (occ) ex.slots[cnt + __popc(m & ((1u << lane) - 1u))] = s0 + lane;
      cnt += __popc(m);
    }
    if (lane == 0) ex.npin = cnt;
  }
  if (tid < NR) {
    ex.m[tid] = -CUDART_INF_F;
    ex.l[tid] = 0.f;
    ex.pm[tid] = -CUDART_INF_F;
    ex.pl[tid] = 0.f;
  }
  __syncthreads();
  const int npin = ex.npin, nres = a.n - a.f, total = npin + nres + a.rows;
  const int agg_j0 = a.agg_row * G.G;
  float acc[NR][4];
#pragma unroll
  for (int j = 0; j < NR; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;

  // row `it` (0 <= it < total): pinned slots, then residual positions, then the in-step rows
  auto row_ptr = [&](int it, const __nv_bfloat16*& kr, const __nv_bfloat16*& vr, int& pos, bool& spec) {
    spec = false;
    pos = -1;
    if (it < npin) {
      const int slot = ex.slots[it];
      pos = pp[slot];
      const size_t o = ((((size_t)b * G.U + unit) * G.k + slot) * G.Hu + hh) * 128;
      kr = B.pool_k + o;
      vr = B.pool_v + o;
    } else if (it < npin + nres) {
      const int p = a.f + (it - npin);
      const size_t o = (((size_t)b * G.H + h) * G.ring + p % G.ring) * 128;
      kr = B.ring_k + o;
      vr = B.ring_v + o;
    } else {
      const int r = it - npin - nres;
      spec = (r == 1);
      const size_t o = (((size_t)b * a.rows + r) * G.H + h) * 128;
      kr = a.k_new + o;
      vr = a.v_new + o;
    }
  };

  for (int c0 = 0; c0 < total; c0 += CH) {
    const int count = min(total, c0 + CH) - c0;
    // ---- scores: kRows rows per warp batch, loads first, one reduce-scatter
    for (int it0 = warp; it0 < count; it0 += kWarps * kRows) {
      uint2 kw[kRows];
      int posr[kRows];
      bool specr[kRows];
#pragma unroll
      for (int u = 0; u < kRows; ++u) {
        const int it = it0 + u * kWarps;
        kw[u] = make_uint2(0u, 0u);
        posr[u] = -1;
        specr[u] = false;
        if (it < count) {
          const __nv_bfloat16 *kr, *vr;
          row_ptr(c0 + it, kr, vr, posr[u], specr[u]);
          kw[u] = *reinterpret_cast<const uint2*>(kr + 4 * lane);
        }
      }
      float v[V];
#pragma unroll
      for (int u = 0; u < kRows; ++u) {
        const __nv_bfloat162 k01 = *reinterpret_cast<const __nv_bfloat162*>(&kw[u].x);
        const __nv_bfloat162 k23 = *reinterpret_cast<const __nv_bfloat162*>(&kw[u].y);
        const float k0 = __low2float(k01), k1 = __high2float(k01), k2 = __low2float(k23), k3 = __high2float(k23);
#pragma unroll
        for (int j = 0; j < NR; ++j)
          v[u * NR + j] = fmaf(Qr[j][0], k0, fmaf(Qr[j][1], k1, fmaf(Qr[j][2], k2, Qr[j][3] * k3)));
      }
      // reduce-scatter: after LV halving steps lane holds value idx = lane >> (5 - LV)
#pragma unroll
      for (int st2 = 0; st2 < LV; ++st2) {
        const int o = 16 >> st2, half = V >> (st2 + 1);
        const bool up = lane & o;
#pragma unroll
        for (int i2 = 0; i2 < half; ++i2) {
          const float keep = up ? v[i2 + half] : v[i2], send = up ? v[i2] : v[i2 + half];
          v[i2] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
#pragma unroll
      for (int o = 16 >> LV; o; o >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
      const int idx = lane >> (5 - LV), u = idx / NR, j = idx - u * NR;
      const int it = it0 + u * kWarps;
      // the lane's row data: select from the unrolled arrays without local memory
      int pos = -1;
      bool spec = false;
#pragma unroll
      for (int uu = 0; uu < kRows; ++uu)
        if (uu == u) {
          pos = posr[uu];
          spec = specr[uu];
        }
      if ((lane & ((1 << (5 - LV)) - 1)) == 0 && it < count) {
        const float sv = v[0];
        const bool m = spec && j < G.G;  // row 0 never sees the speculative column
        ex.sc[j][it] = m ? -CUDART_INF_F : sv;
        if (pos >= 0 && j >= agg_j0 && j < agg_j0 + G.G)
          a.spill[((size_t)b * G.Hq + h * G.G + (j - agg_j0)) * G.L + pos] = sv;
      }
    }
    __syncthreads();
    if (warp < NR) {  // online softmax of row `warp` over the chunk + pinned-only stats
      const int j = warp;
      const int npc = max(0, min(count, npin - c0));  // pinned rows in this chunk
      float mx = -CUDART_INF_F, mxp = -CUDART_INF_F;
      for (int i = lane; i < count; i += 32) {
        const float x = ex.sc[j][i];
        mx = fmaxf(mx, x);
        if (i < npc) mxp = fmaxf(mxp, x);
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        mxp = fmaxf(mxp, __shfl_xor_sync(0xffffffffu, mxp, o));
      }
      const float mold = ex.m[j], mnew = fmaxf(mold, mx);
      const float pmold = ex.pm[j], pmnew = fmaxf(pmold, mxp);
      float sum = 0.f, psum = 0.f;
      for (int i = lane; i < count; i += 32) {
        const float x = ex.sc[j][i];
        const float p = mnew == -CUDART_INF_F ? 0.f : fast_exp2(x - mnew);
        if (i < npc) psum += pmnew == -CUDART_INF_F ? 0.f : fast_exp2(x - pmnew);
        ex.sc[j][i] = p;
        sum += p;
      }
      sum = warp_sum_all(sum);
      psum = warp_sum_all(psum);
      __syncwarp();
      if (lane == 0) {
        const float f = mold == -CUDART_INF_F ? 0.f : exp2f(mold - mnew);
        ex.fac[j] = f;
        ex.m[j] = mnew;
        ex.l[j] = ex.l[j] * f + sum;
        const float pf = pmold == -CUDART_INF_F ? 0.f : exp2f(pmold - pmnew);
        ex.pm[j] = pmnew;
        ex.pl[j] = ex.pl[j] * pf + psum;
      }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      const float f = ex.fac[j];
      acc[j][0] *= f;
      acc[j][1] *= f;
      acc[j][2] *= f;
      acc[j][3] *= f;
    }
    // ---- P.V: kRows value rows per warp batch, loads first
    for (int it0 = warp; it0 < count; it0 += kWarps * kRows) {
      uint2 vwr[kRows];
#pragma unroll
      for (int u = 0; u < kRows; ++u) {
        const int it = it0 + u * kWarps;
        vwr[u] = make_uint2(0u, 0u);
        if (it < count) {
          const __nv_bfloat16 *kr, *vr;
          int pos;
          bool spec;
          row_ptr(c0 + it, kr, vr, pos, spec);
          vwr[u] = *reinterpret_cast<const uint2*>(vr + 4 * lane);
        }
      }
#pragma unroll
      for (int u = 0; u < kRows; ++u) {
        const int it = it0 + u * kWarps;
        if (it < count) {
          const __nv_bfloat162 v01 = *reinterpret_cast<const __nv_bfloat162*>(&vwr[u].x);
          const __nv_bfloat162 v23 = *reinterpret_cast<const __nv_bfloat162*>(&vwr[u].y);
          const float x0 = __low2float(v01), x1 = __high2float(v01), x2 = __low2float(v23), x3 = __high2float(v23);
#pragma unroll
          for (int j = 0; j < NR; ++j) {
            const float p = ex.sc[j][it];
            acc[j][0] = fmaf(p, x0, acc[j][0]);
            acc[j][1] = fmaf(p, x1, acc[j][1]);
            acc[j][2] = fmaf(p, x2, acc[j][2]);
            acc[j][3] = fmaf(p, x3, acc[j][3]);
          }
        }
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < NR; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) ex.o[warp][j][4 * lane + i] = acc[j][i];
  __syncthreads();
  const size_t base = (((size_t)b * G.H + h) * (a.nsplit + 1) + split) * NR;
  for (int i = tid; i < NR * 128; i += kThreads) {
    const int j = i >> 7, c = i & 127;
    float o = 0.f;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) o += ex.o[w][j][c];
    a.part_o[(base + j) * 128 + c] = o;
  }
  if (tid < NR) {
    a.part_ml[(base + tid) * 2 + 0] = ex.m[tid];
    a.part_ml[(base + tid) * 2 + 1] = ex.l[tid];
    const size_t pb = ((size_t)b * G.H + h) * NR + tid;
    a.pin_ml[pb * 2 + 0] = ex.pm[tid];
    a.pin_ml[pb * 2 + 1] = ex.pl[tid];
  }
}

#ifndef SPC_K2_TSC
#define SPC_K2_TSC 1  // 8-row GQA: transposed scores (rows on the MMA M side, P stays in registers)
#endif
#ifndef SPC_K2_UWARP_NR
#define SPC_K2_UWARP_NR 8  // widest row count whose warp index is made uniform (see k_attend_fast)
#endif
#ifndef SPC_K2_GQA_MAXREG
#define SPC_K2_GQA_MAXREG 0
#endif
// Register cap of the wide GQA instantiations (NR >= 4; 0 = the 2-CTA launch
// bound's 128).  At <= 120 registers two resident K2 CTAs leave 4096 registers
// of the SM free, so small side kernels can run beside them instead of waiting
// for a K2 CTA to retire.
template <int NR>
constexpr int k2_maxreg() { return (SPC_K2_GQA_MAXREG > 0 && NR >= 4) ? SPC_K2_GQA_MAXREG : 128; }

template <int BITS, int NR, int FOLD>
__global__ void __maxnreg__(k2_maxreg<NR>()) k_attend_fast(AttnArgs a) {
  constexpr int kSt = stages_of<BITS, NR>();
  // PACK: score MMA columns n = 2*row + plane (hi/lo of each row side by side),
  //       one MMA per k-step and one score row per lane (row = lane & 3).
  // PG:   P.V columns n = group*NR + row, one B fragment for all value groups.
  constexpr bool PACK = (2 * NR <= 8);
  constexpr bool PG = (NR * 4 <= 8);
  constexpr int RPL = PACK ? 1 : 2;  // score rows per lane
  using SL = StageLayout<BITS>;
  const Geo& G = a.G;
  const LayerBufs& B = a.B;
  int split, h, b;
  if (kExactOrder == 0) {
    split = blockIdx.x;
    h = blockIdx.y;
    b = blockIdx.z;
  } else {
    const int units = a.G.H * a.G.batch, nmain = units * a.nsplit;
    const int L = kExactOrder == 1 ? (int)blockIdx.x : ((int)blockIdx.x + nmain) % (nmain + units);
    int u;
    if (L < nmain) {
      u = L / a.nsplit;
      split = L - u * a.nsplit;
    } else {
      u = L - nmain;
      split = a.nsplit;
    }
    h = u % a.G.H;
    b = u / a.G.H;
  }
  extern __shared__ __align__(16) unsigned char smem_raw[];
  if (split == a.nsplit) {
    if constexpr (NR == 8) exact_segment_rows<NR>(a, split, h, b, smem_raw);
    else exact_segment_fast<NR>(a, split, h, b, smem_raw);
    return;
  }
  // warp index through a shuffle: the compiler then treats it (and the block
  // index, ring stage and record address derived from it) as warp-uniform, so
  // the per-block bulk copy takes its operands from uniform registers instead
  // of a divergent R2UR waterfall loop around UBLKCP.  (The 8-row instantiations
  // spilled with it before the transposed scores freed their registers.)
  const int warp = NR <= SPC_K2_UWARP_NR ? __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0) : (int)(threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  WarpSmem<BITS, NR>& ws = reinterpret_cast<WarpSmem<BITS, NR>*>(smem_raw)[warp];

  const int nb_total = a.f / 32;
  const int blk0 = split * a.blocks_per_split;
  const int blk1 = min(nb_total, blk0 + a.blocks_per_split);
  const float cs = BITS == 1 ? 0.5f : (1.f / 3.f);
  const size_t bi0 = blk_index(G, b, h, 0);
  const uint32_t* rec_base = B.kcodes + bi0 * (size_t)SL::words;
  const uint32_t* bm_base = B.bitmap + ((size_t)b * G.U + (G.scope ? h : 0)) * (G.L / 32);

  // ---- TMA ring prologue -------------------------------------------------------------
  // shared addresses of stage 0 / barrier 0 and their strides, computed once
  const unsigned stage0 = smem_u32(ws.stage[0]), bar0 = smem_u32(&ws.bar[0]);
  constexpr unsigned kStageBytes = sizeof(ws.stage[0]);
  auto issue = [&](const uint32_t* src, int st) {
    const unsigned bar = bar0 + 8u * st;
    mbar_expect_tx_u32(bar, SL::bytes);  // the whole block record, one bulk copy
    tma_load_u32(stage0 + kStageBytes * st, src, SL::bytes, bar);
  };
  // refill of a consumed stage (async proxy after the lanes' generic reads).  With a
  // warp-uniform warp index the whole warp runs it and elect.sync picks the issuing
  // lane inside the asm: no divergent branch, so no ELECT loop around UBLKCP.
  auto refill = [&](const uint32_t* src, int st, bool more) {
    if (NR <= SPC_K2_UWARP_NR) {
      if (more) {
        fence_proxy_async();
        const unsigned bar = bar0 + 8u * st, dst = stage0 + kStageBytes * st;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "elect.sync _|p, 0xffffffff;\n\t"
            "@p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t"
            "@p cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%2], [%3], %1, [%0];\n\t}"
            ::"r"(bar), "r"(SL::bytes), "r"(dst), "l"(src)
            : "memory");
      }
    } else if (lane == 0 && more) {
      fence_proxy_async();
      issue(src, st);
    }
  };
  if constexpr (PACK && NR == 2) {  // bk padding columns 4*NR.. are the zero rows of the PACK B fragment
    static_assert(WarpSmem<BITS, NR>::kBkRow >= 4 * NR + 4, "PACK zero padding");
    ws.bk[lane >> 2][4 * NR + (lane & 3)] = make_uint4(0u, 0u, 0u, 0u);
  }
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < kSt; ++s) mbar_init(&ws.bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
#pragma unroll
    for (int s = 0; s < kSt; ++s) {
      const int blk = blk0 + warp + s * kWarps;
      if (blk < blk1) issue(rec_base + (size_t)blk * SL::words, s);
    }
  }
  __syncwarp();

  // ---- per-lane constants ---------------------------------------------------------------
  // key-B role: lane (ks = lane&7, tk = lane>>3) owns channels 32tk + ks + 8m, m = 0..3
  const int kks = lane & 7, ktk = lane >> 3;
  constexpr bool QREG = NR <= 2;  // wide GQA rows keep the query slice in shared memory
  float Qr[QREG ? NR : 1][4];
  float4* Qs = reinterpret_cast<float4*>(smem_raw + kWarps * sizeof(WarpSmem<BITS, NR>));  // [NR][32]
  constexpr bool HKB = kHalfKeyB && !QREG;
  // Transposed scores (TSC, 8 rows): D[row hi | row lo][token] = sum_c (Q s)[row][c] code[c][token],
  // A = the per-block Q*s hi/lo rows (mul_hilo in registers), B = the expanded codes, four n-tiles
  // of 8 tokens.  A lane then holds row gq's scores of tokens 8nt + 2tq + {0, 1}: exactly the
  // P.V B-fragment positions, so P never goes through shared memory; the key B table, its
  // fragment loads and the C_j reduce-scatter disappear too.
  constexpr bool TSC = SPC_K2_TSC && NR == 8 && HKB && !kCMma && kVCoop;
  // [NR][kQhS] {Qhi b0, Qhi b1, Qlo b0, Qlo b1} (HKB); row stride 36 keeps the C-MMA
  // A-fragment loads (rows gq, gq + 1 in one 8-lane phase) conflict-free
  constexpr int kQhS = 36;
  uint4* Qh = reinterpret_cast<uint4*>(Qs + NR * 36);
  // Qs slot of lane' = (kks, ktk)'s channels 32ktk + kks + 8m of row j: TSC reads a row's quarter
  // tq as [4kk + tq] (stride 36 per row: the 8 lanes of a phase hit 8 distinct 16-byte banks)
  auto qs_idx = [&](int j, int l) { return TSC ? j * 36 + 4 * (l & 7) + (l >> 3) : j * 32 + l; };
  float qabs = 0.f;
  // the shared query tables (rows > 2) are loaded by warp 0 alone; the others read its
  // max |Q| from shared memory after the barrier below
  float* const qabs_s = reinterpret_cast<float*>(Qh + NR * kQhS);
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    if (!QREG && warp != 0) break;
    const int r = j / G.G, g2 = j - r * G.G;
    const __nv_bfloat16* qp = a.q + (((size_t)b * a.rows + r) * G.Hq + h * G.G + g2) * 128;
    float qv[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      qv[m] = __bfloat162float(qp[32 * ktk + kks + 8 * m]) * a.sm_scale_log2;
      qabs = fmaxf(qabs, fabsf(qv[m]));
    }
    if (QREG) {
#pragma unroll
      for (int m = 0; m < 4; ++m) Qr[QREG ? j : 0][m] = qv[m];
    } else if (warp == 0) {
      Qs[qs_idx(j, lane)] = make_float4(qv[0], qv[1], qv[2], qv[3]);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) qabs = fmaxf(qabs, __shfl_xor_sync(0xffffffffu, qabs, o));
  if (!QREG && warp == 0 && lane == 0) *qabs_s = qabs;
  auto aq_of = [&](float qa) { return (HKB && qa > 0.f) ? ceil_log2(qa) - 7 : 0; };  // max |Q * 2^-aq| in (2^6, 2^7]
  if (HKB && warp == 0) {
    const float sq = pow2i(-aq_of(qabs));
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      const float4 qq = Qs[qs_idx(j, lane)];  // written by this lane above
      uint4 h;
      if (BITS == 2) {  // pairing of the key B fragment: b0 = (m0, m1), b1 = (m2, m3)
        split2(qq.x * sq, qq.y * sq, h.x, h.z);
        split2(qq.z * sq, qq.w * sq, h.y, h.w);
      } else {  // b0 = (m0, m2), b1 = (m1, m3)
        split2(qq.x * sq, qq.z * sq, h.x, h.z);
        split2(qq.y * sq, qq.w * sq, h.y, h.w);
      }
      Qh[j * kQhS + (TSC ? 4 * kks + ktk : lane)] = h;  // TSC: [row][ks][tq] (conflict-free A loads)
    }
  }
  if (!QREG) {
    __syncthreads();
    qabs = *qabs_s;  // warp 0's reduction over the shared rows
  }
  const int aq = aq_of(qabs);
  const float rk = __uint_as_float(B.rmax[((size_t)b * G.H + h) * 4 + 0]) * cs;
  const float rv = __uint_as_float(B.rmax[((size_t)b * G.H + h) * 4 + 1]) * cs;
  const int Ek = (qabs * rk > 0.f) ? ceil_log2(qabs * rk) - 14 : 0;
  // lazy softmax rescale: P = exp2(s - m_run) may reach 2^kSlack, so the value
  // B exponent keeps kSlack bits of headroom (max|P*s'| <= 2^14 still)
  const int Ev = (rv > 0.f) ? ceil_log2(rv) - 14 + kSlackLog2 : 0;
  const int sp = BITS == 2 ? 2 * (kks & 3) : kks;       // K-index (channel) scale of this lane
  const float kscale = cs * pow2i(-sp - Ek + aq);         // (hi-lo) -> s * 2^(-sp-Ek) (* 2^aq: HKB)
  const float k_out = pow2i(24 + Ek);                     // D * k_out = sum_c code * Q * s
  const float v_out = pow2i(24 + Ev);
  constexpr bool VCO = kVCoop && !PG;
  // VCOOP: zero-points as f16 hi + lo of z * 2^-Ez, max |z * 2^-Ez| <= 2^14
  const float rz = __uint_as_float(B.rmax[((size_t)b * G.H + h) * 4 + 3]);
  const int Ez = (VCO && rz > 0.f) ? ceil_log2(rz) - 14 : 0;
  const float zsc = pow2i(-Ez), z_out = pow2i(Ez);
  // z sums at the value accumulator's scale (exact: powers of two); kept in
  // shared memory, the main loop has no register to spare for it
  if (lane == 0) ws.zfold = VCO ? pow2i(Ez - 24 - Ev) : pow2i(-24 - Ev);
  constexpr bool CMM = kCMma && HKB;

  // C-MMA: key zero-points as f16 hi + lo of z * 2^-Ezk (max <= 2^14); D * 2^(Ezk + aq) = C_j
  const float rzk = __uint_as_float(B.rmax[((size_t)b * G.H + h) * 4 + 2]);
  const int Ezk = (CMM && rzk > 0.f) ? ceil_log2(rzk) - 14 : 0;
  const float zksc = pow2i(-Ezk), c_out = pow2i(Ezk + aq);
  float vscale[4];  // value K-index (token) scales, q = 2ks + khalf
#pragma unroll
  for (int q = 0; q < 4; ++q) vscale[q] = cs * pow2i(-(BITS == 2 ? 2 * q : q) - Ev);
  // PG sz decode: this lane's ks = lane & 1 -> q = 2ks + khalf (kept in registers, no local array)
  const float vs_lane[2] = {(lane & 1) ? vscale[2] : vscale[0], (lane & 1) ? vscale[3] : vscale[1]};
  // VCOOP decode role: lane = (group vg, k-step vks, tq); its tokens 16 vks + 2 tq + {0, 1, 8, 9}
  const int vks = (lane >> 2) & 1;
  const float vs_co[2] = {vks ? vscale[2] : vscale[0], vks ? vscale[3] : vscale[1]};
  // score rows of this lane and their spill rows (aggregate source)
  const int agg_j0 = a.agg_row * G.G;
  int jr[RPL];
  float* spr[RPL];
#pragma unroll
  for (int e = 0; e < RPL; ++e) {
    jr[e] = PACK ? tq : 2 * tq + e;
    spr[e] = (!a.agg_recompute && jr[e] < NR && jr[e] >= agg_j0 && jr[e] < agg_j0 + G.G)
                 ? a.spill + ((size_t)b * G.Hq + h * G.G + (jr[e] - agg_j0)) * G.L : nullptr;
  }


  float* const sprT = (TSC && !a.agg_recompute && gq >= agg_j0 && gq < agg_j0 + G.G)
                          ? a.spill + ((size_t)b * G.Hq + h * G.G + (gq - agg_j0)) * G.L : nullptr;
  float m_run[RPL], l_run[RPL];
#pragma unroll
  for (int e = 0; e < RPL; ++e) {
    m_run[e] = -CUDART_INF_F;
    l_run[e] = 0.f;
  }
  float dv[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) dv[i][0] = dv[i][1] = dv[i][2] = dv[i][3] = 0.f;
  float zacc[PG ? 1 : 4];
#pragma unroll
  for (int i = 0; i < (PG ? 1 : 4); ++i) zacc[i] = 0.f;

  // alpha (softmax rescale) of score row j as seen from any lane
  auto alpha_of_row = [&](const float (&al)[RPL], int j) -> float {
    if (PACK) return __shfl_sync(0xffffffffu, al[0], j & 3);
    const float x0 = __shfl_sync(0xffffffffu, al[0], (j >> 1) & 3);
    const float x1 = __shfl_sync(0xffffffffu, al[RPL - 1], (j >> 1) & 3);
    return (j & 1) ? x1 : x0;
  };

  int st = 0;
  unsigned phase = 0;
  // pin bitmap words of this warp's blocks, 32 iterations per window: lane i
  // holds block (window base + i * kWarps); the next window is loaded one
  // window ahead, so the loop reads its word with one shuffle
  auto bm_window = [&](int base) -> uint32_t {
    const int bb = base + lane * kWarps;
    return bb < blk1 ? bm_base[bb] : 0u;
  };
  uint32_t bm_cur = bm_window(blk0 + warp), bm_next = bm_window(blk0 + warp + 32 * kWarps);
  // record of the block that refills the stage consumed in this iteration
  const uint32_t* next_src = rec_base + (size_t)(blk0 + warp + kSt * kWarps) * SL::words;
  int it = 0;
  for (int blk = blk0 + warp; blk < blk1; blk += kWarps, ++it, next_src += kWarps * SL::words) {
    if ((it & 31) == 0 && it) {
      bm_cur = bm_next;
      bm_next = bm_window(blk + 32 * kWarps);
    }
    if (FOLD > 0 && it && (it % FOLD) == 0) {
      // fold sum_t P z into the value accumulator (the epilogue's combination, early)
      const float zfold = *reinterpret_cast<volatile float*>(&ws.zfold);
      if constexpr (PG) {
        float zt = zacc[0];  // lane partials -> the row group's sum (as after the loop)
        zt += __shfl_xor_sync(0xffffffffu, zt, 1);
        zt += __shfl_xor_sync(0xffffffffu, zt, 2);
        const float zc0 = __shfl_sync(0xffffffffu, zt, 4 * (2 * tq)) * zfold;
        const float zc1 = __shfl_sync(0xffffffffu, zt, 4 * ((2 * tq + 1) & 7)) * zfold;
#pragma unroll
        for (int mt = 0; mt < 8; ++mt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int n = 2 * tq + e;
            if (n < 4 * NR && n / NR == (mt >> 1)) {
              dv[mt][e] += e ? zc1 : zc0;
              dv[mt][2 + e] += e ? zc1 : zc0;
            }
          }
        zacc[0] = 0.f;
      } else if constexpr (VCO) {
        const float zs0 = (zacc[0] + zacc[2 % (PG ? 1 : 4)]) * zfold;
        const float zs1 = (zacc[1 % (PG ? 1 : 4)] + zacc[3 % (PG ? 1 : 4)]) * zfold;
#pragma unroll
        for (int gi = 0; gi < 4; ++gi) {
          const float z0 = __shfl_sync(0xffffffffu, zs0, 4 * gi + tq);
          const float z1 = __shfl_sync(0xffffffffu, zs1, 4 * gi + tq);
#pragma unroll
          for (int mt = 2 * gi; mt < 2 * gi + 2; ++mt) {
            dv[mt][0] += z0;
            dv[mt][2] += z0;
            dv[mt][1] += z1;
            dv[mt][3] += z1;
          }
        }
#pragma unroll
        for (int i = 0; i < (PG ? 1 : 4); ++i) zacc[i] = 0.f;
      }
    }
    const uint32_t bm = __shfl_sync(0xffffffffu, bm_cur, it & 31);
    mbar_wait(&ws.bar[st], phase);
    // order the previous block's reads of ws.sz / ws.P before this block's writes
    // by other lanes (independent thread scheduling; compute-sanitizer racecheck)
    __syncwarp();
    const uint32_t* S = ws.stage[st];

    // ---- key B fragments (cooperative) + zero-point constants C_j -----------------------
    float Cp[NR];
    // TSC tables (in the unused key-B area): [ks][tq] {s hi c0, s hi c1, s lo c0, s lo c1}, then
    // at [4kks + ktk] the zero-points of lane' = (kks, ktk)'s channels 32ktk + kks + 8m
    uint4* const tst = reinterpret_cast<uint4*>(&ws.bk[0][0]);
    float4* const tzt = reinterpret_cast<float4*>(&ws.bk[0][0]) + 32;
    if constexpr (TSC) {
      const uint4 kp4 = *reinterpret_cast<const uint4*>(S + SL::kp + 4 * lane);
      const uint32_t kpw[4] = {kp4.x, kp4.y, kp4.z, kp4.w};
      float s4[4], z4[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const float lo = __uint_as_float(kpw[m] << 16), hi = __uint_as_float(kpw[m] & 0xFFFF0000u);
        s4[m] = (hi - lo) * kscale;
        z4[m] = BITS == 1 ? fmaf(0.75f, lo, 0.25f * hi) : lo;
      }
      uint32_t sh0, sl0, sh1, sl1;
      if (BITS == 2) {
        split2(s4[0], s4[1], sh0, sl0);
        split2(s4[2], s4[3], sh1, sl1);
      } else {
        split2(s4[0], s4[2], sh0, sl0);
        split2(s4[1], s4[3], sh1, sl1);
      }
      tst[4 * kks + ktk] = make_uint4(sh0, sh1, sl0, sl1);
      tzt[4 * kks + ktk] = make_float4(z4[0], z4[1], z4[2], z4[3]);
    } else {
      const uint4 kp4 = *reinterpret_cast<const uint4*>(S + SL::kp + 4 * lane);
      const uint32_t kpw[4] = {kp4.x, kp4.y, kp4.z, kp4.w};
      float s4[4], z4[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const float lo = __uint_as_float(kpw[m] << 16), hi = __uint_as_float(kpw[m] & 0xFFFF0000u);
        s4[m] = (hi - lo) * kscale;
        z4[m] = BITS == 1 ? fmaf(0.75f, lo, 0.25f * hi) : lo;
      }
      uint32_t sh0 = 0, sl0 = 0, sh1 = 0, sl1 = 0;  // HKB: this block's scale pairs, shared by all rows
      if (HKB) {
        if (BITS == 2) {
          split2(s4[0], s4[1], sh0, sl0);
          split2(s4[2], s4[3], sh1, sl1);
        } else {
          split2(s4[0], s4[2], sh0, sl0);
          split2(s4[1], s4[3], sh1, sl1);
        }
      }
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        float q0, q1, q2, q3;
        if (HKB) {
          if (!CMM) {
            const float4 qq = Qs[j * 32 + lane];
            Cp[j] = fmaf(qq.x, z4[0], fmaf(qq.y, z4[1], fmaf(qq.z, z4[2], qq.w * z4[3])));
          }
          const uint4 qh = Qh[j * kQhS + lane];
          uint4 frag;
          mul_hilo(qh.x, qh.z, sh0, sl0, frag.x, frag.z);
          mul_hilo(qh.y, qh.w, sh1, sl1, frag.y, frag.w);
          ws.bk[kks][4 * j + (ktk ^ ((kks >> 1) & 3))] = frag;
          continue;
        }
        if (QREG) {
          q0 = Qr[QREG ? j : 0][0];
          q1 = Qr[QREG ? j : 0][1];
          q2 = Qr[QREG ? j : 0][2];
          q3 = Qr[QREG ? j : 0][3];
        } else {
          const float4 qq = Qs[j * 32 + lane];
          q0 = qq.x;
          q1 = qq.y;
          q2 = qq.z;
          q3 = qq.w;
        }
        const float w0 = q0 * s4[0], w1 = q1 * s4[1], w2 = q2 * s4[2], w3 = q3 * s4[3];
        Cp[j] = fmaf(q0, z4[0], fmaf(q1, z4[1], fmaf(q2, z4[2], q3 * z4[3])));
        uint4 frag;  // {b0hi, b1hi, b0lo, b1lo} of row j for fragment lane (j, tk)
        if (BITS == 2) {  // b0 = (m0, m1), b1 = (m2, m3)
          split2(w0, w1, frag.x, frag.z);
          split2(w2, w3, frag.y, frag.w);
        } else {  // b0 = (m0, m2), b1 = (m1, m3)
          split2(w0, w2, frag.x, frag.z);
          split2(w1, w3, frag.y, frag.w);
        }
        ws.bk[kks][4 * j + (ktk ^ ((kks >> 1) & 3))] = frag;
      }
      if constexpr (CMM) {
        // this lane's key zero-points as f16 hi + lo pairs (same pairing as the Qh table)
        // into the padding columns of bk: slot L = lane -> bk[L >> 2][4 NR + (L & 3)]
        float zz[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) zz[m] = z4[m] * zksc;
        uint32_t zh0, zl0, zh1, zl1;
        if (BITS == 2) {
          split2(zz[0], zz[1], zh0, zl0);
          split2(zz[2], zz[3], zh1, zl1);
        } else {
          split2(zz[0], zz[2], zh0, zl0);
          split2(zz[1], zz[3], zh1, zl1);
        }
        ws.bk[lane >> 2][4 * NR + (lane & 3)] = make_uint4(zh0, zh1, zl0, zl1);
      } else {
        // reduce-scatter of the NR per-lane partials: after log2(NR) halving steps a
        // lane holds one row, r = lane >> (5 - log2 NR); the remaining butterflies
        // finish the sum (NR=8: 9 SHFL instead of 40)
        constexpr int LG = NR == 1 ? 0 : NR == 2 ? 1 : NR == 4 ? 2 : 3;
        float v[NR];
#pragma unroll
        for (int j = 0; j < NR; ++j) v[j] = Cp[j];
#pragma unroll
        for (int st2 = 0; st2 < LG; ++st2) {
          const int o = 16 >> st2, half = NR >> (st2 + 1);
          const bool up = lane & o;
#pragma unroll
          for (int i2 = 0; i2 < half; ++i2) {
            const float keep = up ? v[i2 + half] : v[i2], send = up ? v[i2] : v[i2 + half];
            v[i2] = keep + __shfl_xor_sync(0xffffffffu, send, o);
          }
        }
#pragma unroll
        for (int o = 16 >> LG; o; o >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
        Cp[0] = v[0];  // row (lane >> (5 - LG)) of this lane
      }
    }  // !TSC
    // value params -> (s * 2^-(q+Ev), z) once per block: lane l decodes words 4l..4l+3
    // (group l>>3, tq (l>>1)&3, ks l&1, slots 0..3; slot>>1 = khalf -> q = 2ks + khalf)
    if constexpr (PG) {
      const uint4 vp4 = *reinterpret_cast<const uint4*>(S + SL::vp + 4 * lane);
      const uint32_t vpw[4] = {vp4.x, vp4.y, vp4.z, vp4.w};
      float o[8];
#pragma unroll
      for (int slot = 0; slot < 4; ++slot) {
        const float lo = __uint_as_float(vpw[slot] << 16), hi = __uint_as_float(vpw[slot] & 0xFFFF0000u);
        o[2 * slot] = (hi - lo) * vs_lane[slot >> 1];
        o[2 * slot + 1] = BITS == 1 ? fmaf(0.75f, lo, 0.25f * hi) : lo;
      }
      ws.sz[WarpSmem<BITS, NR>::szidx(2 * lane)] = make_float4(o[0], o[1], o[2], o[3]);
      ws.sz[WarpSmem<BITS, NR>::szidx(2 * lane + 1)] = make_float4(o[4], o[5], o[6], o[7]);
    } else if constexpr (VCO) {
      // lane = (vg = lane >> 3, vks, tq): words 32 vg + 8 tq + 4 vks + slot, slot = (t & 1) + 2 khalf
      const uint4 vq = *reinterpret_cast<const uint4*>(S + SL::vp + 32 * (lane >> 3) + 8 * tq + 4 * vks);
      const uint32_t w4[4] = {vq.x, vq.y, vq.z, vq.w};
      float sv[4], zv[4];
#pragma unroll
      for (int slot = 0; slot < 4; ++slot) {
        const float lo = __uint_as_float(w4[slot] << 16), hi = __uint_as_float(w4[slot] & 0xFFFF0000u);
        sv[slot] = (hi - lo) * vs_co[slot >> 1];
        zv[slot] = (BITS == 1 ? fmaf(0.75f, lo, 0.25f * hi) : lo) * zsc;
      }
      uint4 sb, za;
      split2(sv[0], sv[1], sb.x, sb.z);
      split2(sv[2], sv[3], sb.y, sb.w);
      split2(zv[0], zv[1], za.x, za.y);
      split2(zv[2], zv[3], za.z, za.w);
      uint4* vsb = reinterpret_cast<uint4*>(ws.sz);       // [vg][vks][tq] {sh01, sh89, sl01, sl89}
      // z A fragments [vks][tq][vg ^ swz(tq)] {zh01, zl01, zh89, zl89}: rows g (hi) and g + 8 (lo)
      uint4* vza = reinterpret_cast<uint4*>(ws.sz + 32);
      vsb[lane] = sb;
      vza[vks * 16 + tq * 4 + ((lane >> 3) ^ ((tq >> 1) << 1))] = za;
    }
    // key codes of this lane's tokens T0 = 16mt + gq, T1 = T0 + 8
    uint32_t kw[2][2 * BITS];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        const int T = 16 * mt + gq + 8 * hf;
        if (BITS == 2) {
          const uint2 w = *reinterpret_cast<const uint2*>(S + SL::kc + T * 8 + 2 * tq);
          kw[mt][2 * hf] = w.x;
          kw[mt][2 * hf + 1] = w.y;
        } else {
          kw[mt][hf] = S[SL::kc + T * 4 + tq];
        }
      }
    }
    __syncwarp();

    if constexpr (CMM) {  // C_j = sum_c Q[j,c] z_c: A = Qh rows (hi 0-7, lo 8-15), B = z (hi col 0, lo col 1)
      float cacc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int kc = 0; kc < 8; ++kc) {
        const uint4 qa = gq < NR ? Qh[gq * kQhS + 4 * kc + tq] : make_uint4(0u, 0u, 0u, 0u);
        uint2 zb = make_uint2(0u, 0u);
        if (gq < 2) zb = reinterpret_cast<const uint2*>(&ws.bk[kc][4 * NR + tq])[gq];
        mma16816(cacc, qa.x, qa.z, qa.y, qa.w, zb.x, zb.y);
      }
      Cp[0] = ((cacc[0] + cacc[1]) + (cacc[2] + cacc[3])) * c_out;  // row gq (valid in lanes tq == 0)
    }
    float ptsc[TSC ? 4 : 1][2];  // TSC: P of row gq, tokens 8nt + 2tq + {0, 1}
    if constexpr (TSC) {
      // C_j of row gq over this lane's quarter of the channels (32tq .. 32tq + 31): tables in
      // [4kk + tq] order, so the 8 lanes of a shared-memory phase read 8 distinct 16-byte banks
      // (Qs) or broadcast (z) with immediate offsets
      float cj = 0.f;
      {
        const float4* qrow = Qs + gq * 36 + tq;
        const float4* zrow = tzt + tq;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float4 qq = qrow[4 * k], zz = zrow[4 * k];
          cj = fmaf(qq.x, zz.x, fmaf(qq.y, zz.y, fmaf(qq.z, zz.z, fmaf(qq.w, zz.w, cj))));
        }
        cj += __shfl_xor_sync(0xffffffffu, cj, 1);
        cj += __shfl_xor_sync(0xffffffffu, cj, 2);
      }
      float d[4][4];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) d[nt][0] = d[nt][1] = d[nt][2] = d[nt][3] = 0.f;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const uint4 qh = Qh[gq * kQhS + 4 * ks + tq];  // {Q hi c0, Q hi c1, Q lo c0, Q lo c1} of row gq
        const uint4 sv = tst[4 * ks + tq];
        uint32_t a0, a1, a2, a3;  // rows gq (hi) and gq + 8 (lo); K pairs c0 = (2tq, 2tq+1), c1 = (+8, +9)
        mul_hilo(qh.x, qh.z, sv.x, sv.z, a0, a1);
        mul_hilo(qh.y, qh.w, sv.y, sv.w, a2, a3);
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {  // n-tile 2mt + hf: tokens 16mt + 8hf + (0..7), this lane's gq
            uint32_t b0, b1;
            if (BITS == 2) {
              const uint32_t msk = (3u << (2 * (ks & 3))) | (3u << (16 + 2 * (ks & 3)));
              const int sh = ks < 4 ? 0 : 8;
              b0 = (kw[mt][2 * hf] >> sh) & msk;
              b1 = (kw[mt][2 * hf + 1] >> sh) & msk;
            } else {
              const uint32_t msk = (1u << ks) | (1u << (16 + ks));
              b0 = kw[mt][hf] & msk;
              b1 = (kw[mt][hf] >> 8) & msk;
            }
            mma16816(d[2 * mt + hf], a0, a1, a2, a3, b0, b1);
          }
      }
      // log2 scores of row gq, tokens 8nt + 2tq + e; pins masked; speculative rows spilled
      float sct[4][2];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) sct[nt][e] = fmaf(d[nt][e] + d[nt][2 + e], k_out, cj);
      const uint32_t bq2 = bm >> (2 * tq);
      if (bm) {
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e)
            if ((bq2 >> (8 * nt + e)) & 1u) sct[nt][e] = -CUDART_INF_F;
      }
      if (!kNoSpill && sprT) {
        float* sp = sprT + blk * 32 + 2 * tq;
        if (!(bq2 & 0x03030303u)) {  // no pinned token among this lane's 8: four 8-byte stores
#pragma unroll
          for (int nt = 0; nt < 4; ++nt)
            *reinterpret_cast<float2*>(sp + 8 * nt) = make_float2(sct[nt][0], sct[nt][1]);
        } else {
#pragma unroll
          for (int nt = 0; nt < 4; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e)
              if (!((bq2 >> (8 * nt + e)) & 1u)) sp[8 * nt + e] = sct[nt][e];
        }
      }
      float mloc = fmaxf(fmaxf(sct[0][0], sct[0][1]), fmaxf(sct[1][0], sct[1][1]));
      mloc = fmaxf(mloc, fmaxf(fmaxf(sct[2][0], sct[2][1]), fmaxf(sct[3][0], sct[3][1])));
      if (__any_sync(0xffffffffu, mloc > m_run[0] + kSlack)) {
        float mx = fmaxf(mloc, __shfl_xor_sync(0xffffffffu, mloc, 1));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        const float mn = fmaxf(m_run[0], mx);
        const float al = m_run[0] == -CUDART_INF_F ? 0.f : fast_exp2(m_run[0] - mn);
        l_run[0] *= al;
        m_run[0] = mn;
        // value accumulator columns = rows 2tq, 2tq + 1 (their alphas from lanes of those rows)
        const float ac0 = __shfl_sync(0xffffffffu, al, 8 * tq), ac1 = __shfl_sync(0xffffffffu, al, 8 * tq + 4);
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
          dv[mt][0] *= ac0;
          dv[mt][1] *= ac1;
          dv[mt][2] *= ac0;
          dv[mt][3] *= ac1;
        }
        zacc[0] *= ac0;
        zacc[1 % (PG ? 1 : 4)] *= ac1;
        zacc[2 % (PG ? 1 : 4)] *= ac0;
        zacc[3 % (PG ? 1 : 4)] *= ac1;
      }
      const float mr = m_run[0] == -CUDART_INF_F ? 0.f : m_run[0];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          ptsc[TSC ? nt : 0][e] = fast_exp2(sct[nt][e] - mr);
          l_run[0] += ptsc[TSC ? nt : 0][e];
        }
    } else {
    // ---- scores -------------------------------------------------------------------------
    float dk[2][4], dl[2][4];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int i = 0; i < 4; ++i) dk[mt][i] = dl[mt][i] = 0.f;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      uint32_t b0, b1, b2 = 0, b3 = 0;
      if (PACK) {  // column n = gq = 2*row + plane; rows >= NR are zero columns
        uint2 bb = make_uint2(0, 0);
        if constexpr (NR == 2) {  // rows >= NR read the zeroed padding of bk (no predicate, no zeroing)
          bb = reinterpret_cast<const uint2*>(&ws.bk[ks][4 * min(gq >> 1, NR) + (tq ^ ((ks >> 1) & 3))])[gq & 1];
        } else if ((gq >> 1) < NR) {
          bb = reinterpret_cast<const uint2*>(&ws.bk[ks][4 * (gq >> 1) + (tq ^ ((ks >> 1) & 3))])[gq & 1];
        }
        b0 = bb.x;
        b1 = bb.y;
      } else {
        const uint4 bb = ws.bk[ks][4 * gq + (tq ^ ((ks >> 1) & 3))];
        b0 = bb.x;
        b1 = bb.y;
        b2 = bb.z;
        b3 = bb.w;
      }
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
          a0 = kw[mt][0] & msk;         // T0, channels (32tq+ks, +16)
          a2 = (kw[mt][0] >> 8) & msk;  // T0, channels (32tq+8+ks, +24)
          a1 = kw[mt][1] & msk;
          a3 = (kw[mt][1] >> 8) & msk;
        }
        // PACK: hi/lo split over k-step parity into two independent chains
        if (PACK) {
          if (ks & 1) mma16816(dl[mt], a0, a1, a2, a3, b0, b1);
          else mma16816(dk[mt], a0, a1, a2, a3, b0, b1);
        } else {
          mma16816(dk[mt], a0, a1, a2, a3, b0, b1);
          mma16816(dl[mt], a0, a1, a2, a3, b2, b3);
        }
      }
    }

    // ---- epilogue: log2 scores, mask, spill, online softmax ----------------------------
    float cr[RPL];
    {
      constexpr int LG = NR == 1 ? 0 : NR == 2 ? 1 : NR == 4 ? 2 : 3;
#pragma unroll
      for (int e = 0; e < RPL; ++e)
        cr[e] = __shfl_sync(0xffffffffu, Cp[0], CMM ? 4 * (jr[e] & (NR - 1)) : (jr[e] & (NR - 1)) << (5 - LG));
    }
    // sc[mt][hf][e]: token T = 16mt + gq + 8hf, row jr[e]
    float sc[2][2][RPL];
    const int pos0 = blk * 32;
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
#pragma unroll
        for (int e = 0; e < RPL; ++e) {
          float d;
          if (PACK) d = (dk[mt][2 * hf] + dl[mt][2 * hf]) + (dk[mt][2 * hf + 1] + dl[mt][2 * hf + 1]);
          else d = dk[mt][2 * hf + e] + dl[mt][2 * hf + e];
          sc[mt][hf][e] = fmaf(d, k_out, cr[e]);
        }
      }
    }
    // this lane's tokens T = 16mt + gq + 8hf are bits 0, 8, 16, 24 of bq
    const uint32_t bq = bm >> gq;
    if (bm) {  // pinned positions are attended from their exact rows (exact segment)
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int hf = 0; hf < 2; ++hf)
          if ((bq >> (16 * mt + 8 * hf)) & 1u) {
#pragma unroll
            for (int e = 0; e < RPL; ++e) sc[mt][hf][e] = -CUDART_INF_F;
          }
    }
#pragma unroll
    for (int e = 0; e < RPL; ++e) {
      if (!kNoSpill && spr[e]) {  // aggregate-row logits (one writer per position: pinned ones by the exact segment)
        float* sp = spr[e] + pos0 + gq;
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int hf = 0; hf < 2; ++hf)
            if (!((bq >> (16 * mt + 8 * hf)) & 1u)) sp[16 * mt + 8 * hf] = sc[mt][hf][e];
      }
    }
    float mloc[RPL];
    bool grow = false;
#pragma unroll
    for (int e = 0; e < RPL; ++e) {
      mloc[e] = fmaxf(fmaxf(sc[0][0][e], sc[0][1][e]), fmaxf(sc[1][0][e], sc[1][1][e]));
      grow |= mloc[e] > m_run[e] + kSlack;  // -inf + kSlack = -inf: any finite score grows
    }
    if (__any_sync(0xffffffffu, grow)) {
      float al[RPL];
#pragma unroll
      for (int e = 0; e < RPL; ++e) {
        const float mn = fmaxf(m_run[e], warp_max_g(mloc[e]));
        al[e] = m_run[e] == -CUDART_INF_F ? 0.f : fast_exp2(m_run[e] - mn);
        l_run[e] *= al[e];
        m_run[e] = mn;
      }
      // value accumulator columns n = 2tq + e' and the z role of this lane
      float ac[2], az;
      if (PG) {
        ac[0] = alpha_of_row(al, (2 * tq) % NR);
        ac[1] = alpha_of_row(al, (2 * tq + 1) % NR);
        az = alpha_of_row(al, gq % NR);
      } else {
        ac[0] = alpha_of_row(al, 2 * tq);
        ac[1] = alpha_of_row(al, 2 * tq + 1);
        az = alpha_of_row(al, gq);
      }
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        dv[mt][0] *= ac[0];
        dv[mt][1] *= ac[1];
        dv[mt][2] *= ac[0];
        dv[mt][3] *= ac[1];
      }
      if (VCO) {  // z MMA accumulator: D columns = rows 2tq, 2tq+1 like dv
        zacc[0] *= ac[0];
        zacc[1] *= ac[1];
        zacc[2 % (PG ? 1 : 4)] *= ac[0];
        zacc[3 % (PG ? 1 : 4)] *= ac[1];
      } else {
#pragma unroll
        for (int i = 0; i < (PG ? 1 : 4); ++i) zacc[i] *= az;
      }
    }
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        const int T = 16 * mt + gq + 8 * hf;
#pragma unroll
        for (int e = 0; e < RPL; ++e) {
          // m_run = -inf only while every score so far is masked: P = 0, not exp2(NaN)
          const float p = fast_exp2(sc[mt][hf][e] - (m_run[e] == -CUDART_INF_F ? 0.f : m_run[e]));
          l_run[e] += p;
          if (jr[e] < NR) ws.P[WarpSmem<BITS, NR>::pidx(jr[e], T)] = p;
        }
      }
    }
    }  // !TSC
    __syncwarp();

    if constexpr (PG) {
    // value codes of this lane
    uint32_t vw[4 * BITS];
    {
      const uint4 w0 = *reinterpret_cast<const uint4*>(S + SL::vc + lane * 4);
      vw[0] = w0.x;
      vw[1] = w0.y;
      vw[2] = w0.z;
      vw[3] = w0.w;
      if (BITS == 2) {
        const uint4 w1 = *reinterpret_cast<const uint4*>(S + SL::vc + 128 + lane * 4);
        vw[4 % (4 * BITS)] = w1.x;
        vw[5 % (4 * BITS)] = w1.y;
        vw[6 % (4 * BITS)] = w1.z;
        vw[7 % (4 * BITS)] = w1.w;
      }
    }
    __syncwarp();
    // the stage is consumed (codes in registers, params decoded to ws.sz): refill it
    // with block it + kSt (async proxy after generic reads)
    refill(next_src, st, blk + kSt * kWarps < blk1);

    // ---- P.V: B fragments (f16 hi + lo: sum_t P*z and sum_t P*s*code may nearly
    // cancel) and MMAs over 8 channel m-tiles x 2 token k-steps.  PG: one B for
    // all groups (column n = gq -> (grp = gq / NR, row = gq % NR)); otherwise
    // row = gq and group gi's fragment is built right before its two m-tiles.
#pragma unroll
    for (int gi = 0; gi < (PG ? 1 : 4); ++gi) {
      const int grp = PG ? ((gq / NR) & 3) : gi;
      const int row = PG ? (gq % NR) : gq;
      const bool live = PG ? (gq < 4 * NR) : (gq < NR);
      const int prow = row < NR ? row : 0;
      uint32_t vb[2][4];  // [ks] {b0hi, b1hi, b0lo, b1lo}
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        // (s', z) of tokens 16ks + 2tq + {0,1,8,9} of group grp: words 32grp + 8tq + 4ks + slot
        const float4 sz0 = ws.sz[WarpSmem<BITS, NR>::szidx(16 * grp + 4 * tq + 2 * ks)];
        const float4 sz1 = ws.sz[WarpSmem<BITS, NR>::szidx(16 * grp + 4 * tq + 2 * ks + 1)];
        const float spr4[4] = {sz0.x, sz0.z, sz1.x, sz1.z}, zz4[4] = {sz0.y, sz0.w, sz1.y, sz1.w};
        float x[4];
        // P of tokens (t0, t0+1) and (t0+8, t0+9): two 8-byte loads
        const int t0 = 16 * ks + 2 * tq;
        float2 p01 = *reinterpret_cast<const float2*>(&ws.P[WarpSmem<BITS, NR>::pidx(prow, t0)]);
        float2 p89 = *reinterpret_cast<const float2*>(&ws.P[WarpSmem<BITS, NR>::pidx(prow, t0 + 8)]);
        if (!live) p01 = p89 = make_float2(0.f, 0.f);
        const float pv[4] = {p01.x, p01.y, p89.x, p89.y};
#pragma unroll
        for (int slot = 0; slot < 4; ++slot) {
          const float p = pv[slot];
          zacc[gi] = fmaf(p, zz4[slot], zacc[gi]);
          x[slot] = p * spr4[slot];
        }
        split2(x[0], x[1], vb[ks][0], vb[ks][2]);
        split2(x[2], x[3], vb[ks][1], vb[ks][3]);
      }
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
#pragma unroll
        for (int mt = PG ? 0 : 2 * gi; mt < (PG ? 8 : 2 * gi + 2); ++mt) {
          uint32_t a0, a1, a2, a3;
          const int q0 = 2 * ks, q1 = 2 * ks + 1;
          if (BITS == 2) {
            const uint32_t W = vw[mt % (4 * BITS)], W8 = W >> 8;
            const uint32_t m0 = (3u << (2 * q0)) | (3u << (16 + 2 * q0));
            const uint32_t m1 = (3u << (2 * q1)) | (3u << (16 + 2 * q1));
            a0 = W & m0;
            a1 = W8 & m0;
            a2 = W & m1;
            a3 = W8 & m1;
          } else {
            const uint32_t W = vw[(mt >> 1) % (4 * BITS)] >> (8 * (mt & 1)), W4 = W >> 4;
            const uint32_t m0 = (1u << q0) | (1u << (16 + q0));
            const uint32_t m1 = (1u << q1) | (1u << (16 + q1));
            a0 = W & m0;
            a1 = W4 & m0;
            a2 = W & m1;
            a3 = W4 & m1;
          }
          mma16816(dv[mt], a0, a1, a2, a3, vb[ks][0], vb[ks][1]);
          mma16816(dv[mt], a0, a1, a2, a3, vb[ks][2], vb[ks][3]);
        }
      }
    }
    } else {
    // ---- value B fragments (f16 hi + lo: sum_t P*z and sum_t P*s*code may nearly cancel)
    // PG: lane column n = gq -> (grp = gq / NR, row = gq % NR); else row = gq, per group
    // Token-outer order: the lane's P values of a k-step (and P * token scale,
    // P / 4 for the 1-bit zero point z = lo + (hi - lo) / 4) are formed once and
    // shared by the four groups; per group and token only lo, hi, hi - lo and
    // two products remain.
    uint32_t vb[4][2][4];  // [grp][ks] {b0hi, b1hi, b0lo, b1lo}
    if constexpr (VCO) {
      // P pairs of this lane's row gq, tokens 16ks + 2tq + {0,1} (half 0) / {8,9} (half 1), f16 hi + lo
      const bool live = gq < NR;
      const int prow = live ? gq : 0;
      uint32_t ph[2][2], pl[2][2];
#pragma unroll
      for (int ks = 0; ks < 2; ++ks)
#pragma unroll
        for (int hf2 = 0; hf2 < 2; ++hf2) {
          const int t = 16 * ks + 2 * tq + 8 * hf2;
          float2 pp;
          if constexpr (TSC) {  // tokens 8 (2ks + hf2) + 2tq + {0, 1} of row gq: this lane's own P
            pp = make_float2(ptsc[TSC ? 2 * ks + hf2 : 0][0], ptsc[TSC ? 2 * ks + hf2 : 0][1]);
          } else {
            pp = *reinterpret_cast<const float2*>(&ws.P[WarpSmem<BITS, NR>::pidx(prow, t)]);
            if (!live) pp = make_float2(0.f, 0.f);
          }
          split2(pp.x, pp.y, ph[ks][hf2], pl[ks][hf2]);
        }
      // sum_t P z on the tensor cores: A rows g = z' hi, g + 8 = z' lo of group g (lanes gq < 4;
      // lanes gq >= 4 load group gq & 3 again and fill D rows 4-7 / 12-15, which are ignored)
      const uint4* vza = reinterpret_cast<const uint4*>(ws.sz + 32);
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const uint4 za = vza[ks * 16 + tq * 4 + ((gq & 3) ^ ((tq >> 1) << 1))];
        mma16816(zacc, za.x, za.y, za.z, za.w, ph[ks][0], ph[ks][1]);
        mma16816(zacc, za.x, za.y, za.z, za.w, pl[ks][0], pl[ks][1]);
      }
      const uint4* vsb = reinterpret_cast<const uint4*>(ws.sz);
#pragma unroll
      for (int gi = 0; gi < 4; ++gi)
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const uint4 sv = vsb[(gi * 2 + ks) * 4 + tq];
          mul_hilo(ph[ks][0], pl[ks][0], sv.x, sv.z, vb[gi][ks][0], vb[gi][ks][2]);
          mul_hilo(ph[ks][1], pl[ks][1], sv.y, sv.w, vb[gi][ks][1], vb[gi][ks][3]);
        }
    } else {
    {
      const int row = gq;
      const bool live = gq < NR;
      const int prow = row < NR ? row : 0;
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        float p[4], pv[4], p4[4];
#pragma unroll
        for (int slot = 0; slot < 4; ++slot) {
          const int khalf = slot >> 1;
          const int t = 16 * ks + 2 * tq + (slot & 1) + 8 * khalf;
          p[slot] = live ? ws.P[WarpSmem<BITS, NR>::pidx(prow, t)] : 0.f;
          pv[slot] = p[slot] * vscale[2 * ks + khalf];
          p4[slot] = 0.25f * p[slot];
        }
#pragma unroll
        for (int gi = 0; gi < 4; ++gi) {
          // (lo | hi) words of tokens 16ks + 2tq + {0,1,8,9} of group gi
          const uint4 vq = *reinterpret_cast<const uint4*>(S + SL::vp + 32 * gi + 8 * tq + 4 * ks);
          const uint32_t w4[4] = {vq.x, vq.y, vq.z, vq.w};
          float x[4];
#pragma unroll
          for (int slot = 0; slot < 4; ++slot) {
            const float lo = __uint_as_float(w4[slot] << 16), hi = __uint_as_float(w4[slot] & 0xFFFF0000u);
            const float dd = hi - lo;
            x[slot] = pv[slot] * dd;
            zacc[gi] = fmaf(p[slot], lo, zacc[gi]);                  // sum_t P * lo
            if (BITS == 1) zacc[gi] = fmaf(p4[slot], dd, zacc[gi]);  // + sum_t P * (hi - lo) / 4
          }
          split2(x[0], x[1], vb[gi][ks][0], vb[gi][ks][2]);
          split2(x[2], x[3], vb[gi][ks][1], vb[gi][ks][3]);
        }
      }
    }
    }
    // value codes of this lane
    uint32_t vw[4 * BITS];
    {
      const uint4 w0 = *reinterpret_cast<const uint4*>(S + SL::vc + lane * 4);
      vw[0] = w0.x;
      vw[1] = w0.y;
      vw[2] = w0.z;
      vw[3] = w0.w;
      if (BITS == 2) {
        const uint4 w1 = *reinterpret_cast<const uint4*>(S + SL::vc + 128 + lane * 4);
        vw[4 % (4 * BITS)] = w1.x;
        vw[5 % (4 * BITS)] = w1.y;
        vw[6 % (4 * BITS)] = w1.z;
        vw[7 % (4 * BITS)] = w1.w;
      }
    }
    __syncwarp();
    // the stage is consumed: refill it with block it + kSt (async proxy after generic reads)
    refill(next_src, st, blk + kSt * kWarps < blk1);

    // ---- P.V over 8 channel m-tiles x 2 token k-steps -------------------------------------
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        uint32_t a0, a1, a2, a3;
        const int q0 = 2 * ks, q1 = 2 * ks + 1;
        if (BITS == 2) {
          const uint32_t W = vw[mt % (4 * BITS)], W8 = W >> 8;
          const uint32_t m0 = (3u << (2 * q0)) | (3u << (16 + 2 * q0));
          const uint32_t m1 = (3u << (2 * q1)) | (3u << (16 + 2 * q1));
          a0 = W & m0;
          a1 = W8 & m0;
          a2 = W & m1;
          a3 = W8 & m1;
        } else {
          const uint32_t W = vw[(mt >> 1) % (4 * BITS)] >> (8 * (mt & 1)), W4 = W >> 4;
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
    }
    if (++st == kSt) {
      st = 0;
      phase ^= 1u;
    }
  }

  // ---- warp results -> shared, CTA merge -> partial ----------------------------------
  __syncwarp();
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < kSt; ++s)
      asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(smem_u32(&ws.bar[s])) : "memory");
  }
  if constexpr (TSC) {  // row gq's sum over its four tq lanes
    l_run[0] += __shfl_xor_sync(0xffffffffu, l_run[0], 1);
    l_run[0] += __shfl_xor_sync(0xffffffffu, l_run[0], 2);
  } else {
#pragma unroll
    for (int e = 0; e < RPL; ++e) l_run[e] = warp_sum_g(l_run[e]);
  }
  if (VCO) {  // z MMA: D rows gq (z' hi) + gq + 8 (z' lo) of group gq, lanes gq < 4
    zacc[0] += zacc[2 % (PG ? 1 : 4)];
    zacc[1] += zacc[3 % (PG ? 1 : 4)];
  } else {
#pragma unroll
    for (int i = 0; i < (PG ? 1 : 4); ++i) {  // z sums over the 4 lanes of a row group
      zacc[i] += __shfl_xor_sync(0xffffffffu, zacc[i], 1);
      zacc[i] += __shfl_xor_sync(0xffffffffu, zacc[i], 2);
    }
  }
  __syncthreads();
  MergeSmem<NR>& ms = *reinterpret_cast<MergeSmem<NR>*>(smem_raw);
  if (TSC) {
    if (tq == 0) {
      ms.m[warp][gq] = m_run[0];
      ms.l[warp][gq] = l_run[0];
    }
  } else if (gq == 0) {
#pragma unroll
    for (int e = 0; e < RPL; ++e) {
      if (jr[e] < NR) {
        ms.m[warp][jr[e]] = m_run[e];
        ms.l[warp][jr[e]] = l_run[e];
      }
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
      // VCO: lane (gq = gi, tq) holds group gi's z sums of rows 2tq, 2tq + 1 (scale 2^-Ez)
      const float z0 = VCO ? __shfl_sync(0xffffffffu, zacc[0], 4 * gi + tq) * z_out
                           : __shfl_sync(0xffffffffu, zacc[gi], 4 * (2 * tq));
      const float z1 = VCO ? __shfl_sync(0xffffffffu, zacc[1], 4 * gi + tq) * z_out
                           : __shfl_sync(0xffffffffu, zacc[gi], 4 * ((2 * tq + 1) & 7));
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
  // merge factors once per (warp, row), then one FFMA per warp and element
  if (threadIdx.x < NR) {
    const int j = threadIdx.x;
    float M = -CUDART_INF_F;
#pragma unroll
    for (int w = 0; w < kWarps; ++w)
      if (ms.l[w][j] > 0.f) M = fmaxf(M, ms.m[w][j]);
    float L = 0.f;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const float f = ms.l[w][j] > 0.f ? exp2f(ms.m[w][j] - M) : 0.f;
      ms.f[w][j] = f;
      L = fmaf(ms.l[w][j], f, L);
    }
    ms.M[j] = M;
    ms.L[j] = L;
  }
  __syncthreads();
  const size_t base = (((size_t)b * G.H + h) * (a.nsplit + 1) + split) * NR;
  for (int i = threadIdx.x; i < NR * 128; i += kThreads) {
    const int j = i >> 7, c = i & 127;
    float o = 0.f;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) o = fmaf(ms.o[w][j][c], ms.f[w][j], o);
    a.part_o[(base + j) * 128 + c] = o;
    if (c == 0) {
      a.part_ml[(base + j) * 2 + 0] = ms.M[j];
      a.part_ml[(base + j) * 2 + 1] = ms.L[j];
    }
  }
}

template <int BITS, int NR, int FOLD>
void launch_fast_f(const AttnArgs& a, cudaStream_t st) {
  constexpr size_t smem = fast_smem_bytes<BITS, NR>();
  // two CTAs per SM (228 KB, 1 KB reserved per CTA) is the design point
  static_assert(smem * kMinBlocks <= 227 * 1024, "K2 shared memory exceeds kMinBlocks CTAs/SM");
  static std::atomic<unsigned long long> done{0};  // one per <BITS, NR, FOLD> instantiation
  ensure_smem_attr(done, k_attend_fast<BITS, NR, FOLD>, (int)smem);
  dim3 grid = kExactOrder == 0 ? dim3(a.nsplit + 1, a.G.H, a.G.batch)
                                : dim3((a.nsplit + 1) * a.G.H * a.G.batch);
  k_attend_fast<BITS, NR, FOLD><<<grid, kThreads, smem, st>>>(a);
}

// The fold's code costs K2 0.7-1.5% even where it never runs (C2), so it is a
// separate instantiation, used when a warp walks more than kFoldMinBlocks blocks
template <int BITS, int NR>
void launch_fast_t(const AttnArgs& a, cudaStream_t st) {
  constexpr int F = NR * 4 <= 8 ? kFoldPG : kFold;
  if (F > 0 && a.blocks_per_split > kFoldMinBlocks * kWarps) launch_fast_f<BITS, NR, F>(a, st);
  else launch_fast_f<BITS, NR, 0>(a, st);
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
  // Split count: SPC_SPLIT_WAVES=w forces ~w waves; by default a wave model
  // picks it.  With `slots` = 2 CTAs x SMs resident, a launch of C CTAs (the
  // splits plus one exact CTA per unit) of b blocks costs about ceil(C / slots)
  // rounds of (b + c0) block-times, c0 ~ 40 blocks covering a CTA's prologue
  // (ring fill, first DRAM round trip) and merge.  Short CTAs pay c0 too often,
  // few CTAs quantize badly.  Measured sweeps (SPC_NSPLIT).
  static const int waves = [] {
    const char* e = getenv("SPC_SPLIT_WAVES");
    return e ? std::max(1, atoi(e)) : 0;
  }();
  static const int slots = [] {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return kMinBlocks * sms;
  }();
  static const int forced = [] {
    const char* e = getenv("SPC_NSPLIT");  // tuning only: exact split count (0 = model)
    return e ? std::max(0, atoi(e)) : 0;
  }();
  const int cap = std::min(127, std::max(1, nblk / 8));
  int want;
  if (forced) {
    want = std::min(forced, cap);
  } else if (waves) {
    want = std::max(1, std::min((waves * slots + units - 1) / units, cap));
  } else {
    // c0 = 40 since the transposed-score K2 (r3): C3 picks 17 splits instead of 22, +1.6% in
    // the 32-layer bench (profiles/r3_03_ab_k2_uniform.txt); C2 (7), C4 share (8), C1 (8) unchanged
    constexpr long long c0 = 40;
    auto cost_of = [&](int w, long long* rounds_out) {
      const int bps = std::max(1, (nblk + w - 1) / w), ns = std::max(1, (nblk + bps - 1) / bps);
      const long long rounds = ((long long)units * (ns + 1) + slots - 1) / slots;  // + the exact CTA
      if (rounds_out) *rounds_out = rounds;
      // a launch that needs a second round pays ~bps/10 more in the layer loop (its
      // later CTAs start behind the side kernels' CTAs): the C4 rank share's single
      // 8-split wave beats the model's 17-split two rounds by 10% in the bench
      // (profiles/r2_34_*), while C2 (7) and C3 (22) keep their picks
      return rounds * (bps + c0) + (rounds > 1 ? bps / 10 : 0);
    };
    long long best = -1, best_rounds = 1;
    want = 1;
    for (int w = 1; w <= cap; ++w) {
      long long rounds;
      const long long cost = cost_of(w, &rounds);
      if (best < 0 || cost < best) {
        best = cost;
        best_rounds = rounds;
        want = w;
      }
    }
    // MHA rows (one or two per kv head): of the multi-round picks within 3% of the model's
    // best, the fewest splits (longest CTAs).  C2: 7 -> 4, +0.9% in the 32-layer bench
    // (profiles/r3_03_ab_k2_uniform.txt); the model underprices these CTAs' fixed cost
    if (a.rows * G.G <= 2 && best_rounds > 1) {
      for (int w = 1; w < want; ++w) {
        long long rounds;
        const long long cost = cost_of(w, &rounds);
        if (rounds > 1 && cost * 100 <= best * 103) {
          want = w;
          break;
        }
      }
    }
    // A pick that fits in one round of long CTAs keeps ~15% of the slots free: in the layer
    // loop the side kernels (gather, aggregate, top-k) hold some, and a K2 CTA that has to
    // wait for one of them costs a whole second round.  C4 rank share: 8 -> 6 splits, +2.5%
    // in the 32-layer bench (profiles/r3_03_ab_k2_uniform.txt); multi-round picks unchanged.
    while (want > 1) {
      const int bps = std::max(1, (nblk + want - 1) / want), ns = std::max(1, (nblk + bps - 1) / bps);
      const long long ctas = (long long)units * (ns + 1);
      if (bps < 128 || ctas > slots || ctas * 100 <= (long long)slots * 85) break;
      --want;
    }
  }
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
