// common.cuh -- geometry, HBM layout and exact-arithmetic helpers shared by
// every kernel of the SpeCache decode path (sm_100a).
//
// HBM layout per (layer) -- blocks are [seq][kv head][block] records of G.rec
// words, one contiguous record per tb-token block so a block moves with a
// single bulk copy.  tb = g in the generic layout; the fast layout (d=128,
// bits 1|2) always uses 32-token records, and for g=64 each 64-token group
// spans two records that both carry its key params, while every 32-channel
// value slot carries the params of the 64-channel group containing it (the
// MMA kernel is then the same for g=32 and g=64).  Within a record (pointers
// kcodes/vcodes/kparams/vparams are the field bases, the block stride is G.rec
// for all four):
//   kcodes  uint32 [tb][krw]              key codes, token-major rows, LSB-first
//                                         channel order (a key group is a column
//                                         of the g/tb records of its group)
//   vcodes  uint32 [tb*vrw]               value codes; token-major rows in the
//                                         generic layout, MMA-fragment-native in
//                                         the fast layout (see vloc)
//   kparams uint32 [d]                    bf16 (lo | hi<<16) per key group (kpi)
//   vparams uint32 [tb*vps]               bf16 (lo | hi<<16) per value slot (vpi)
//   ring_k/v bf16  [b][H][r+g][d]         residual window, slot = pos % (r+g)
//   pool_k/v bf16  [b][U][k][Hu][d]       pinned full-precision rows (slots)
//   pin_pos int32  [b][U][k]              position held by each slot (-1 empty)
//   bitmap  uint32 [b][U][L/32]           1 = position pinned (masked in K2)
// 16-bit tier: kcodes/vcodes hold bf16 rows verbatim ([g][d] per block).
//
// Quantizer parameters are stored as the group's (min, max) in bf16.  Inputs
// are bf16, so min/max are exact and the reference's float64 (zero, scale)
// (quant.py:59-73) is reconstructed bit-exactly on device; the normative fp16
// (zero, scale) is a direct float64->fp16 rounding of those (quant.py:150-160).
#pragma once
#include <atomic>
#include <cuda_runtime.h>
// Threads per CTA of the side kernels that run beside K2 on the copy and
// selection streams (K3b aggregate, K5 PCIe gather).  128 with <= 32 registers
// fits in the 4096 registers two 120-register K2 CTAs leave free on an SM
// (SPC_K2_GQA_MAXREG=120), so they need not wait for a K2 CTA to retire.
#ifndef SPC_SIDE_THREADS
#define SPC_SIDE_THREADS 256
#endif
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace spc {
// Raise a kernel's dynamic shared-memory limit once per (kernel, device), thread
// safe: the attribute is per device, so a process-wide "done" flag would skip
// the second device (round-1 advisor finding), and setting it on every launch
// costs a driver call on the launch path.  `done` is the kernel's own bit mask.
template <typename F>
inline void ensure_smem_attr(std::atomic<unsigned long long>& done, F* kernel, int bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return;
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  done.fetch_or(bit, std::memory_order_acq_rel);
}
constexpr int kSideThreads = SPC_SIDE_THREADS;
// launch-bound occupancy hint that caps the side kernels at 32 registers when narrow
constexpr int kSideMinBlocks = kSideThreads <= 128 ? 16 : 1;

struct Geo {
  int layers, batch, H, Hq, d, bits, g, r, k, L, scope, host_layers;
  int G;      // q heads per kv head
  int U;      // top-k units per (seq, layer): 1 (layer scope) or H
  int Hu;     // kv heads per unit
  int nblk;   // block records per (seq, head): L / tb
  int ring;   // r + g
  int nch;    // value groups per token: ceil(d / g)
  int krw;    // uint32 words per key-code row
  int vrw;    // uint32 words per value-code row (generic) / per block = g*vrw
  int fast;   // fast MMA layout (d=128, g=32|64, bits 1|2)
  int tb;     // tokens per block record: g (generic) / 32 (fast)
  int vps;    // value param words per token in a record: nch (generic) / d/32 (fast)
  int bwords; // uint32 words of (key or value) codes per record = tb*krw
  int rec;    // uint32 words per block record [kcodes | vcodes | kparams | vparams]
};

struct LayerBufs {
  uint32_t* kcodes;
  uint32_t* vcodes;
  uint32_t* kparams;
  uint32_t* vparams;
  __nv_bfloat16* ring_k;
  __nv_bfloat16* ring_v;
  __nv_bfloat16* pool_k;
  __nv_bfloat16* pool_v;
  int32_t* pin_pos;
  uint32_t* bitmap;
  float* agg;          // [b][U][L]
  int32_t* sel;        // [b][U][k] ticket positions (ascending, -1 padded)
  int32_t* newcnt;     // [b][U]
  int32_t* fetch_slot; // [b][U][k]
  int32_t* fetch_pos;  // [b][U][k]
  uint32_t* rmax;      // [b][H][4] fp32 bits: max group range (hi-lo) of keys, of values; max |key|; max |value|
  unsigned long long* pf_rows;  // cache-wide count of prefetched (new) pin rows (profiling)
};

// ---- element offsets ---------------------------------------------------------
__host__ __device__ inline size_t blk_index(const Geo& G, int b, int h, int blk) {
  return ((size_t)b * G.H + h) * G.nblk + blk;
}

// ---- bf16 helpers --------------------------------------------------------------
__host__ __device__ inline float bf16_bits_to_float(uint32_t bits16) {
#ifdef __CUDA_ARCH__
  return __uint_as_float(bits16 << 16);
#else
  union { uint32_t u; float f; } v; v.u = bits16 << 16; return v.f;
#endif
}
__device__ inline uint32_t float_to_bf16_bits_exact(float x) {
  // caller guarantees x is bf16-representable (min/max of bf16 inputs)
  return __float_as_uint(x) >> 16;
}

// ---- exact reference arithmetic (quant.py:59-93), float64, no contraction ------
struct GroupParams {
  double zero, scale;
};
__device__ inline GroupParams params_from_minmax(double lo, double hi, int bits) {
  GroupParams p;
  if (bits == 1) {
    // x / 2^k == x * 2^-k bit for bit (one rounding of the same real value)
    p.zero = __dmul_rn(__dadd_rn(__dmul_rn(3.0, lo), hi), 0.25);
    p.scale = __dmul_rn(__dsub_rn(hi, lo), 0.5);
  } else {
    p.zero = lo;
    p.scale = __ddiv_rn(__dsub_rn(hi, lo), (double)((1 << bits) - 1));
  }
  return p;
}
__device__ inline GroupParams params_from_word(uint32_t w, int bits) {
  return params_from_minmax((double)bf16_bits_to_float(w & 0xFFFFu),
                            (double)bf16_bits_to_float(w >> 16), bits);
}
__device__ inline uint32_t quantize_code(float xf, GroupParams p, int bits) {
  if (p.scale == 0.0) return 0u;  // degenerate group (quant.py:79-80)
  double x = (double)xf;
  if (bits == 1) {  // threshold at zero + scale/2, boundary maps up (quant.py:81-84)
    return x >= __dadd_rn(p.zero, __dmul_rn(p.scale, 0.5)) ? 1u : 0u;
  }
  double c = rint(__ddiv_rn(__dsub_rn(x, p.zero), p.scale));  // half-even (quant.py:86)
  double top = (double)((1 << bits) - 1);
  c = c < 0.0 ? 0.0 : (c > top ? top : c);
  return (uint32_t)c;
}
__device__ inline float dequant_exact(uint32_t code, GroupParams p) {
  // float32(code * scale + zero), float64 multiply then add (quant.py:90-93)
  return __double2float_rn(__dadd_rn(__dmul_rn((double)code, p.scale), p.zero));
}

// float64 -> fp16 bits, single rounding (RN-even), like np.float16(float64).
__device__ inline uint16_t double_to_half_bits_rn(double x) {
  uint64_t u = (uint64_t)__double_as_longlong(x);
  uint16_t sign = (uint16_t)((u >> 48) & 0x8000u);
  uint64_t ax = u & 0x7FFFFFFFFFFFFFFFull;
  if (ax >= 0x7FF0000000000000ull)  // inf / nan
    return sign | (ax > 0x7FF0000000000000ull ? 0x7E00u : 0x7C00u);
  int e = (int)(ax >> 52) - 1023;
  uint64_t m = (ax & 0xFFFFFFFFFFFFFull) | (e > -1023 ? 0x10000000000000ull : 0);
  if (e > -1023) {
  } else {
    e = -1022;
  }
  // value = m * 2^(e-52).  half: normal if e >= -14 (mantissa 10 bits).
  int shift;  // bits to drop from m (53-bit significand) to get the half significand
  uint32_t hexp;
  if (e >= -14) {
    if (e > 15) return sign | 0x7C00u;
    shift = 42;                        // keep 11 bits (implicit + 10)
    hexp = (uint32_t)(e + 15);
  } else {
    shift = 42 + (-14 - e);            // subnormal: value / 2^-24
    hexp = 0;
    if (shift > 63) return sign;       // rounds to zero
  }
  uint64_t keep = m >> shift;
  uint64_t rem = m & ((1ull << shift) - 1);
  uint64_t half = 1ull << (shift - 1);
  if (rem > half || (rem == half && (keep & 1))) keep += 1;
  uint32_t out;
  if (hexp == 0) {
    out = (uint32_t)keep;               // may carry into the smallest normal: correct encoding
  } else {
    // keep has the implicit bit at position 10; a carry to 2^11 bumps the exponent
    if (keep >= (1ull << 11)) { keep >>= 1; hexp += 1; }
    if (hexp >= 31) return sign | 0x7C00u;
    out = (hexp << 10) | (uint32_t)(keep & 0x3FFu);
  }
  return sign | (uint16_t)out;
}

// ---- code locations ------------------------------------------------------------------
// Key codes: token-major row t of block, channel c at bit (c*B) of the row.
__host__ __device__ inline void kloc(const Geo& G, int t, int c, int* word, int* bit) {
  int pos = c * G.bits;
  *word = t * G.krw + (pos >> 5);
  *bit = pos & 31;
}
// Value codes.  Generic: same as keys.  Fast (d=128, g=32): MMA-fragment-native.
// The value MMA is D[ch][row] += A[ch][tok] * B[tok][row] (m16n8k16): m-tile mt
// covers channels 16mt..16mt+15, k-step ks tokens 16ks..16ks+15.  Lane L=4gq+tq
// holds a0=(ch gq, tok 2tq|2tq+1), a1=(ch gq+8, ..), a2=(ch gq, tok 2tq+8|+9),
// a3=(ch gq+8, ..); even token in the low f16 half, odd in the high half.  The
// lane's registers live contiguously so each lane loads its codes with one
// 16/32-byte read, and each register is produced by one AND (plus one shared
// shift) as an f16 subnormal code*2^(2q-24) (B=2) / code*2^(q-24) (B=1), q =
// 2ks + khalf -- a K-only scale folded into the B operand.
__host__ __device__ inline void vloc(const Geo& G, int t, int c, int* word, int* bit) {
  if (!G.fast) {
    kloc(G, t, c, word, bit);
    return;
  }
  int mt = c >> 4, mrow = c & 15, gq = mrow & 7, rh = mrow >> 3;
  int ks = t >> 4, kk = t & 15, khalf = kk >> 3, kr = kk & 7, tq = kr >> 1, odd = kr & 1;
  int lane = 4 * gq + tq, q = 2 * ks + khalf;
  if (G.bits == 2) {
    *word = (mt >> 2) * 128 + lane * 4 + (mt & 3);  // two 512-byte halves: 16 B per lane each
    *bit = 16 * odd + 2 * (4 * rh + q);
  } else {
    *word = lane * 4 + (mt >> 1);
    *bit = 16 * odd + (8 * (mt & 1) + 4 * rh + q);
  }
}

// Group-param word index within a block.  Generic: key c -> c, value (t, j) ->
// t*nch + j.  Fast layout: permuted so every lane of the MMA kernel reads its
// own params with 128-bit loads: key channel c = 32*tk + ks + 8*m is owned by
// lane 8*tk + ks (word 4*lane + m); value (token t, group j) sits at
// 32*j + 8*tq + 4*ks + slot with t = 16*ks + 2*tq + (slot & 1) + 8*(slot >> 1).
__host__ __device__ inline int kpi(const Geo& G, int c) {
  return G.fast ? (8 * (c >> 5) + (c & 7)) * 4 + ((c >> 3) & 3) : c;
}
__host__ __device__ inline int vpi(const Geo& G, int t, int j) {
  if (!G.fast) return t * G.nch + j;
  const int ks = t >> 4, khalf = (t >> 3) & 1, tq = (t >> 1) & 3, odd = t & 1;
  return 32 * j + 8 * tq + 4 * ks + 2 * khalf + odd;
}

// Value-param slot of channel c within a token's record words, and the first
// slot of value group j (the fast layout repeats a g=64 group's params in both
// of its 32-channel slots).
__host__ __device__ inline int vslot(const Geo& G, int c) { return G.fast ? (c >> 5) : c / G.g; }
__host__ __device__ inline int vslot_of_group(const Geo& G, int j) { return G.fast ? j * (G.g >> 5) : j; }

__device__ inline uint32_t read_code(const uint32_t* blk_words, int word, int bit, int bits) {
  return (blk_words[word] >> bit) & ((1u << bits) - 1u);
}

inline int ceil_div(int a, int b) { return (a + b - 1) / b; }

}  // namespace spc
