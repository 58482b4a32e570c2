// quant.cu -- K1: group quantizer + bit packing on device, and the two parity
// readers (normative export, exact materialize).
//
// Reference: quant.py:59-190 (params, codes, LSB-first packing, per-channel key
// groups, per-token value groups), kvcache.py:173-192 (migrate_residual),
// kvcache.py:222-243 (materialize), kvcache.py:270-281 (snapshot).
#include <math_constants.h>

#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace spc {

// One CTA quantizes one g-token group of one (seq, kv head) -- R = g/tb block
// records (R = 1 except the fast layout at g=64).  The group is staged in
// shared memory as fp32 (exact copies of the bf16 inputs), group (min, max)
// are reduced there, codes are computed in float64 exactly as the reference
// does and OR-ed into the records' packed words in shared memory, then the
// words stream out coalesced.
__global__ void __launch_bounds__(256) k_quantize(Geo G, LayerBufs B, QuantSrc S, int blk0) {
  const int blk = blk0 + blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int g = G.g, d = G.d, tid = threadIdx.x, nt = blockDim.x;
  const int R = g / G.tb, nw = R * G.bwords;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* sk = reinterpret_cast<float*>(smem_raw);            // [g][d]
  float* sv = sk + g * d;                                    // [g][d]
  uint32_t* wk = reinterpret_cast<uint32_t*>(sv + g * d);    // [R][tb*krw]
  uint32_t* wv = wk + nw;                                    // [R][tb*vrw]
  // float64 params start at the next 8-byte boundary after the code words
  double* kz = reinterpret_cast<double*>(smem_raw + ((sizeof(float) * 2 * g * d + sizeof(uint32_t) * 2 * nw + 7) & ~size_t(7)));  // [d]
  double* ks = kz + d;
  double* vz = ks + d;                                       // [g][nch]
  double* vs = vz + g * G.nch;

  for (int i = tid; i < g * d; i += nt) {
    int t = i / d, c = i - t * d;
    long long pos = (long long)blk * g + t;
    long long row = S.ring ? pos % S.ring : pos;
    long long off = b * S.seq_stride + row * S.tok_stride + (long long)h * S.head_stride + c;
    sk[i] = __bfloat162float(S.k[off]);
    sv[i] = __bfloat162float(S.v[off]);
  }
  __syncthreads();
  const size_t bi = blk_index(G, b, h, blk * R);  // first record of the group

  if (G.bits == 16) {  // verbatim full-precision tier (kvcache.py:185-187)
    __nv_bfloat16* okc = reinterpret_cast<__nv_bfloat16*>(B.kcodes + bi * (size_t)G.rec);
    __nv_bfloat16* ovc = reinterpret_cast<__nv_bfloat16*>(B.vcodes + bi * (size_t)G.rec);
    for (int i = tid; i < g * d; i += nt) {
      okc[i] = __float2bfloat16_rn(sk[i]);
      ovc[i] = __float2bfloat16_rn(sv[i]);
    }
    return;
  }

  __shared__ float s_rk, s_rv, s_av, s_ak;
  if (tid == 0) {
    s_rk = 0.f;
    s_rv = 0.f;
    s_av = 0.f;
    s_ak = 0.f;
  }
  __syncthreads();
  // key groups: one per channel over the block's tokens (quant.py:163-169)
  for (int c = tid; c < d; c += nt) {
    float lo = sk[c], hi = sk[c];
    for (int t = 1; t < g; ++t) {
      float x = sk[t * d + c];
      lo = fminf(lo, x);
      hi = fmaxf(hi, x);
    }
    const uint32_t pw = float_to_bf16_bits_exact(lo) | (float_to_bf16_bits_exact(hi) << 16);
    for (int r = 0; r < R; ++r) B.kparams[(bi + r) * G.rec + kpi(G, c)] = pw;  // every record of the group
    atomicMax(reinterpret_cast<unsigned*>(&s_rk), __float_as_uint(hi - lo));
    atomicMax(reinterpret_cast<unsigned*>(&s_ak), __float_as_uint(fmaxf(fabsf(lo), fabsf(hi))));
    GroupParams p = params_from_minmax((double)lo, (double)hi, G.bits);
    kz[c] = p.zero;
    ks[c] = p.scale;
  }
  // value groups: per token, chunks of g channels, last may be ragged (quant.py:177-186)
  for (int i = tid; i < g * G.nch; i += nt) {
    int t = i / G.nch, j = i - t * G.nch;
    int c0 = j * g, c1 = min(d, c0 + g);
    float lo = sv[t * d + c0], hi = lo;
    for (int c = c0 + 1; c < c1; ++c) {
      float x = sv[t * d + c];
      lo = fminf(lo, x);
      hi = fmaxf(hi, x);
    }
    const uint32_t pw = float_to_bf16_bits_exact(lo) | (float_to_bf16_bits_exact(hi) << 16);
    const int r = t / G.tb, tt = t - r * G.tb, s0 = vslot_of_group(G, j), s1 = vslot_of_group(G, j + 1);
    for (int sl = s0; sl < s1 && sl < G.vps; ++sl) B.vparams[(bi + r) * (size_t)G.rec + vpi(G, tt, sl)] = pw;
    atomicMax(reinterpret_cast<unsigned*>(&s_rv), __float_as_uint(hi - lo));
    atomicMax(reinterpret_cast<unsigned*>(&s_av), __float_as_uint(fmaxf(fabsf(lo), fabsf(hi))));
    GroupParams p = params_from_minmax((double)lo, (double)hi, G.bits);
    vz[i] = p.zero;
    vs[i] = p.scale;
  }
  for (int i = tid; i < nw; i += nt) {
    wk[i] = 0u;
    wv[i] = 0u;
  }
  __syncthreads();
  if (tid == 0) {  // per-(seq, head) range maxima: exponent choice of the MMA path
    atomicMax(&B.rmax[((size_t)b * G.H + h) * 4 + 0], __float_as_uint(s_rk));
    atomicMax(&B.rmax[((size_t)b * G.H + h) * 4 + 1], __float_as_uint(s_rv));
    atomicMax(&B.rmax[((size_t)b * G.H + h) * 4 + 3], __float_as_uint(s_av));
    atomicMax(&B.rmax[((size_t)b * G.H + h) * 4 + 2], __float_as_uint(s_ak));
  }
  for (int i = tid; i < g * d; i += nt) {
    int t = i / d, c = i - t * d, w, bit;
    const int r = t / G.tb, tt = t - r * G.tb;
    GroupParams pk{kz[c], ks[c]};
    uint32_t ck = quantize_code(sk[i], pk, G.bits);
    kloc(G, tt, c, &w, &bit);
    if (ck) atomicOr(&wk[r * G.bwords + w], ck << bit);
    int j = c / g;
    GroupParams pv{vz[t * G.nch + j], vs[t * G.nch + j]};
    uint32_t cv = quantize_code(sv[i], pv, G.bits);
    vloc(G, tt, c, &w, &bit);
    if (cv) atomicOr(&wv[r * G.bwords + w], cv << bit);
  }
  __syncthreads();
  for (int r = 0; r < R; ++r) {
    uint32_t* okc = B.kcodes + (bi + r) * (size_t)G.rec;
    uint32_t* ovc = B.vcodes + (bi + r) * (size_t)G.rec;
    for (int i = tid; i < G.bwords; i += nt) {
      okc[i] = wk[r * G.bwords + i];
      ovc[i] = wv[r * G.bwords + i];
    }
  }
}

// Fast-layout quantizer (d = 128, g = 32, 1 or 2 bits): one CTA per g-token
// block of one (seq, kv head), 256 threads, and every output word built in
// registers by the thread that owns it -- no shared-memory atomics.
//  * rows are staged with 16-byte loads into padded fp32 tiles;
//  * threads 0..127 reduce a key group (one channel over the 32 tokens),
//    threads 128..255 a value group (32 channels of one token);
//  * codes: 1-bit is x >= thr where thr is the smallest fp32 >= the reference's
//    float64 threshold zero + scale/2 (quant.py:81-84), so the fp32 compare is
//    exact.  2-bit evaluates q ~= (x - z) / s in fp32 (error < 1.2e-6 on [0, 3])
//    and takes rint/clip from it unless q lies within 1e-5 of a rounding
//    boundary 0.5 / 1.5 / 2.5; those few elements (and degenerate scales) go
//    through the reference's float64 division (quantize_code) -- bit-exact
//    codes at fp32 cost.
//  * key words are token-major rows (kloc), value words the MMA-fragment
//    permutation (vloc), inverted here so each thread knows which (t, c) each
//    of its word's bit fields holds.
template <int BITS>
__global__ void __launch_bounds__(256) k_quantize_fast(Geo G, LayerBufs B, QuantSrc S, int blk0) {
  // tile rows padded so both code-word passes read shared memory conflict-free:
  // key words (lanes = 4 tokens x 8 channel runs, rotated start) want LD = 1 mod 32,
  // value words (lanes = tokens 2tq.. x channels gq) want LD = 4 mod 32
  constexpr int g = 32, d = 128, LDK = 129, LDV = 132;
  const int blk = blk0 + blockIdx.x, h = blockIdx.y, b = blockIdx.z, tid = threadIdx.x;
  __shared__ float xk[g * LDK];
  __shared__ float xv[g * LDV];
  __shared__ float kz[d], krs[d], kthr[d];     // key groups (fp32 fast-path data)
  __shared__ double kz64[d], ks64[d];
  __shared__ float vz[g * 4], vrs[g * 4], vthr[g * 4];
  __shared__ double vz64[g * 4], vs64[g * 4];
  __shared__ float s_rk, s_rv, s_av, s_ak;
  // ---- stage: 32 rows x 16 chunks of 16 bytes, for K and V
  for (int i = tid; i < g * 16; i += 256) {
    const int t = i >> 4, ch = i & 15;
    const long long pos = (long long)blk * g + t;
    const long long row = S.ring ? pos % S.ring : pos;
    const long long off = b * S.seq_stride + row * S.tok_stride + (long long)h * S.head_stride + ch * 8;
    const uint4 wk = *reinterpret_cast<const uint4*>(S.k + off);
    const uint4 wv = *reinterpret_cast<const uint4*>(S.v + off);
    const uint32_t ak[4] = {wk.x, wk.y, wk.z, wk.w}, av[4] = {wv.x, wv.y, wv.z, wv.w};
    float* dk = xk + t * LDK + ch * 8;
    float* dv = xv + t * LDV + ch * 8;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      dk[2 * e] = __uint_as_float(ak[e] << 16);
      dk[2 * e + 1] = __uint_as_float(ak[e] & 0xFFFF0000u);
      dv[2 * e] = __uint_as_float(av[e] << 16);
      dv[2 * e + 1] = __uint_as_float(av[e] & 0xFFFF0000u);
    }
  }
  if (tid == 0) {
    s_rk = 0.f;
    s_rv = 0.f;
    s_av = 0.f;
    s_ak = 0.f;
  }
  __syncthreads();
  const size_t bi = blk_index(G, b, h, blk);
  // ---- group parameters
  {
    float lo, hi;
    int gidx;
    const bool key = tid < 128;
    if (key) {  // key group: channel c over the block's tokens (quant.py:163-169)
      const int c = tid;
      lo = hi = xk[c];
      for (int t = 1; t < g; ++t) {
        const float x = xk[t * LDK + c];
        lo = fminf(lo, x);
        hi = fmaxf(hi, x);
      }
      B.kparams[bi * G.rec + kpi(G, c)] = float_to_bf16_bits_exact(lo) | (float_to_bf16_bits_exact(hi) << 16);
      atomicMax(reinterpret_cast<unsigned*>(&s_rk), __float_as_uint(hi - lo));
      atomicMax(reinterpret_cast<unsigned*>(&s_ak), __float_as_uint(fmaxf(fabsf(lo), fabsf(hi))));
      gidx = c;
    } else {    // value group: 32 channels of token t (quant.py:177-186); rotated reads spread banks
      const int i = tid - 128, t = i >> 2, j = i & 3;
      const float* r = xv + t * LDV + 32 * j;
      lo = hi = r[j];
      for (int k = 1; k < 32; ++k) {
        const float x = r[(k + j) & 31];
        lo = fminf(lo, x);
        hi = fmaxf(hi, x);
      }
      B.vparams[bi * (size_t)G.rec + vpi(G, t, j)] =
          float_to_bf16_bits_exact(lo) | (float_to_bf16_bits_exact(hi) << 16);
      atomicMax(reinterpret_cast<unsigned*>(&s_rv), __float_as_uint(hi - lo));
      atomicMax(reinterpret_cast<unsigned*>(&s_av), __float_as_uint(fmaxf(fabsf(lo), fabsf(hi))));
      gidx = i;
    }
    const GroupParams p = params_from_minmax((double)lo, (double)hi, BITS);
    float thr = CUDART_INF_F, rs = 0.f, zf = 0.f;
    if (p.scale != 0.0) {
      if (BITS == 1) {
        thr = __double2float_ru(__dadd_rn(p.zero, __dmul_rn(p.scale, 0.5)));
      } else {
        zf = (float)p.zero;  // = lo, exact
        // fast code only: |error| << the 1e-5 boundary margin; an fp32-subnormal
        // scale gives NaN, i.e. the float64 path for every code of the group
        rs = (float)p.scale >= 1.17549435e-38f ? __frcp_rn((float)p.scale) : __int_as_float(0x7fc00000);
      }
    }
    if (key) {
      kz[gidx] = zf; krs[gidx] = rs; kthr[gidx] = thr; kz64[gidx] = p.zero; ks64[gidx] = p.scale;
    } else {
      vz[gidx] = zf; vrs[gidx] = rs; vthr[gidx] = thr; vz64[gidx] = p.zero; vs64[gidx] = p.scale;
    }
  }
  __syncthreads();
  if (tid == 0) {  // per-(seq, head) range maxima: exponent choice of the MMA path
    atomicMax(&B.rmax[((size_t)b * G.H + h) * 4 + 0], __float_as_uint(s_rk));
    atomicMax(&B.rmax[((size_t)b * G.H + h) * 4 + 1], __float_as_uint(s_rv));
    atomicMax(&B.rmax[((size_t)b * G.H + h) * 4 + 3], __float_as_uint(s_av));
    atomicMax(&B.rmax[((size_t)b * G.H + h) * 4 + 2], __float_as_uint(s_ak));
  }
  // Fast code of element x in its group: 1-bit x >= thr; 2-bit rint via the
  // 1.5*2^23 magic add (round-to-nearest-even, as rint) clipped to 3.  `near`
  // flags q within 1e-5 of a rounding boundary (or a non-finite q); those
  // elements alone are redone in float64 (quantize_code) after the word's
  // fast pass -- a short divergent loop, usually one element.  Degenerate groups have
  // rs = 0 -> q = 0 -> code 0 and thr = +inf (quant.py:79-80).
  auto fast_code = [&](float x, float z, float rs, float thr, bool& near) -> uint32_t {
    if (BITS == 1) return x >= thr ? 1u : 0u;
    const float dq = (x - z) * rs;
    const float y = dq + 12582912.0f;                  // 1.5 * 2^23: rint(dq) in the low mantissa bits
    const float r = y - 12582912.0f;                   // rint(dq), exact for 0 <= dq < 2^22
    near = fabsf(fabsf(dq - r) - 0.5f) < 1e-5f || !(dq < 4194304.f);
    const uint32_t c = __float_as_uint(y) & 0x3FFFFFu;
    return c < 3u ? c : 3u;
  };
  constexpr int KW = g * 4 * BITS;  // key (and value) code words per block: 256 (2-bit) / 128 (1-bit)
  constexpr int PER = 32 / BITS;    // codes per word
  uint32_t* okc = B.kcodes + bi * (size_t)G.rec;
  uint32_t* ovc = B.vcodes + bi * (size_t)G.rec;
  for (int w = tid; w < KW; w += 256) {
    // key word: token t, channels c0 .. c0 + PER - 1, LSB first (kloc); start rotated by the run index
    {
      const int t = w / (4 * BITS), run = w % (4 * BITS), c0 = run * PER, rot = (2 * run) % PER;
      uint32_t word = 0, nmask = 0;
#pragma unroll
      for (int jj = 0; jj < PER; ++jj) {
        const int j = (jj + rot) % PER, c = c0 + j;
        bool near;
        word |= fast_code(xk[t * LDK + c], kz[c], krs[c], kthr[c], near) << (BITS * j);
        if (BITS == 2) nmask |= (uint32_t)near << j;
      }
      while (BITS == 2 && nmask) {  // rare: exact float64 code of each boundary element
        const int j = __ffs(nmask) - 1, c = c0 + j;
        nmask &= nmask - 1u;
        const uint32_t cd = quantize_code(xk[t * LDK + c], GroupParams{kz64[c], ks64[c]}, 2);
        word = (word & ~(3u << (2 * j))) | (cd << (2 * j));
      }
      okc[w] = word;
    }
    // value word: inverse of vloc (common.cuh)
    {
      int mt_base, lane;
      if (BITS == 2) {
        mt_base = 4 * (w >> 7) + (w & 3);
        lane = (w >> 2) & 31;
      } else {
        mt_base = 2 * (w & 3);
        lane = w >> 2;
      }
      const int gq = lane >> 2, tq = lane & 3;
      auto tc = [&](int j, int& t, int& c) {
        const int bit = BITS * j, odd = bit >> 4, r = (bit & 15) / BITS;
        const int mt = BITS == 2 ? mt_base : mt_base + (r >> 3);
        const int rh = BITS == 2 ? (r >> 2) : ((r >> 2) & 1);
        const int q = r & 3;
        c = 16 * mt + 8 * rh + gq;
        t = 16 * (q >> 1) + 8 * (q & 1) + 2 * tq + odd;
      };
      uint32_t word = 0, nmask = 0;
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        int t, c;
        tc(j, t, c);
        const int gi = t * 4 + (c >> 5);
        bool near;
        word |= fast_code(xv[t * LDV + c], vz[gi], vrs[gi], vthr[gi], near) << (BITS * j);
        if (BITS == 2) nmask |= (uint32_t)near << j;
      }
      while (BITS == 2 && nmask) {
        const int j = __ffs(nmask) - 1;
        nmask &= nmask - 1u;
        int t, c;
        tc(j, t, c);
        const int gi = t * 4 + (c >> 5);
        const uint32_t cd = quantize_code(xv[t * LDV + c], GroupParams{vz64[gi], vs64[gi]}, 2);
        word = (word & ~(3u << (2 * j))) | (cd << (2 * j));
      }
      ovc[w] = word;
    }
  }
}

// K1 v2 (round 2): the same bit-exact codes and layout as k_quantize_fast with
// about half the instructions (ncu r1: 8.9k warp-instructions per block, 76%
// issue-active; three shared-memory loads and the inverted (t, c) index math
// per element were the bulk, the 4-way bank conflicts of the fp32 staging a
// symptom).
//  * rows are staged as raw bf16 with 16-byte stores (272-byte rows:
//    conflict-free), not converted to fp32;
//  * group (min, max) and the float64 parameters as before;
//  * codes elementwise: thread (c = tid & 127) keeps its key channel's
//    parameters in registers and walks 16 tokens; value parameters are
//    warp-uniform broadcasts; one byte per code into shared memory (key codes
//    [t][c], value codes [c][t] with 36-byte rows, both conflict-free);
//  * words from bytes: a key word is one 16-byte (2-bit) / 2 x 16-byte (1-bit)
//    load and a shift/mask gather; a value word reads its 8 / 16 (token pair)
//    16-bit code pairs of the MMA-fragment layout (vloc).
template <int BITS>
__global__ void __launch_bounds__(256) k_quantize_fast2(Geo G, LayerBufs B, QuantSrc S, int blk0) {
  constexpr int g = 32, d = 128, LD = 136;  // bf16 tile rows: 272 B = 68 words
  const int blk = blk0 + blockIdx.x, h = blockIdx.y, b = blockIdx.z, tid = threadIdx.x;
  __shared__ __align__(16) uint16_t tk[g * LD];
  __shared__ __align__(16) uint16_t tv[g * LD];
  __shared__ __align__(16) uint8_t ck[g * d];   // key codes [t][c]
  // value codes [c][t], 42-byte rows: conflict-free for both the code stores
  // (lanes: channels 2l, token t) and the packing loads (the fragment order's
  // (mt, gq, tq) lanes); 34-byte rows left the packing loads 2-way
  constexpr int CVS = 42;
  __shared__ __align__(16) uint8_t cv[d * CVS];
  __shared__ float kz[d], krs[d], kthr[d];
  __shared__ double kz64[d], ks64[d];
  __shared__ float vz[g * 4], vrs[g * 4], vthr[g * 4];
  __shared__ double vz64[g * 4], vs64[g * 4];
  __shared__ float s_rk, s_rv, s_av, s_ak;
  auto bf = [](uint16_t u) { return __uint_as_float((uint32_t)u << 16); };
  // ---- stage: 32 rows x 16 chunks of 16 bytes, for K and V (raw bf16)
  for (int i = tid; i < g * 16; i += 256) {
    const int t = i >> 4, ch = i & 15;
    const long long pos = (long long)blk * g + t;
    const long long row = S.ring ? pos % S.ring : pos;
    const long long off = b * S.seq_stride + row * S.tok_stride + (long long)h * S.head_stride + ch * 8;
    *reinterpret_cast<uint4*>(tk + t * LD + ch * 8) = *reinterpret_cast<const uint4*>(S.k + off);
    *reinterpret_cast<uint4*>(tv + t * LD + ch * 8) = *reinterpret_cast<const uint4*>(S.v + off);
  }
  if (tid == 0) {
    s_rk = 0.f;
    s_rv = 0.f;
    s_av = 0.f;
    s_ak = 0.f;
  }
  __syncthreads();
  const size_t bi = blk_index(G, b, h, blk);
  // ---- group parameters (quant.py:59-73 via :163-186): threads 0-127 a key
  // group (channel c over the 32 tokens), threads 128-255 a value group
  {
    float lo, hi;
    int gidx;
    const bool key = tid < 128;
    if (key) {
      const int c = tid;
      lo = hi = bf(tk[c]);
#pragma unroll 8
      for (int t = 1; t < g; ++t) {
        const float x = bf(tk[t * LD + c]);
        lo = fminf(lo, x);
        hi = fmaxf(hi, x);
      }
      B.kparams[bi * G.rec + kpi(G, c)] = float_to_bf16_bits_exact(lo) | (float_to_bf16_bits_exact(hi) << 16);
      atomicMax(reinterpret_cast<unsigned*>(&s_rk), __float_as_uint(hi - lo));
      atomicMax(reinterpret_cast<unsigned*>(&s_ak), __float_as_uint(fmaxf(fabsf(lo), fabsf(hi))));
      gidx = c;
    } else {  // 32 channels of token t, rotated start (a 2j rotation is conflict-free
      // but costs 2% more instructions than the 2-way conflicts it removes)
      const int i = tid - 128, t = i >> 2, j = i & 3;
      const uint16_t* r = tv + t * LD + 32 * j;
      lo = hi = bf(r[j]);
#pragma unroll 8
      for (int k = 1; k < 32; ++k) {
        const float x = bf(r[(k + j) & 31]);
        lo = fminf(lo, x);
        hi = fmaxf(hi, x);
      }
      B.vparams[bi * (size_t)G.rec + vpi(G, t, j)] =
          float_to_bf16_bits_exact(lo) | (float_to_bf16_bits_exact(hi) << 16);
      atomicMax(reinterpret_cast<unsigned*>(&s_rv), __float_as_uint(hi - lo));
      atomicMax(reinterpret_cast<unsigned*>(&s_av), __float_as_uint(fmaxf(fabsf(lo), fabsf(hi))));
      gidx = i;
    }
    const GroupParams p = params_from_minmax((double)lo, (double)hi, BITS);
    float thr = CUDART_INF_F, rs = 0.f, zf = 0.f;
    if (p.scale != 0.0) {
      if (BITS == 1) {
        thr = __double2float_ru(__dadd_rn(p.zero, __dmul_rn(p.scale, 0.5)));
      } else {
        zf = (float)p.zero;  // = lo, exact
        // fast code only: |error| << the 1e-5 boundary margin; an fp32-subnormal
        // scale gives NaN, i.e. the float64 path for every code of the group
        rs = (float)p.scale >= 1.17549435e-38f ? __frcp_rn((float)p.scale) : __int_as_float(0x7fc00000);
      }
    }
    if (key) {
      kz[gidx] = zf; krs[gidx] = rs; kthr[gidx] = thr; kz64[gidx] = p.zero; ks64[gidx] = p.scale;
    } else {
      vz[gidx] = zf; vrs[gidx] = rs; vthr[gidx] = thr; vz64[gidx] = p.zero; vs64[gidx] = p.scale;
    }
  }
  __syncthreads();
  if (tid == 0) {  // per-(seq, head) range maxima: exponent choice of the MMA path
    atomicMax(&B.rmax[((size_t)b * G.H + h) * 4 + 0], __float_as_uint(s_rk));
    atomicMax(&B.rmax[((size_t)b * G.H + h) * 4 + 1], __float_as_uint(s_rv));
    atomicMax(&B.rmax[((size_t)b * G.H + h) * 4 + 3], __float_as_uint(s_av));
    atomicMax(&B.rmax[((size_t)b * G.H + h) * 4 + 2], __float_as_uint(s_ak));
  }
  // fast code: see k_quantize_fast (1-bit: x >= thr exact; 2-bit: fp32 rint with a
  // float64 redo within 1e-5 of a rounding boundary)
  // In-group values give q = (x - z) / s in [0, 3], so "within 1e-5 of a .5
  // boundary" is |q - rint(q)| > 0.5 - 1e-5; written as !(<=) so that a NaN or
  // infinite q (1/s overflowing fp32 for subnormal-range scales) also takes the
  // float64 path.
  auto fast_code = [&](float x, float z, float rs, float thr, bool& near) -> uint32_t {
    if (BITS == 1) return x >= thr ? 1u : 0u;
    const float dq = (x - z) * rs;
    const float y = dq + 12582912.0f;
    near = !(fabsf(dq - (y - 12582912.0f)) <= 0.49999f);
    return min(__float_as_uint(y) & 0x3FFFFFu, 3u);
  };
  // ---- codes, one byte each, channel pairs (32-bit loads); the rare float64
  // redo is taken once per warp
  {
    const int c = 2 * (tid & 63), t0 = tid >> 6, j = c >> 5;
    const float z0 = kz[c], rs0 = krs[c], thr0 = kthr[c], z1 = kz[c + 1], rs1 = krs[c + 1], thr1 = kthr[c + 1];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int t = t0 + 4 * k;
      const int gi = t * 4 + j;
      const uint32_t uk = *reinterpret_cast<const uint32_t*>(tk + t * LD + c);
      const uint32_t uv = *reinterpret_cast<const uint32_t*>(tv + t * LD + c);
      const float xk0 = __uint_as_float(uk << 16), xk1 = __uint_as_float(uk & 0xFFFF0000u);
      const float xv0 = __uint_as_float(uv << 16), xv1 = __uint_as_float(uv & 0xFFFF0000u);
      const float vzz = vz[gi], vrr = vrs[gi], vth = vthr[gi];
      bool n0 = false, n1 = false, n2 = false, n3 = false;
      uint32_t k0 = fast_code(xk0, z0, rs0, thr0, n0), k1 = fast_code(xk1, z1, rs1, thr1, n1);
      uint32_t v0 = fast_code(xv0, vzz, vrr, vth, n2), v1 = fast_code(xv1, vzz, vrr, vth, n3);
      if (BITS == 2 && __any_sync(0xffffffffu, n0 || n1 || n2 || n3)) {
        if (n0) k0 = quantize_code(xk0, GroupParams{kz64[c], ks64[c]}, 2);
        if (n1) k1 = quantize_code(xk1, GroupParams{kz64[c + 1], ks64[c + 1]}, 2);
        if (n2) v0 = quantize_code(xv0, GroupParams{vz64[gi], vs64[gi]}, 2);
        if (n3) v1 = quantize_code(xv1, GroupParams{vz64[gi], vs64[gi]}, 2);
      }
      *reinterpret_cast<uint16_t*>(ck + t * d + c) = (uint16_t)(k0 | (k1 << 8));
      cv[c * CVS + t] = (uint8_t)v0;
      cv[(c + 1) * CVS + t] = (uint8_t)v1;
    }
  }
  __syncthreads();
  // ---- words
  constexpr int KW = g * 4 * BITS;  // key (and value) code words per block: 256 (2-bit) / 128 (1-bit)
  uint32_t* okc = B.kcodes + bi * (size_t)G.rec;
  uint32_t* ovc = B.vcodes + bi * (size_t)G.rec;
  for (int w = tid; w < KW; w += 256) {
    {  // key word: token t, channels c0.. (kloc: LSB-first)
      const int t = w / (4 * BITS), c0 = (w % (4 * BITS)) * (32 / BITS);
      uint32_t word = 0;
      if (BITS == 2) {
        const uint4 q = *reinterpret_cast<const uint4*>(ck + t * d + c0);
        const uint32_t qq[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          uint32_t x = qq[e];
          x = (x | (x >> 6)) & 0x000F000Fu;
          x = (x | (x >> 12)) & 0xFFu;
          word |= x << (8 * e);
        }
      } else {
        const uint4 q0 = *reinterpret_cast<const uint4*>(ck + t * d + c0);
        const uint4 q1 = *reinterpret_cast<const uint4*>(ck + t * d + c0 + 16);
        const uint32_t qq[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          uint32_t x = qq[e];
          x = x | (x >> 7);
          x = (x | (x >> 14)) & 0xFu;
          word |= x << (4 * e);
        }
      }
      okc[w] = word;
    }
    {  // value word: inverse of vloc (common.cuh), code pairs (odd = 0, 1) per 16-bit load
      int mt_base, lane;
      if (BITS == 2) {
        mt_base = 4 * (w >> 7) + (w & 3);
        lane = (w >> 2) & 31;
      } else {
        mt_base = 2 * (w & 3);
        lane = w >> 2;
      }
      const int gq = lane >> 2, tq = lane & 3;
      uint32_t word = 0;
      constexpr int NR = BITS == 2 ? 8 : 16;  // (rh, q) [+ mt step] fields per half word
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const int mt = BITS == 2 ? mt_base : mt_base + (r >> 3);
        const int rh = BITS == 2 ? (r >> 2) : ((r >> 2) & 1);
        const int q = r & 3;
        const int c = 16 * mt + 8 * rh + gq;
        const int t = 16 * (q >> 1) + 8 * (q & 1) + 2 * tq;
        const uint32_t x = *reinterpret_cast<const uint16_t*>(cv + c * CVS + t);
        const uint32_t m = BITS == 2 ? 3u : 1u;
        word |= ((x & m) << (BITS * r)) | (((x >> 8) & m) << (16 + BITS * r));
      }
      ovc[w] = word;
    }
  }
}

size_t quantize_smem_bytes(const Geo& G) {
  size_t s = 2 * sizeof(float) * G.g * G.d;
  s += sizeof(uint32_t) * (2 * (G.g / G.tb) * G.bwords);
  s = (s + 7) & ~size_t(7);
  s += sizeof(double) * (2 * G.d + 2 * G.g * G.nch);
  return s;
}

void launch_quantize(const Geo& G, const LayerBufs& B, const QuantSrc& S, int blk0, int nblocks,
                     cudaStream_t st) {
  if (nblocks <= 0) return;
  static std::atomic<unsigned long long> done{0};
  ensure_smem_attr(done, k_quantize, 200 * 1024);
  dim3 grid(nblocks, G.H, G.batch);
  if (G.fast && G.d == 128 && G.g == 32 && (G.bits == 1 || G.bits == 2)) {
    static const bool v1 = [] {  // SPC_K1_V1=1: the round-1 kernel (A/B)
      const char* e = getenv("SPC_K1_V1");
      return e && atoi(e) != 0;
    }();
    if (v1) {
      if (G.bits == 2) k_quantize_fast<2><<<grid, 256, 0, st>>>(G, B, S, blk0);
      else k_quantize_fast<1><<<grid, 256, 0, st>>>(G, B, S, blk0);
    } else {
      if (G.bits == 2) k_quantize_fast2<2><<<grid, 256, 0, st>>>(G, B, S, blk0);
      else k_quantize_fast2<1><<<grid, 256, 0, st>>>(G, B, S, blk0);
    }
    return;
  }
  k_quantize<<<grid, 256, quantize_smem_bytes(G), st>>>(G, B, S, blk0);
}

// ---------------------------------------------------------------------------------
// Normative export of one (layer, seq): the arrays TwoTierCache.snapshot() would
// serialise (kvcache.py:270-281), codes LSB-first per group (quant.py:96-109),
// fp16 zero/scale as a direct float64 -> fp16 rounding (quant.py:150-160).
__global__ void k_export(Geo G, LayerBufs B, int seq, int nblocks, uint8_t* kcodes,
                         uint16_t* kzero, uint16_t* kscale, uint8_t* vcodes, uint16_t* vzero,
                         uint16_t* vscale) {
  const int blk = blockIdx.x, h = blockIdx.y, tid = threadIdx.x;   // blk: g-token group
  const int g = G.g, d = G.d, bits = G.bits, nb = (g * bits + 7) / 8;
  const int R = g / G.tb;
  const size_t bi = blk_index(G, seq, h, blk * R);   // the group's first record
  // token t of the group: record t / tb, row t % tb
  auto kw_of = [&](int t) { return B.kcodes + (bi + t / G.tb) * (size_t)G.rec; };
  auto vw_of = [&](int t) { return B.vcodes + (bi + t / G.tb) * (size_t)G.rec; };
  const int per = 8 / bits;
  // key groups [nblocks][H][d][nb]
  for (int i = tid; i < d * nb; i += blockDim.x) {
    int c = i / nb, byte = i - c * nb;
    uint32_t v = 0;
    for (int j = 0; j < per; ++j) {
      int t = byte * per + j;
      if (t >= g) break;
      int w, bit;
      kloc(G, t % G.tb, c, &w, &bit);
      v |= read_code(kw_of(t), w, bit, bits) << (j * bits);
    }
    kcodes[(((size_t)blk * G.H + h) * d + c) * nb + byte] = (uint8_t)v;
  }
  for (int c = tid; c < d; c += blockDim.x) {
    GroupParams p = params_from_word(B.kparams[bi * G.rec + kpi(G, c)], bits);
    size_t o = ((size_t)blk * G.H + h) * d + c;
    kzero[o] = double_to_half_bits_rn(p.zero);
    kscale[o] = double_to_half_bits_rn(p.scale);
  }
  // value groups [nblocks*g][H][nch][nb]
  for (int i = tid; i < g * G.nch * nb; i += blockDim.x) {
    int t = i / (G.nch * nb), rem = i - t * G.nch * nb, j = rem / nb, byte = rem - j * nb;
    uint32_t v = 0;
    for (int jj = 0; jj < per; ++jj) {
      int c = j * g + byte * per + jj;
      if (c >= min(d, (j + 1) * g)) break;
      int w, bit;
      vloc(G, t % G.tb, c, &w, &bit);
      v |= read_code(vw_of(t), w, bit, bits) << (jj * bits);
    }
    vcodes[((((size_t)blk * g + t) * G.H + h) * G.nch + j) * nb + byte] = (uint8_t)v;
  }
  for (int i = tid; i < g * G.nch; i += blockDim.x) {
    int t = i / G.nch, j = i - t * G.nch;
    GroupParams p = params_from_word(
        B.vparams[(bi + t / G.tb) * (size_t)G.rec + vpi(G, t % G.tb, vslot_of_group(G, j))], bits);
    size_t o = (((size_t)blk * g + t) * G.H + h) * G.nch + j;
    vzero[o] = double_to_half_bits_rn(p.zero);
    vscale[o] = double_to_half_bits_rn(p.scale);
  }
}

void launch_export(const Geo& G, const LayerBufs& B, int seq, int nblocks, uint8_t* kc,
                   uint16_t* kz, uint16_t* ks, uint8_t* vc, uint16_t* vz, uint16_t* vs,
                   cudaStream_t st) {
  if (nblocks <= 0) return;
  k_export<<<dim3(nblocks, G.H), 256, 0, st>>>(G, B, seq, nblocks, kc, kz, ks, vc, vz, vs);
}

// ---------------------------------------------------------------------------------
// Exact materialize of one (seq, head): float32 [n][d] keys and values,
// bit-identical to TwoTierCache.materialize (kvcache.py:222-243).
__device__ inline float packed_key(const Geo& G, const LayerBufs& B, int b, int h, int pos, int c) {
  int blk = pos / G.tb, t = pos - blk * G.tb;
  size_t bi = blk_index(G, b, h, blk);
  if (G.bits == 16)
    return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(B.kcodes + bi * (size_t)G.rec)[t * G.d + c]);
  int w, bit;
  kloc(G, t, c, &w, &bit);
  uint32_t code = read_code(B.kcodes + bi * (size_t)G.rec, w, bit, G.bits);
  return dequant_exact(code, params_from_word(B.kparams[bi * G.rec + kpi(G, c)], G.bits));
}
__device__ inline float packed_val(const Geo& G, const LayerBufs& B, int b, int h, int pos, int c) {
  int blk = pos / G.tb, t = pos - blk * G.tb;
  size_t bi = blk_index(G, b, h, blk);
  if (G.bits == 16)
    return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(B.vcodes + bi * (size_t)G.rec)[t * G.d + c]);
  int w, bit;
  vloc(G, t, c, &w, &bit);
  uint32_t code = read_code(B.vcodes + bi * (size_t)G.rec, w, bit, G.bits);
  return dequant_exact(code, params_from_word(B.vparams[bi * (size_t)G.rec + vpi(G, t, vslot(G, c))], G.bits));
}

__global__ void k_materialize(Geo G, LayerBufs B, int b, int h, int n, int f, float* keys,
                              float* values) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (size_t)n * G.d) return;
  int pos = (int)(i / G.d), c = (int)(i - (size_t)pos * G.d);
  float kv, vv;
  if (pos < f) {
    kv = packed_key(G, B, b, h, pos, c);
    vv = packed_val(G, B, b, h, pos, c);
  } else {
    size_t o = (((size_t)b * G.H + h) * G.ring + pos % G.ring) * G.d + c;
    kv = __bfloat162float(B.ring_k[o]);
    vv = __bfloat162float(B.ring_v[o]);
  }
  keys[i] = kv;
  values[i] = vv;
}

// pinned overrides (second pass): slot rows of the unit that contains head h
__global__ void k_materialize_pins(Geo G, LayerBufs B, int b, int h, float* keys, float* values) {
  int u = G.scope ? h : 0, hh = G.scope ? 0 : h;
  int slot = blockIdx.x;
  int pos = B.pin_pos[((size_t)b * G.U + u) * G.k + slot];
  if (pos < 0) return;
  size_t src = ((((size_t)b * G.U + u) * G.k + slot) * G.Hu + hh) * G.d;
  for (int c = threadIdx.x; c < G.d; c += blockDim.x) {
    keys[(size_t)pos * G.d + c] = __bfloat162float(B.pool_k[src + c]);
    values[(size_t)pos * G.d + c] = __bfloat162float(B.pool_v[src + c]);
  }
}

void launch_materialize(const Geo& G, const LayerBufs& B, int b, int h, int n, int f, float* keys,
                        float* values, cudaStream_t st) {
  size_t total = (size_t)n * G.d;
  if (total) {
    k_materialize<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(G, B, b, h, n, f, keys, values);
    k_materialize_pins<<<G.k, 128, 0, st>>>(G, B, b, h, keys, values);
  }
}

}  // namespace spc
