// exact_segment.cuh -- the exact (float64-dequant / full-precision) attention
// CTA, shared by the generic kernel (every split) and the tensor-core kernel
// (its last split: pinned slots + residual window + in-step rows).
// Reference semantics: engine.py:51-63,299-321; kvcache.py:222-243.
#pragma once
#include <math_constants.h>

#include "common.cuh"
#include "kernels.h"

namespace spc {

// 128-thread barrier so a 256-thread CTA can run this body on its first half
__device__ __forceinline__ void cta_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

constexpr int kCH = 128;   // items (tokens / rows) per chunk = threads per CTA
constexpr int kMaxR = 16;  // query rows per kv head (rows * Hq/H)
constexpr int kMaxD = 256;

__device__ inline float dq_key(const Geo& G, const LayerBufs& B, size_t bi, int t, int c) {
  if (G.bits == 16)
    return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(B.kcodes + bi * (size_t)G.rec)[t * G.d + c]);
  int w, bit;
  kloc(G, t, c, &w, &bit);
  uint32_t code = read_code(B.kcodes + bi * (size_t)G.rec, w, bit, G.bits);
  return dequant_exact(code, params_from_word(B.kparams[bi * G.rec + kpi(G, c)], G.bits));
}
__device__ inline float dq_val(const Geo& G, const LayerBufs& B, size_t bi, int t, int c) {
  if (G.bits == 16)
    return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(B.vcodes + bi * (size_t)G.rec)[t * G.d + c]);
  int w, bit;
  vloc(G, t, c, &w, &bit);
  uint32_t code = read_code(B.vcodes + bi * (size_t)G.rec, w, bit, G.bits);
  return dequant_exact(code, params_from_word(
      B.vparams[bi * (size_t)G.rec + vpi(G, t, vslot(G, c))], G.bits));
}

// One CTA (kCH threads, named barrier 1) of the exact path for (split, h, b).
// sm: dynamic shared memory of at least generic_smem_bytes().
__device__ __forceinline__ void generic_cta(const AttnArgs& a, const int split, const int h,
                                            const int b, float* sm) {
  const Geo& G = a.G;
  const LayerBufs& B = a.B;
  const int tid = threadIdx.x;
  const int R = a.rows * G.G, d = G.d;
  const bool exact_seg = (split == a.nsplit);
  const int unit = G.scope ? h : 0, hh = G.scope ? 0 : h;

  float* qs = sm;                      // [R][d]
  float* sc = qs + R * d;              // [R][kCH]  scores -> probabilities
  float* fac = sc + R * kCH;           // [R]
  float* mrow = fac + kMaxR;           // [R]
  float* lrow = mrow + kMaxR;          // [R]
  int* item_pos = reinterpret_cast<int*>(lrow + kMaxR);  // [kCH] spill position or -1
  int* slots = item_pos + kCH;         // [k] occupied slots (exact segment)
  __shared__ int s_npin;

  for (int i = tid; i < R * d; i += kCH) {
    int j = i / d, c = i - j * d, r = j / G.G, gq = j - r * G.G;
    qs[i] = __bfloat162float(a.q[(((size_t)b * a.rows + r) * G.Hq + h * G.G + gq) * d + c]);
  }
  if (tid < kMaxR) {
    mrow[tid] = -CUDART_INF_F;
    lrow[tid] = 0.f;
  }
  if (exact_seg && tid == 0) {
    int cnt = 0;
    const int32_t* pp = B.pin_pos + ((size_t)b * G.U + unit) * G.k;
    for (int s = 0; s < G.k; ++s)
      if (pp[s] >= 0) slots[cnt++] = s;
    s_npin = cnt;
  }
  cta_bar();

  float acc[kMaxR][kMaxD / kCH];
#pragma unroll
  for (int j = 0; j < kMaxR; ++j)
#pragma unroll
    for (int x = 0; x < kMaxD / kCH; ++x) acc[j][x] = 0.f;

  const uint32_t* bitmap = B.bitmap + ((size_t)b * G.U + unit) * (G.L / 32);
  const int npin = exact_seg ? s_npin : 0;
  const int nres = exact_seg ? (a.n - a.f) : 0;
  int total, begin = 0;
  if (exact_seg) {
    total = npin + nres + a.rows;
  } else {
    int blk0 = split * a.blocks_per_split;
    int blk1 = min(blk0 + a.blocks_per_split, a.f / G.tb);
    begin = blk0 * G.tb;
    total = max(0, blk1 - blk0) * G.tb;
  }

  float pin_m[kMaxR], pin_l[kMaxR];
  bool pin_recorded = false;
  // chunks never straddle the pinned / non-pinned boundary of the exact segment
  for (int c0 = 0; c0 < total;) {
    int cend = min(total, c0 + kCH);
    if (exact_seg && c0 < npin) cend = min(cend, npin);
    const int count = cend - c0;
    // ---- phase S: scores for item tid -------------------------------------------
    {
      float s[kMaxR];
#pragma unroll
      for (int j = 0; j < kMaxR; ++j) s[j] = 0.f;
      bool valid = tid < count, masked_all = false, spec = false;
      int pos = -1;
      const __nv_bfloat16* krow = nullptr;
      size_t bi = 0;
      int tb = 0;
      if (valid) {
        int it = c0 + tid;
        if (!exact_seg) {
          pos = begin + it;
          masked_all = (bitmap[pos >> 5] >> (pos & 31)) & 1u;
          int blk = pos / G.tb;
          tb = pos - blk * G.tb;
          bi = blk_index(G, b, h, blk);
        } else if (it < npin) {
          int slot = slots[it];
          pos = B.pin_pos[((size_t)b * G.U + unit) * G.k + slot];
          krow = B.pool_k + ((((size_t)b * G.U + unit) * G.k + slot) * G.Hu + hh) * d;
        } else if (it < npin + nres) {
          int p = a.f + (it - npin);
          krow = B.ring_k + (((size_t)b * G.H + h) * G.ring + p % G.ring) * d;
        } else {
          int r = it - npin - nres;
          spec = (r == 1);
          krow = a.k_new + (((size_t)b * a.rows + r) * G.H + h) * d;
        }
        if (!masked_all) {
          for (int c = 0; c < d; ++c) {
            float kv = krow ? __bfloat162float(krow[c]) : dq_key(G, B, bi, tb, c);
#pragma unroll
            for (int j = 0; j < kMaxR; ++j)
              if (j < R) s[j] = fmaf(qs[j * d + c], kv, s[j]);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < kMaxR; ++j) {
        if (j < R) {
          bool m = !valid || masked_all || (spec && j < G.G);  // row 0 never sees spec column
          // reference: (q.K) * float32(d^-0.5) in fp32, then exp(s - max); log2 domain here
          sc[j * kCH + tid] = m ? -CUDART_INF_F : s[j] * a.sm_scale_log2;
        }
      }
      item_pos[tid] = (valid && !masked_all && pos >= 0) ? pos : -1;
    }
    cta_bar();
    // spill the aggregate row's logits (one writer per position)
    if (item_pos[tid] >= 0) {
      int r = a.agg_row;
      for (int gq = 0; gq < G.G; ++gq)
        a.spill[((size_t)b * G.Hq + h * G.G + gq) * G.L + item_pos[tid]] = sc[(r * G.G + gq) * kCH + tid];
    }
    cta_bar();
    // ---- phase M: online softmax per row (warp per row) ---------------------------
    {
      int warp = tid >> 5, lane = tid & 31;
      for (int j = warp; j < R; j += kCH / 32) {
        float v[kCH / 32], mx = -CUDART_INF_F;
#pragma unroll
        for (int x = 0; x < kCH / 32; ++x) {
          v[x] = sc[j * kCH + lane + 32 * x];
          mx = fmaxf(mx, v[x]);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        float mold = mrow[j], mnew = fmaxf(mold, mx);
        float sum = 0.f;
#pragma unroll
        for (int x = 0; x < kCH / 32; ++x) {
          float p = (mnew == -CUDART_INF_F) ? 0.f : exp2f(v[x] - mnew);
          sc[j * kCH + lane + 32 * x] = p;
          sum += p;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        __syncwarp();
        if (lane == 0) {
          float f = (mold == -CUDART_INF_F) ? 0.f : exp2f(mold - mnew);
          fac[j] = f;
          mrow[j] = mnew;
          lrow[j] = lrow[j] * f + sum;
        }
      }
    }
    cta_bar();
    // ---- phase V: O += P V, thread per channel -------------------------------------
#pragma unroll
    for (int x = 0; x < kMaxD / kCH; ++x) {
      int c = tid + x * kCH;
      if (c < d) {
#pragma unroll
        for (int j = 0; j < kMaxR; ++j)
          if (j < R) acc[j][x] *= fac[j];
        for (int t = 0; t < count; ++t) {
          int it = c0 + t;
          float vv;
          if (!exact_seg) {
            int pos = begin + it;
            if ((bitmap[pos >> 5] >> (pos & 31)) & 1u) continue;  // p == 0
            int blk = pos / G.tb;
            vv = dq_val(G, B, blk_index(G, b, h, blk), pos - blk * G.tb, c);
          } else if (it < npin) {
            int slot = slots[it];
            vv = __bfloat162float(B.pool_v[((((size_t)b * G.U + unit) * G.k + slot) * G.Hu + hh) * d + c]);
          } else if (it < npin + nres) {
            int p = a.f + (it - npin);
            vv = __bfloat162float(B.ring_v[(((size_t)b * G.H + h) * G.ring + p % G.ring) * d + c]);
          } else {
            int r = it - npin - nres;
            vv = __bfloat162float(a.v_new[(((size_t)b * a.rows + r) * G.H + h) * d + c]);
          }
#pragma unroll
          for (int j = 0; j < kMaxR; ++j)
            if (j < R) acc[j][x] = fmaf(sc[j * kCH + t], vv, acc[j][x]);
        }
      }
    }
    cta_bar();
    c0 = cend;
    if (exact_seg && c0 == npin && !pin_recorded) {
#pragma unroll
      for (int j = 0; j < kMaxR; ++j) {
        pin_m[j] = j < R ? mrow[j] : 0.f;
        pin_l[j] = j < R ? lrow[j] : 0.f;
      }
      pin_recorded = true;
    }
  }
  if (exact_seg && !pin_recorded) {  // npin == 0
#pragma unroll
    for (int j = 0; j < kMaxR; ++j) {
      pin_m[j] = -CUDART_INF_F;
      pin_l[j] = 0.f;
    }
  }

  const size_t base = (((size_t)b * G.H + h) * (a.nsplit + 1) + split) * R;
#pragma unroll
  for (int x = 0; x < kMaxD / kCH; ++x) {
    int c = tid + x * kCH;
    if (c < d) {
#pragma unroll
      for (int j = 0; j < kMaxR; ++j)
        if (j < R) a.part_o[(base + j) * d + c] = acc[j][x];
    }
  }
  if (tid < R) {
    a.part_ml[(base + tid) * 2 + 0] = mrow[tid];
    a.part_ml[(base + tid) * 2 + 1] = lrow[tid];
    if (exact_seg) {
      size_t pb = ((size_t)b * G.H + h) * R + tid;
      a.pin_ml[pb * 2 + 0] = pin_m[tid];
      a.pin_ml[pb * 2 + 1] = pin_l[tid];
    }
  }
}


inline size_t generic_smem_bytes(const Geo& G, int rows) {
  int R = rows * G.G;
  return sizeof(float) * (R * G.d + R * kCH + 3 * kMaxR) + sizeof(int) * (kCH + G.k);
}

}  // namespace spc
