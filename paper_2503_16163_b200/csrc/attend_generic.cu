// attend_generic.cu -- K2 (exact path) + K3 (split combine, cross-head aggregate).
//
// Reference semantics (one layer of SpeculativeDecoder.decode_step,
// engine.py:299-321, and predecode, engine.py:245-268):
//   keys = [materialize (packed dequantized, pinned overridden, residual) ;
//           in-step rows], mask row 0 x speculative column (engine.py:310),
//   S = (q K^T) * float32(d^-0.5), A = masked softmax, O = A V (engine.py:51-63),
//   pinned_mass_j = sum_{i in P} A_j[0,i] (engine.py:314-316),
//   agg[i] = sum_{q heads} A_j[agg_row, i] (engine.py:317 / :262).
//
// This kernel dequantizes with the reference's exact float64 arithmetic, so
// the keys/values it attends over are bit-identical to materialize(); it is
// the correctness path for every geometry (bits 1/2/4/16, any d <= 256, any g)
// and the cross-check for the tensor-core fast path (attend_mma.cu).
//
// Grid (nsplit + 1, H, batch).  Splits 0..nsplit-1 stream contiguous ranges of
// packed g-token blocks with the pinned positions masked out; split nsplit is
// the "exact segment": pinned slot rows, the residual window and the in-step
// rows, all full precision.  Each CTA leaves an unnormalised partial (m, l, O)
// in the log2 domain; K3 merges them.
#include <math_constants.h>

#include <algorithm>
#include <cstdlib>

#include "exact_segment.cuh"

namespace spc {

__global__ void __launch_bounds__(kCH) k_attend_generic(AttnArgs a) {
  extern __shared__ __align__(16) float sm[];
  generic_cta(a, blockIdx.x, blockIdx.y, blockIdx.z, sm);
}

void launch_attend_generic(const AttnArgs& a, cudaStream_t st) {
  const Geo& G = a.G;
  size_t smem = generic_smem_bytes(G, a.rows);
  static std::atomic<unsigned long long> done{0};
  ensure_smem_attr(done, k_attend_generic, 200 * 1024);
  dim3 grid(a.nsplit + 1, G.H, G.batch);
  k_attend_generic<<<grid, kCH, smem, st>>>(a);
}

// ---------------------------------------------------------------------------------
// K3a: merge split partials -> O (bf16), agg-row (max, sum), pinned mass.
// One CTA per (q head, seq, row).  Warp 0 reduces the row's per-split (max,
// sum) with lanes striding the splits and leaves one factor exp2(m_s - M) per
// split in shared memory; every thread then sums its channel over the splits,
// eight independent loads at a time.  The kernel sits on the compute stream
// between two attention launches and is memory-latency bound (ncu: 87%
// long-scoreboard stalls, 11% warps active in round 1's one-CTA-per-head form).
constexpr int kCombineSplits = 132;  // >= kSplitCap + 1 (api.cu) + padding
__global__ void __launch_bounds__(128) k_combine(AttnArgs a) {
  const Geo G = a.G;
  const int hq = blockIdx.x, b = blockIdx.y, r = blockIdx.z, h = hq / G.G, gq = hq - h * G.G;
  const int R = a.rows * G.G, S = a.nsplit + 1, j = r * G.G + gq;
  const int lane = threadIdx.x & 31;
  __shared__ float sf[kCombineSplits];
  __shared__ float sML[2];
  const size_t base = ((size_t)b * G.H + h) * S * R;
  // the first 16 splits' partials are loaded before the barrier: they do not
  // depend on the factors, so their latency overlaps warp 0's (max, sum) pass
  const size_t sstride = (size_t)R * G.d;
  const int c0 = threadIdx.x;
  const bool cl = c0 < G.d;
  const float* po = a.part_o + (base + j) * G.d + (cl ? c0 : 0);
  float pre[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) pre[u] = (cl && u < S) ? po[(size_t)u * sstride] : 0.f;
  if (threadIdx.x < 32) {
    float M = -CUDART_INF_F;
    for (int s = lane; s < S; s += 32) {
      const float2 ml = *reinterpret_cast<const float2*>(&a.part_ml[(base + (size_t)s * R + j) * 2]);
      if (ml.y > 0.f) M = fmaxf(M, ml.x);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    float L = 0.f;
    for (int s = lane; s < S; s += 32) {
      const float2 ml = *reinterpret_cast<const float2*>(&a.part_ml[(base + (size_t)s * R + j) * 2]);
      const float f = ml.y > 0.f ? exp2f(ml.x - M) : 0.f;
      sf[s] = f;
      L = fmaf(ml.y, f, L);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
    if (lane == 0) {
      sML[0] = M;
      sML[1] = L;
    }
  }
  __syncthreads();
  const float M = sML[0], L = sML[1], invL = 1.f / L;
  for (int c = c0; c < G.d; c += blockDim.x) {
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    int s0 = 0;
    if (c == c0) {
#pragma unroll
      for (int u = 0; u < 16; ++u)
        if (u < S) acc[u & 7] = fmaf(pre[u], sf[u], acc[u & 7]);
      s0 = 16;
    }
    const float* pc = a.part_o + (base + j) * G.d + c;
    for (; s0 + 8 <= S; s0 += 8) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = pc[(size_t)(s0 + u) * sstride];
#pragma unroll
      for (int u = 0; u < 8; ++u) acc[u] = fmaf(v[u], sf[s0 + u], acc[u]);
    }
    for (int s = s0; s < S; ++s) acc[0] = fmaf(pc[(size_t)s * sstride], sf[s], acc[0]);
    const float o = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
    const size_t oi = (((size_t)b * a.rows + r) * G.Hq + hq) * G.d + c;
    a.out[oi] = __float2bfloat16_rn(o * invL);
    if (a.out_f32) a.out_f32[oi] = o * invL;
  }
  if (a.ring_append && r == 0 && gq == 0) {
    // K6a fused: row 0's K and V of kv head h into the residual ring, slot n % ring
    // (kvcache.py:162-171; the attention of this layer has finished reading the ring)
    const size_t ro = (((size_t)b * G.H + h) * G.ring + a.n % G.ring) * G.d;
    const size_t io = ((size_t)b * a.rows * G.H + h) * G.d;
    for (int x = threadIdx.x * 8; x < G.d; x += blockDim.x * 8) {
      *reinterpret_cast<uint4*>(a.B.ring_k + ro + x) = *reinterpret_cast<const uint4*>(a.k_new + io + x);
      *reinterpret_cast<uint4*>(a.B.ring_v + ro + x) = *reinterpret_cast<const uint4*>(a.v_new + io + x);
    }
  }
  if (threadIdx.x == 0) {
    if (r == a.agg_row) {
      a.mz[((size_t)b * G.Hq + hq) * 2 + 0] = M;
      a.mz[((size_t)b * G.Hq + hq) * 2 + 1] = L;
    }
    if (r == 0 && a.pinned_mass) {
      size_t pb = ((size_t)b * G.H + h) * R + j;
      float pl = a.pin_ml[pb * 2 + 1];
      a.pinned_mass[(size_t)b * G.Hq + hq] = pl > 0.f ? pl * exp2f(a.pin_ml[pb * 2] - M) * invL : 0.f;
    }
  }
}

void launch_combine(const AttnArgs& a, cudaStream_t st) {
  k_combine<<<dim3(a.G.Hq, a.G.batch, a.rows), 128, 0, st>>>(a);
}

// K3b: agg[i] = sum over the unit's q heads of A_j[agg_row, i], i < f, in
// ascending head order like np.sum(axis=0) (engine.py:317).
__global__ void __launch_bounds__(kSideThreads, kSideMinBlocks) k_agg(AttnArgs a) {
  const Geo G = a.G;
  const int u = blockIdx.y, b = blockIdx.z;
  const int h0 = G.scope ? u * G.G : 0, h1 = G.scope ? (u + 1) * G.G : G.Hq;
  extern __shared__ float s_mi[];  // [heads] max, [heads] 1/sum
  float* sM = s_mi;
  float* sI = s_mi + (h1 - h0);
  for (int x = threadIdx.x; x < h1 - h0; x += blockDim.x) {
    sM[x] = a.mz[((size_t)b * G.Hq + h0 + x) * 2];
    sI[x] = 1.f / a.mz[((size_t)b * G.Hq + h0 + x) * 2 + 1];
  }
  __syncthreads();
  const float* sp = a.spill + ((size_t)b * G.Hq + h0) * G.L;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.f; i += gridDim.x * blockDim.x) {
    // unrolled so that up to 8 heads' spill loads are in flight at once; the
    // sum stays in ascending head order
    float acc = 0.f;
#pragma unroll 8
    for (int x = 0; x < h1 - h0; ++x) acc += exp2f(sp[(size_t)x * G.L + i] - sM[x]) * sI[x];
    a.B.agg[((size_t)b * G.U + u) * G.L + i] = acc;
  }
}

void launch_agg(const AttnArgs& a, cudaStream_t st) {
  if (a.f <= 0) return;
  // total CTA budget of the launch (tuning: SPC_AGG_CTAS).  K3 runs on a copy
  // stream while the next layer's K2 fills the machine; every K3 CTA takes a
  // slot a retiring K2 CTA leaves
  static const int budget = [] {
    const char* e = getenv("SPC_AGG_CTAS");
    return e ? std::max(1, atoi(e)) : 2 * 148 * 4;
  }();
  const int blocks = std::min((a.f + 255) / 256, std::max(1, budget / (a.G.U * a.G.batch)));
  const int heads = a.G.scope ? a.G.G : a.G.Hq;
  k_agg<<<dim3(blocks, a.G.U, a.G.batch), kSideThreads, 2 * heads * sizeof(float), st>>>(a);
}

// K3r (spc_set_agg_mode(cache, 1), SURVEY hard part (b) option 2): the
// aggregate without the spill.  K2 writes no packed-position logits; this
// kernel re-reads each 32-token record's key codes and key params and
// recomputes the speculative row's log2 scores of the unit's q heads on the
// CUDA cores (fp32, dequantized keys like materialize, kvcache.py:222-243),
// then agg[i] = sum_h exp2(s_h[i] - M_h) / Z_h with the combined (M, Z).
// Pinned positions keep the exact-row logits the exact segment spilled.  The
// measured point of this option: it streams the key half of the packed tier
// again (48 B / 32 B per token per KV head at 2 / 1 bit) against the spill's
// 8 B / 32 B write + read.
constexpr int kAggRcWarps = 8;
__global__ void __launch_bounds__(kAggRcWarps * 32) k_agg_recompute(AttnArgs a) {
  const Geo G = a.G;
  const int u = blockIdx.y, b = blockIdx.z, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kh0 = G.scope ? u : 0, nkv = G.scope ? 1 : G.H, nq = nkv * G.G, j0 = kh0 * G.G;
  extern __shared__ float sm[];
  float* sQ = sm;                      // [nq][d] speculative-row queries * d^-0.5 * log2(e)
  float* sM = sQ + nq * G.d;           // [nq]
  float* sI = sM + nq;                 // [nq]
  float* sP = sI + nq;                 // [warps][2][d] key params (s, z) of the warp's current head
  float* sAcc = sP + kAggRcWarps * 2 * G.d;  // [warps][32]
  for (int x = threadIdx.x; x < nq * G.d; x += blockDim.x) {
    const int j = x / G.d, c = x - j * G.d;
    sQ[x] = __bfloat162float(a.q[(((size_t)b * a.rows + a.agg_row) * G.Hq + j0 + j) * G.d + c]) * a.sm_scale_log2;
  }
  for (int x = threadIdx.x; x < nq; x += blockDim.x) {
    sM[x] = a.mz[((size_t)b * G.Hq + j0 + x) * 2];
    sI[x] = 1.f / a.mz[((size_t)b * G.Hq + j0 + x) * 2 + 1];
  }
  __syncthreads();
  const int nblk = a.f / G.tb;
  const uint32_t* bm = a.B.bitmap + ((size_t)b * G.U + u) * (G.L / 32);
  const uint32_t mask = (1u << G.bits) - 1u;
  float* wp = sP + warp * 2 * G.d;
  for (int blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    const int t = lane, pos = blk * G.tb + t;
    const bool pinned = (bm[pos >> 5] >> (pos & 31)) & 1u;
    float acc = 0.f;
    for (int kq = warp; kq < nkv; kq += kAggRcWarps) {
      const int kh = kh0 + kq;
      const size_t bi = blk_index(G, b, kh, blk);
      const uint32_t* rec = a.B.kcodes + bi * (size_t)G.rec;
      const uint32_t* kp = a.B.kparams + bi * (size_t)G.rec;
      __syncwarp();
      for (int c = lane; c < G.d; c += 32) {  // group params of this record, per channel
        const GroupParams p = params_from_word(kp[kpi(G, c)], G.bits);
        wp[c] = (float)p.scale;
        wp[G.d + c] = (float)p.zero;
      }
      __syncwarp();
      float dot[8];
#pragma unroll
      for (int g2 = 0; g2 < 8; ++g2) dot[g2] = 0.f;
      const uint32_t* row = rec + t * G.krw;  // token t's key codes, channels LSB-first (kloc)
      for (int w = 0; w < G.krw; ++w) {
        const uint32_t word = row[w];
        const int per = 32 / G.bits;
#pragma unroll 4
        for (int e = 0; e < per; ++e) {
          const int c = w * per + e;
          if (c >= G.d) break;
          const float kv = fmaf((float)((word >> (G.bits * e)) & mask), wp[c], wp[G.d + c]);
#pragma unroll
          for (int g2 = 0; g2 < 8; ++g2)
            if (g2 < G.G) dot[g2] = fmaf(kv, sQ[(kq * G.G + g2) * G.d + c], dot[g2]);
        }
      }
#pragma unroll
      for (int g2 = 0; g2 < 8; ++g2) {
        if (g2 >= G.G) break;
        const int jl = kq * G.G + g2;
        const float s2 = pinned ? a.spill[((size_t)b * G.Hq + j0 + jl) * G.L + pos] : dot[g2];
        acc += exp2f(s2 - sM[jl]) * sI[jl];
      }
    }
    sAcc[warp * 32 + lane] = acc;
    __syncthreads();
    if (warp == 0) {
      float tot = 0.f;
#pragma unroll
      for (int w2 = 0; w2 < kAggRcWarps; ++w2) tot += sAcc[w2 * 32 + lane];
      a.B.agg[((size_t)b * G.U + u) * G.L + pos] = tot;
    }
    __syncthreads();
  }
}

void launch_agg_recompute(const AttnArgs& a, cudaStream_t st) {
  if (a.f <= 0) return;
  const Geo& G = a.G;
  const int nq = (G.scope ? 1 : G.H) * G.G;
  const size_t smem = sizeof(float) * ((size_t)nq * G.d + 2 * nq + kAggRcWarps * 2 * G.d + kAggRcWarps * 32);
  cudaFuncSetAttribute(k_agg_recompute, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int nblk = a.f / G.tb;
  const int blocks = std::min(nblk, std::max(1, 2 * 148 * 4 / (G.U * G.batch)));
  k_agg_recompute<<<dim3(blocks, G.U, G.batch), kAggRcWarps * 32, smem, st>>>(a);
}

}  // namespace spc
