// hitrate.cu -- the hit-rate study on the device:
// attention tracing of a full-cache decode and the two retention curves the
// paper compares (Fig. 2-left): query-dependent top-k vs greedy cumulative-
// attention eviction (H2O-style).
//
//   spc_full_attend       exact fp32 attention of one decode step over a full
//                         cache, writing the per-q-head probability rows into a
//                         trace (3 chunked passes)             engine.py:51-63
//   spc_trace_row_sums    np.sum(row) of every trace row (float32 pairwise),
//                         the AttentionTrace.validate check   hitrate.py:27-31
//   spc_topk_hitrate      mass of the k largest entries of each row
//                                                             hitrate.py:34-43
//   spc_eviction_hitrate  greedy budget-k eviction driven by cumulative
//                         renormalised scores                 hitrate.py:46-77
//
// Trace layout: row (sequence s, query step t) starts at rows + s*seq_ld +
// t*row_ld and holds lens[t] fp32 probabilities (a "sequence" is one
// (layer, q head) of AttentionTrace.sequences(), hitrate.py:23-25).
//
// Parity.  The reference's arithmetic is reproduced operation for operation so
// the rates are bit-identical to hitrate.py on the same rows:
//  * top-k: the k largest values sorted descending, summed with numpy's
//    pairwise summation (the float64 add.reduce of np.sort(row)[::-1][:take],
//    hitrate.py:42) -- leaves of <= 128 elements with 8 strided accumulators,
//    splits at n/2 rounded down to a multiple of 8;
//  * eviction: mass and rate are left-to-right float64 sums over the
//    candidate list in its order (Python sum, hitrate.py:66,76), which is
//    ascending position order (retained positions keep their relative order
//    and new positions are appended above them); cumulative scores are
//    float64 x/mass increments (hitrate.py:69); the victims of one query are
//    the (len - k) smallest (cumulative, position) keys, i.e. repeated
//    min() with ties to the lower position (hitrate.py:71-73).
// Work: one CTA per row (top-k, sums) or per sequence (eviction, sequential in
// the query steps); the select is an MSB-first 8-bit radix select, the
// eviction compaction a block scan.
#include <cub/block/block_scan.cuh>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/specache.h"
#include "kernels.h"

namespace {

constexpr int kT = 256;  // threads per CTA for every kernel here

int cuda_status(cudaError_t e) {
  return e == cudaSuccess ? SPC_OK : spc::set_error(SPC_ECUDA, cudaGetErrorString(e));
}
int bad(const char* what) { return spc::set_error(SPC_EINVAL, what); }

// ---- numpy pairwise summation (loops_utils.h pairwise_sum), parallel leaves ----------
// Leaves are the n <= 128 nodes of the split tree; they are independent, so
// the CTA computes them in parallel and thread 0 folds them back in tree order.
constexpr int kMaxLeaves = 2056;  // >= 2049 leaves: n up to 262144 elements per call

struct PairwiseScratch {
  int leaf_lo[kMaxLeaves];
  int leaf_n[kMaxLeaves];
  double leaf_sum[kMaxLeaves];
  int nleaves;
};

// leaf sum with numpy's 8-accumulator loop (n <= 128) or the n < 8 loop
template <typename Acc, typename Get>
__device__ Acc pw_leaf(const Get& get, int lo, int n) {
  if (n < 8) {
    Acc res = Acc(0);
    for (int i = 0; i < n; ++i) res += (Acc)get(lo + i);
    return res;
  }
  Acc r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = (Acc)get(lo + j);
  int i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] += (Acc)get(lo + i + j);
  }
  Acc res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; ++i) res += (Acc)get(lo + i);
  return res;
}

// enumerate leaves left to right (thread 0): iterative DFS over the split tree
__device__ void pw_enumerate(PairwiseScratch& ps, int n) {
  int st_lo[40], st_n[40], sp = 0, cnt = 0;
  st_lo[sp] = 0;
  st_n[sp++] = n;
  while (sp) {
    const int lo = st_lo[--sp], m = st_n[sp];
    if (m <= 128) {
      ps.leaf_lo[cnt] = lo;
      ps.leaf_n[cnt++] = m;
    } else {
      int n2 = m / 2;
      n2 -= n2 % 8;
      st_lo[sp] = lo + n2;  // right pushed first: left is visited first
      st_n[sp++] = m - n2;
      st_lo[sp] = lo;
      st_n[sp++] = n2;
    }
  }
  ps.nleaves = cnt;
}

// fold leaf sums back in the recursion's order (thread 0)
template <typename Acc>
__device__ Acc pw_fold(const PairwiseScratch& ps, int n) {
  // post-order evaluation: (node size, state) stack; leaves consumed in order
  int st_n[40], st_state[40], sp = 0, leaf = 0;
  Acc val[40];
  int vp = 0;
  st_n[sp] = n;
  st_state[sp++] = 0;
  while (sp) {
    const int m = st_n[sp - 1];
    if (m <= 128) {
      --sp;
      val[vp++] = (Acc)ps.leaf_sum[leaf++];
      continue;
    }
    int n2 = m / 2;
    n2 -= n2 % 8;
    if (st_state[sp - 1] == 0) {
      st_state[sp - 1] = 1;
      st_n[sp] = n2;
      st_state[sp++] = 0;
    } else if (st_state[sp - 1] == 1) {
      st_state[sp - 1] = 2;
      st_n[sp] = m - n2;
      st_state[sp++] = 0;
    } else {
      --sp;
      const Acc b = val[--vp], a = val[--vp];
      val[vp++] = a + b;
    }
  }
  return val[0];
}

// CTA-wide numpy pairwise sum of get(0..n-1); result valid in thread 0
template <typename Acc, typename Get>
__device__ Acc pairwise_sum(PairwiseScratch& ps, const Get& get, int n) {
  if (n <= 128) {  // a single leaf
    Acc r = Acc(0);
    if (threadIdx.x == 0) r = pw_leaf<Acc>(get, 0, n);
    return r;
  }
  if (threadIdx.x == 0) pw_enumerate(ps, n);
  __syncthreads();
  for (int i = threadIdx.x; i < ps.nleaves; i += blockDim.x)
    ps.leaf_sum[i] = (double)pw_leaf<Acc>(get, ps.leaf_lo[i], ps.leaf_n[i]);
  __syncthreads();
  Acc r = Acc(0);
  if (threadIdx.x == 0) r = pw_fold<Acc>(ps, n);
  __syncthreads();
  return r;
}

__device__ __forceinline__ uint32_t ord32(float x) {  // order-preserving float -> uint
  const uint32_t b = __float_as_uint(x);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float unord32(uint32_t u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u);
}
__device__ __forceinline__ uint64_t ord64(double x) {
  const uint64_t b = (uint64_t)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// ---- exact fp32 attention of one step (engine.py:51-63) --------------------------------
// Three passes over position chunks of kFaChunk, grid (chunks, q heads) each, so a
// 32k-position row spreads over the whole GPU:
//   1. scores s_i = (q . k_i) * scale into the trace row (a warp per key row,
//      lanes over channels, coalesced) + the chunk max;
//   2. e_i = exp(s_i - M) with M the row max, the chunk sum, and the chunk's
//      partial P.V (thread per channel, rows of the chunk);
//   3. p_i = e_i / L with L the float64 sum of the chunk sums rounded to fp32
//      (masked_softmax_rows, numerics.py:24-39), and out = sum(partials) / L.
constexpr int kFaChunk = 1024;

__global__ void __launch_bounds__(kT) k_fa_scores(const float* __restrict__ q, const float* __restrict__ K, int n,
                                                  int group, int Hkv, int d, float scale, float* __restrict__ probs,
                                                  int64_t probs_ld, float* __restrict__ cmax, int nchunk) {
  const int chunk = blockIdx.x, hq = blockIdx.y, hk = hq / group;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* p = probs + (int64_t)hq * probs_ld;
  const float* qh = q + (size_t)hq * d;
  __shared__ float red[kT / 32];
  const int i0 = chunk * kFaChunk, i1 = min(n, i0 + kFaChunk);
  float mx = -INFINITY;
  for (int i = i0 + warp; i < i1; i += kT / 32) {
    const float* kr = K + ((size_t)i * Hkv + hk) * d;
    float s = 0.f;
    for (int c = lane; c < d; c += 32) s = fmaf(qh[c], kr[c], s);
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    s = s * scale;  // (q K^T) * float32(d^-1/2), two roundings like the reference
    if (lane == 0) p[i] = s;
    mx = fmaxf(mx, s);
  }
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = red[0];
    for (int w = 1; w < kT / 32; ++w) m = fmaxf(m, red[w]);
    cmax[(size_t)hq * nchunk + chunk] = m;
  }
}

__global__ void __launch_bounds__(kT) k_fa_exp(const float* __restrict__ V, int n, int group, int Hkv, int d,
                                               float* __restrict__ probs, int64_t probs_ld,
                                               const float* __restrict__ cmax, double* __restrict__ csum,
                                               float* __restrict__ opart, int nchunk) {
  const int chunk = blockIdx.x, hq = blockIdx.y, hk = hq / group;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* p = probs + (int64_t)hq * probs_ld;
  __shared__ float sM;
  __shared__ double dred[kT / 32];
  __shared__ float part[kT];
  if (threadIdx.x < 32) {
    float m = -INFINITY;
    for (int c = lane; c < nchunk; c += 32) m = fmaxf(m, cmax[(size_t)hq * nchunk + c]);
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) sM = m;
  }
  __syncthreads();
  const float M = sM;
  const int i0 = chunk * kFaChunk, i1 = min(n, i0 + kFaChunk);
  double sum = 0.0;
  for (int i = i0 + threadIdx.x; i < i1; i += kT) {
    const float e = expf(p[i] - M);
    p[i] = e;
    sum += (double)e;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if (lane == 0) dred[warp] = sum;
  __syncthreads();  // also orders this CTA's e_i writes before the P.V reads below
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kT / 32; ++w) s += dred[w];
    csum[(size_t)hq * nchunk + chunk] = s;
  }
  const int per = d <= kT ? kT / d : 1;
  const int c = threadIdx.x % d, grp = threadIdx.x / d;
  float acc = 0.f;
  if (threadIdx.x < per * d)
    for (int i = i0 + grp; i < i1; i += per) acc = fmaf(p[i], V[((size_t)i * Hkv + hk) * d + c], acc);
  part[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x < d) {
    float o = 0.f;
    for (int g2 = 0; g2 < per; ++g2) o += part[g2 * d + threadIdx.x];
    opart[((size_t)hq * nchunk + chunk) * d + threadIdx.x] = o;
  }
}

__global__ void __launch_bounds__(kT) k_fa_finish(int n, int d, float* __restrict__ probs, int64_t probs_ld,
                                                  const double* __restrict__ csum,
                                                  const float* __restrict__ opart, float* __restrict__ out,
                                                  int nchunk) {
  const int chunk = blockIdx.x, hq = blockIdx.y;
  float* p = probs + (int64_t)hq * probs_ld;
  __shared__ float sL;
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int c = 0; c < nchunk; ++c) s += csum[(size_t)hq * nchunk + c];
    sL = (float)s;
  }
  __syncthreads();
  const float L = sL;
  const int i0 = chunk * kFaChunk, i1 = min(n, i0 + kFaChunk);
  for (int i = i0 + threadIdx.x; i < i1; i += kT) p[i] = p[i] / L;
  if (chunk == 0 && threadIdx.x < d) {
    float o = 0.f;
    for (int c = 0; c < nchunk; ++c) o += opart[((size_t)hq * nchunk + c) * d + threadIdx.x];
    out[(size_t)hq * d + threadIdx.x] = o / L;
  }
}

// ---- np.sum(row) in float32 (AttentionTrace.validate) ----------------------------------
__global__ void __launch_bounds__(kT) k_row_sums(const float* __restrict__ rows, int64_t seq_ld, int64_t row_ld,
                                                 const int32_t* __restrict__ lens, int steps,
                                                 double* __restrict__ sums) {
  __shared__ PairwiseScratch ps;
  const int s = blockIdx.x / steps, t = blockIdx.x % steps;
  const float* x = rows + s * seq_ld + t * row_ld;
  const int n = lens[t];
  auto get = [&](int i) { return x[i]; };
  const float r = pairwise_sum<float>(ps, get, n);
  if (threadIdx.x == 0) sums[blockIdx.x] = (double)r;
}

// ---- top-k hit rate (hitrate.py:34-43) ------------------------------------------------------
// dynamic smem: [cap] float buffer for the k largest values (cap = pow2 >= take)
__global__ void __launch_bounds__(kT) k_topk_mass(const float* __restrict__ rows, int64_t seq_ld, int64_t row_ld,
                                                  const int32_t* __restrict__ lens, int steps, int k,
                                                  float* __restrict__ gscratch, int gcap,
                                                  double* __restrict__ rates) {
  extern __shared__ float sbuf[];
  __shared__ PairwiseScratch ps;
  __shared__ int hist[256];
  __shared__ uint32_t s_prefix;
  __shared__ int s_remaining, s_cnt;
  const int s = blockIdx.x / steps, t = blockIdx.x % steps;
  const float* x = rows + s * seq_ld + t * row_ld;
  const int n = lens[t];
  const int take = k < n ? k : n;
  if (take <= 0) {
    if (threadIdx.x == 0) rates[blockIdx.x] = 0.0;
    return;
  }
  int cap = 1;
  while (cap < take) cap <<= 1;
  float* buf = gscratch ? gscratch + (size_t)blockIdx.x * gcap : sbuf;
  // 1) radix select of the take-th largest key, MSB first
  uint32_t prefix = 0, mask = 0;
  int remaining = take;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += kT) hist[i] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += kT) {
      const uint32_t u = ord32(x[i]);
      if ((u & mask) == prefix) atomicAdd(&hist[(u >> shift) & 255u], 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // descending bins: find the bin holding the remaining-th largest
      int acc = 0, b = 255;
      for (; b > 0; --b) {
        if (acc + hist[b] >= remaining) break;
        acc += hist[b];
      }
      s_prefix = prefix | ((uint32_t)b << shift);
      s_remaining = remaining - acc;
    }
    __syncthreads();
    prefix = s_prefix;
    remaining = s_remaining;
    mask |= 255u << shift;
    __syncthreads();
  }
  // 2) gather: every key above the threshold, then `remaining` copies of it
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += kT) {
    const float v = x[i];
    if (ord32(v) > prefix) buf[atomicAdd(&s_cnt, 1)] = v;
  }
  __syncthreads();
  const int above = s_cnt;  // == take - remaining
  const float thr = unord32(prefix);
  for (int i = above + threadIdx.x; i < cap; i += kT) buf[i] = i < take ? thr : -INFINITY;
  __syncthreads();
  // 3) bitonic sort, descending
  for (int size = 2; size <= cap; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < cap; i += kT) {
        const int j = i ^ stride;
        if (j > i) {
          const bool desc = (i & size) == 0;
          const float a = buf[i], b = buf[j];
          if (desc ? (ord32(a) < ord32(b)) : (ord32(a) > ord32(b))) {
            buf[i] = b;
            buf[j] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  // 4) float64 pairwise sum of the descending values
  auto get = [&](int i) { return (double)buf[i]; };
  const double r = pairwise_sum<double>(ps, get, take);
  if (threadIdx.x == 0) rates[blockIdx.x] = r;
}

// ---- greedy eviction hit rate (hitrate.py:46-77) ----------------------------------------------
// one CTA per sequence; workspace per sequence: pos[2][cap] int32 + cum[2][cap] f64
__global__ void __launch_bounds__(kT) k_eviction(const float* __restrict__ rows, int64_t seq_ld, int64_t row_ld,
                                                 const int32_t* __restrict__ lens, int steps, int k, int cap,
                                                 int32_t* __restrict__ ws_pos, double* __restrict__ ws_cum,
                                                 double* __restrict__ rates) {
  using Scan = cub::BlockScan<int, kT>;
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ int hist[256];
  __shared__ uint64_t s_prefix;
  __shared__ int s_remaining, s_carry_eq, s_carry_keep;
  __shared__ double s_mass;
  const int s = blockIdx.x;
  int32_t* pos[2] = {ws_pos + (size_t)s * 2 * cap, ws_pos + (size_t)s * 2 * cap + cap};
  double* cum[2] = {ws_cum + (size_t)s * 2 * cap, ws_cum + (size_t)s * 2 * cap + cap};
  int cur = 0, r = 0, seen = 0;
  for (int t = 0; t < steps; ++t) {
    const float* x = rows + s * seq_ld + t * row_ld;
    const int n = lens[t];
    // cand = retained + range(seen, n) (hitrate.py:64-65), new cumulative 0.0
    const int add = n > seen ? n - seen : 0;
    for (int i = threadIdx.x; i < add; i += kT) {
      pos[cur][r + i] = seen + i;
      cum[cur][r + i] = 0.0;
    }
    const int m = r + add;
    seen = seen > n ? seen : n;
    __syncthreads();
    // mass: left-to-right float64 sum over cand (hitrate.py:66)
    if (threadIdx.x == 0) {
      double acc = 0.0;
      const int32_t* P = pos[cur];
      int i = 0;
      for (; i + 4 <= m; i += 4) {
        const float a = x[P[i]], b = x[P[i + 1]], c = x[P[i + 2]], e = x[P[i + 3]];
        acc += (double)a;
        acc += (double)b;
        acc += (double)c;
        acc += (double)e;
      }
      for (; i < m; ++i) acc += (double)x[P[i]];
      s_mass = acc;
    }
    __syncthreads();
    const double mass = s_mass;
    if (mass > 0.0)  // hitrate.py:67-69
      for (int i = threadIdx.x; i < m; i += kT) cum[cur][i] = cum[cur][i] + (double)x[pos[cur][i]] / mass;
    __syncthreads();
    int kept = m;
    if (m > k) {  // evict the e smallest (cumulative, position) keys (hitrate.py:70-73)
      const int e = m - k;
      uint64_t prefix = 0, mask = 0;
      int remaining = e;
      for (int shift = 56; shift >= 0; shift -= 8) {
        for (int i = threadIdx.x; i < 256; i += kT) hist[i] = 0;
        __syncthreads();
        for (int i = threadIdx.x; i < m; i += kT) {
          const uint64_t u = ord64(cum[cur][i]);
          if ((u & mask) == prefix) atomicAdd(&hist[(u >> shift) & 255u], 1);
        }
        __syncthreads();
        if (threadIdx.x == 0) {  // ascending bins: the bin holding the remaining-th smallest
          int acc = 0, b = 0;
          for (; b < 255; ++b) {
            if (acc + hist[b] >= remaining) break;
            acc += hist[b];
          }
          s_prefix = prefix | ((uint64_t)b << shift);
          s_remaining = remaining - acc;
        }
        __syncthreads();
        prefix = s_prefix;
        remaining = s_remaining;
        mask |= 255ull << shift;
        __syncthreads();
      }
      // evict keys < threshold and the first `remaining` keys == threshold (lowest positions)
      if (threadIdx.x == 0) {
        s_carry_eq = 0;
        s_carry_keep = 0;
      }
      __syncthreads();
      const int nxt = cur ^ 1;
      for (int base = 0; base < m; base += kT) {
        const int i = base + threadIdx.x;
        uint64_t u = 0;
        int eq = 0;
        if (i < m) {
          u = ord64(cum[cur][i]);
          eq = u == prefix;
        }
        int eq_rank, eq_tot;
        Scan(scan_tmp).ExclusiveSum(eq, eq_rank, eq_tot);
        __syncthreads();
        const int keep = (i < m) && (u > prefix || (eq && s_carry_eq + eq_rank >= remaining));
        int dst, keep_tot;
        Scan(scan_tmp).ExclusiveSum(keep, dst, keep_tot);
        if (keep) {
          pos[nxt][s_carry_keep + dst] = pos[cur][i];
          cum[nxt][s_carry_keep + dst] = cum[cur][i];
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          s_carry_eq += eq_tot;
          s_carry_keep += keep_tot;
        }
        __syncthreads();
      }
      kept = s_carry_keep;
      cur = nxt;
    }
    r = kept;
    __syncthreads();
    // rate: left-to-right float64 sum over the retained set (hitrate.py:76)
    if (threadIdx.x == 0) {
      double acc = 0.0;
      const int32_t* P = pos[cur];
      for (int i = 0; i < r; ++i) acc += (double)x[P[i]];
      rates[(size_t)s * steps + t] = acc;
    }
    __syncthreads();
  }
}

}  // namespace

extern "C" {

int spc_full_attend(const float* q, const float* k, const float* v, int n, int q_heads, int kv_heads,
                    int head_dim, float scale, float* out, float* probs, int64_t probs_ld, void* stream) {
  if (!q || !k || !v || !out || !probs) return bad("full_attend: null pointer");
  if (n <= 0) return bad("softmax row with every cell masked");
  if (q_heads <= 0 || kv_heads <= 0 || q_heads % kv_heads) return bad("q_heads must be a multiple of kv_heads");
  if (head_dim <= 0 || head_dim > kT) return bad("full_attend: head_dim must be in [1, 256]");
  if (probs_ld < n) return bad("full_attend: probs_ld < n");
  cudaStream_t st = (cudaStream_t)stream;
  const int nchunk = (n + kFaChunk - 1) / kFaChunk;
  const size_t nst = (size_t)q_heads * nchunk;
  char* ws = nullptr;
  if (cudaMallocAsync((void**)&ws, nst * (sizeof(float) + sizeof(double) + (size_t)head_dim * sizeof(float)), st) !=
      cudaSuccess)
    return spc::set_error(SPC_ENOMEM, "full_attend workspace");
  double* csum = reinterpret_cast<double*>(ws);
  float* cmax = reinterpret_cast<float*>(csum + nst);
  float* opart = cmax + nst;
  const dim3 grid(nchunk, q_heads);
  const int group = q_heads / kv_heads;
  k_fa_scores<<<grid, kT, 0, st>>>(q, k, n, group, kv_heads, head_dim, scale, probs, probs_ld, cmax, nchunk);
  k_fa_exp<<<grid, kT, 0, st>>>(v, n, group, kv_heads, head_dim, probs, probs_ld, cmax, csum, opart, nchunk);
  k_fa_finish<<<grid, kT, 0, st>>>(n, head_dim, probs, probs_ld, csum, opart, out, nchunk);
  cudaError_t e = cudaGetLastError();
  cudaFreeAsync(ws, st);
  return cuda_status(e);
}

int spc_trace_row_sums(const float* rows, int64_t seq_ld, int64_t row_ld, const int32_t* lens, int nseq, int steps,
                       int max_len, double* sums, void* stream) {
  if (!rows || !lens || !sums || nseq < 0 || steps < 0) return bad("trace_row_sums: bad arguments");
  if (max_len > 262144) return bad("trace rows longer than 262144 are unsupported");
  if (nseq == 0 || steps == 0) return SPC_OK;
  k_row_sums<<<nseq * steps, kT, 0, (cudaStream_t)stream>>>(rows, seq_ld, row_ld, lens, steps, sums);
  return cuda_status(cudaGetLastError());
}

int spc_topk_hitrate(const float* rows, int64_t seq_ld, int64_t row_ld, const int32_t* lens, int nseq, int steps,
                     int max_len, int k, double* rates, void* stream) {
  if (k < 0) return bad("k must be >= 0");
  if (!rows || !lens || !rates || nseq < 0 || steps < 0 || max_len < 0) return bad("topk_hitrate: bad arguments");
  if (max_len > 262144) return bad("trace rows longer than 262144 are unsupported");
  if (nseq == 0 || steps == 0) return SPC_OK;
  const int take = k < max_len ? k : max_len;
  int cap = 1;
  while (cap < take) cap <<= 1;
  cudaStream_t st = (cudaStream_t)stream;
  constexpr int kSmemCap = 16384;  // 64 KB of the value buffer in shared memory
  float* scratch = nullptr;
  size_t smem = 0;
  if (cap <= kSmemCap) {
    smem = (size_t)cap * sizeof(float);
    cudaFuncSetAttribute(k_topk_mass, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kSmemCap * 4));
  } else {
    cudaError_t e = cudaMallocAsync((void**)&scratch, (size_t)nseq * steps * cap * sizeof(float), st);
    if (e != cudaSuccess) return spc::set_error(SPC_ENOMEM, "topk_hitrate scratch");
  }
  k_topk_mass<<<nseq * steps, kT, smem, st>>>(rows, seq_ld, row_ld, lens, steps, k, scratch, cap, rates);
  cudaError_t e = cudaGetLastError();
  if (scratch) cudaFreeAsync(scratch, st);
  return cuda_status(e);
}

int spc_eviction_hitrate(const float* rows, int64_t seq_ld, int64_t row_ld, const int32_t* lens, int nseq,
                         int steps, int max_len, int k, double* rates, void* stream) {
  if (k < 0) return bad("k must be >= 0");
  if (!rows || !lens || !rates || nseq < 0 || steps < 0 || max_len < 0) return bad("eviction_hitrate: bad arguments");
  if (nseq == 0 || steps == 0) return SPC_OK;
  const int cap = max_len > 1 ? max_len : 1;  // candidates never exceed the longest row
  cudaStream_t st = (cudaStream_t)stream;
  int32_t* wpos = nullptr;
  double* wcum = nullptr;
  if (cudaMallocAsync((void**)&wpos, (size_t)nseq * 2 * cap * sizeof(int32_t), st) != cudaSuccess ||
      cudaMallocAsync((void**)&wcum, (size_t)nseq * 2 * cap * sizeof(double), st) != cudaSuccess) {
    if (wpos) cudaFreeAsync(wpos, st);
    return spc::set_error(SPC_ENOMEM, "eviction_hitrate workspace");
  }
  k_eviction<<<nseq, kT, 0, st>>>(rows, seq_ld, row_ld, lens, steps, k, cap, wpos, wcum, rates);
  cudaError_t e = cudaGetLastError();
  cudaFreeAsync(wpos, st);
  cudaFreeAsync(wcum, st);
  return cuda_status(e);
}

}  // extern "C"
