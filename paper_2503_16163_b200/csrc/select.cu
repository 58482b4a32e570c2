// select.cu -- K4 top-k selection + pin diff, K5 prefetch gather, K6 append.
//
// K4 replaces select_topk (engine.py:75-84) + the pin-set diff of
// _issue_ticket (engine.py:270-284) + pin (kvcache.py:194-218): a radix select
// over the fp32 bit patterns of agg (agg >= 0, so uint32 order == float order),
// ties to the lower position, emitted ascending; retained pins keep their slot,
// new pins take the slots of dropped pins, and only new pins are fetched
// (bytes charged = row_bytes(|new|), engine.py:274-276).
//
// K5 replaces slow_fetch + the ticket's worker fetch (kvcache.py:245-259,
// transfer.py:126-144): a zero-copy gather of the new rows from the pinned
// host slow tier over PCIe into the device slot pool, on the copy stream.
//
// K6 replaces append_verified (kvcache.py:162-171): row 0's K/V go to the
// residual ring (HBM) and to the slow tier (pinned host, zero-copy store).
#include <cstdlib>
#include "common.cuh"
#include "kernels.h"

namespace spc {

namespace {
constexpr int kTopkThreads = 1024;
constexpr int kMaxK = 1024;

__device__ inline int block_exclusive_scan(int v, int* warp_sums, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = lane < nw ? warp_sums[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nw) warp_sums[lane] = w;  // inclusive
    if (lane == nw - 1) *total = w;
  }
  __syncthreads();
  int before = (warp ? warp_sums[warp - 1] : 0) + x - v;
  __syncthreads();
  return before;
}
}  // namespace

// Radix select of the K largest of agg[0, f) (uint32 bit patterns of
// non-negative fp32), ties to the lower position, written ascending to sel[].
// Whole-CTA cooperative (kTopkThreads threads).
//
// Memory-level parallelism decides its speed (ncu, C4 rank share: 30% of the
// stall samples were long-scoreboard and 29% LSU throttle): every pass reads
// agg coalesced, 16 bytes per thread and four loads in flight, and the final
// position-ordered selection runs per warp over contiguous 32-element steps
// with ballots (round 1 gave each thread a private contiguous range: 32 cache
// lines per warp load).
__device__ void select_topk_cta(const uint32_t* __restrict__ agg, int f, int K, int* sel) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int kW = kTopkThreads / 32;
  __shared__ int hist[256];
  __shared__ int warp_sums[32];
  __shared__ int s_total, s_digit, s_remaining;
  __shared__ int w_gt[kW], w_eq[kW];
  uint32_t prefix = 0, pmask = 0;
  int remaining = K;
  const bool vec = ((reinterpret_cast<uintptr_t>(agg) & 15) == 0);
  const int f4 = vec ? (f >> 2) : 0;
  const uint4* agg4 = reinterpret_cast<const uint4*>(agg);
  if (K > 0) {
    for (int shift = 24; shift >= 0; shift -= 8) {
      for (int i = tid; i < 256; i += kTopkThreads) hist[i] = 0;
      __syncthreads();
      constexpr int U = 4;
      for (int i0 = tid; i0 < f4; i0 += U * kTopkThreads) {
        uint4 v4[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int i = i0 + u * kTopkThreads;
          v4[u] = i < f4 ? agg4[i] : make_uint4(~0u, ~0u, ~0u, ~0u);  // ~0u: never matches a prefix of agg >= 0
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t vv[4] = {v4[u].x, v4[u].y, v4[u].z, v4[u].w};
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (i0 + u * kTopkThreads < f4 && (vv[e] & pmask) == prefix) atomicAdd(&hist[(vv[e] >> shift) & 255u], 1);
        }
      }
      for (int i = 4 * f4 + tid; i < f; i += kTopkThreads) {
        uint32_t v = agg[i];
        if ((v & pmask) == prefix) atomicAdd(&hist[(v >> shift) & 255u], 1);
      }
      __syncthreads();
      if (tid < 32) {
        // find the digit, scanning bins from the top (warp-cooperative)
        int acc = 0, found = -1, before = 0;
        for (int base = 224; base >= 0 && found < 0; base -= 32) {
          int bin = base + (31 - tid);  // lane 0 -> highest bin of this slab
          int c = hist[bin];
          int x = c;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, x, o);
            if (tid >= o) x += y;
          }
          // x = count in bins [bin, base+31] (inclusive prefix from the top)
          unsigned hit = __ballot_sync(0xffffffffu, acc + x >= remaining);
          if (hit) {
            int l = __ffs(hit) - 1;
            int xl = __shfl_sync(0xffffffffu, x, l), cl = __shfl_sync(0xffffffffu, c, l);
            found = base + 31 - l;
            before = acc + xl - cl;
          } else {
            acc += __shfl_sync(0xffffffffu, x, 31);
          }
        }
        if (tid == 0) {
          s_digit = found;
          s_remaining = remaining - before;
        }
      }
      __syncthreads();
      prefix |= (uint32_t)s_digit << shift;
      pmask |= 255u << shift;
      remaining = s_remaining;
      __syncthreads();
    }
  }
  const uint32_t T = prefix;
  const int need_eq = remaining;  // elements == T to take, lowest positions first
  // selection in position order: warp w owns the contiguous range [w*per, (w+1)*per),
  // walked in coalesced 32-element steps; ballots order the lanes within a step
  const int per = ((f + kW - 1) / kW + 31) & ~31;
  const int r0 = min(f, warp * per), r1 = min(f, r0 + per);
  const unsigned lt = (1u << lane) - 1u;
  int n_gt = 0, n_eq = 0;
  if (K > 0)
    for (int i = r0 + lane; i - lane < r1; i += 32) {
      const uint32_t v = i < r1 ? agg[i] : 0u;
      n_gt += __popc(__ballot_sync(0xffffffffu, i < r1 && v > T));
      n_eq += __popc(__ballot_sync(0xffffffffu, i < r1 && v == T));
    }
  if (lane == 0) {
    w_gt[warp] = n_gt;
    w_eq[warp] = n_eq;
  }
  __syncthreads();
  if (K > 0) {
    int eq_before = 0, out = 0;  // exclusive prefix over the warps before this one
    for (int w = 0; w < warp; ++w) {
      const int te = max(0, min(w_eq[w], need_eq - eq_before));
      out += w_gt[w] + te;
      eq_before += w_eq[w];
    }
    int eq_left = max(0, need_eq - eq_before);  // equal elements this warp may still take
    for (int i = r0 + lane; i - lane < r1; i += 32) {
      const uint32_t v = i < r1 ? agg[i] : 0u;
      const unsigned beq = __ballot_sync(0xffffffffu, i < r1 && v == T);
      const bool eq_take = ((beq >> lane) & 1u) && __popc(beq & lt) < eq_left;
      const unsigned bt = __ballot_sync(0xffffffffu, (i < r1 && v > T) || eq_take);
      if ((bt >> lane) & 1u) sel[out + __popc(bt & lt)] = i;
      out += __popc(bt);
      eq_left -= min(eq_left, __popc(beq));
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kTopkThreads) k_topk(Geo G, LayerBufs B, int f) {
  const int u = blockIdx.x, b = blockIdx.y, tid = threadIdx.x;
  const size_t bu = (size_t)b * G.U + u;
  const uint32_t* agg = reinterpret_cast<const uint32_t*>(B.agg + bu * G.L);
  const int K = min(G.k, f);
  __shared__ int warp_sums[32];
  __shared__ int s_total;
  __shared__ int sel[kMaxK];
  __shared__ int keep[kMaxK];
  __shared__ int freelist[kMaxK];
  __shared__ int newlist[kMaxK];
  select_topk_cta(agg, f, K, sel);
  // ---- pin diff + slot assignment ------------------------------------------------
  int32_t* pin_pos = B.pin_pos + bu * G.k;
  uint32_t* bitmap = B.bitmap + bu * (G.L / 32);
  for (int s = tid; s < G.k; s += kTopkThreads) {
    int p = pin_pos[s], kp = 0;
    if (p >= 0) {  // binary search in the ascending selection
      int lo = 0, hi = K - 1;
      while (lo <= hi) {
        int mid = (lo + hi) >> 1;
        int v = sel[mid];
        if (v == p) { kp = 1; break; }
        if (v < p) lo = mid + 1; else hi = mid - 1;
      }
    }
    keep[s] = kp;
  }
  int is_new_cnt = 0, my_new[8];  // K <= kMaxK = 1024 -> at most 1 per thread
  for (int i = tid; i < K; i += kTopkThreads) {
    int p = sel[i];
    bool pinned = (bitmap[p >> 5] >> (p & 31)) & 1u;
    if (!pinned) my_new[is_new_cnt++] = p;
  }
  __syncthreads();
  int nfree_mine = 0;
  for (int s = tid; s < G.k; s += kTopkThreads) nfree_mine += !keep[s];
  int free_off = block_exclusive_scan(nfree_mine, warp_sums, &s_total);
  for (int s = tid; s < G.k; s += kTopkThreads)
    if (!keep[s]) freelist[free_off++] = s;
  int new_off = block_exclusive_scan(is_new_cnt, warp_sums, &s_total);
  const int nnew = s_total;
  for (int x = 0; x < is_new_cnt; ++x) newlist[new_off + x] = my_new[x];
  __syncthreads();
  // drop pins that were not re-selected
  for (int s = tid; s < G.k; s += kTopkThreads) {
    int p = pin_pos[s];
    if (p >= 0 && !keep[s]) {
      atomicAnd(&bitmap[p >> 5], ~(1u << (p & 31)));
      pin_pos[s] = -1;
    }
  }
  __syncthreads();
  for (int i = tid; i < nnew; i += kTopkThreads) {
    int slot = freelist[i], p = newlist[i];
    pin_pos[slot] = p;
    atomicOr(&bitmap[p >> 5], 1u << (p & 31));
    B.fetch_slot[bu * G.k + i] = slot;
    B.fetch_pos[bu * G.k + i] = p;
  }
  for (int i = tid; i < G.k; i += kTopkThreads) B.sel[bu * G.k + i] = i < K ? sel[i] : -1;
  if (tid == 0) {
    B.newcnt[bu] = nnew;
    atomicAdd(B.pf_rows, (unsigned long long)nnew);
  }
}

void launch_topk(const Geo& G, const LayerBufs& B, int f, cudaStream_t st) {
  k_topk<<<dim3(G.U, G.batch), kTopkThreads, 0, st>>>(G, B, f);
}

// Standalone select_topk (engine.py:75-84) over eligible = [0, n): out[k]
// ascending, -1 padded.  Used by the K4 parity tests on exact inputs.
__global__ void __launch_bounds__(kTopkThreads) k_select(const float* scores, int n, int k, int32_t* out) {
  __shared__ int sel[kMaxK];
  const int K = min(k, n);
  select_topk_cta(reinterpret_cast<const uint32_t*>(scores), n, K, sel);
  for (int i = threadIdx.x; i < k; i += kTopkThreads) out[i] = i < K ? sel[i] : -1;
}

void launch_select(const float* scores, int n, int k, int32_t* out, cudaStream_t st) {
  k_select<<<1, kTopkThreads, 0, st>>>(scores, n, k, out);
}

// Explicit pin() from the host API: replace the pinned set of one (seq, unit)
// with `pos` (ascending, unique, validated on the host), slot i <- pos[i].
__global__ void k_set_pins(Geo G, LayerBufs B, int seq, int unit, const int32_t* pos, int npos) {
  const size_t bu = (size_t)seq * G.U + unit;
  int32_t* pin_pos = B.pin_pos + bu * G.k;
  uint32_t* bitmap = B.bitmap + bu * (G.L / 32);
  for (int s = threadIdx.x; s < G.k; s += blockDim.x) {
    int p = pin_pos[s];
    if (p >= 0) atomicAnd(&bitmap[p >> 5], ~(1u << (p & 31)));
  }
  __syncthreads();
  for (int s = threadIdx.x; s < G.k; s += blockDim.x) {
    int p = s < npos ? pos[s] : -1;
    pin_pos[s] = p;
    if (p >= 0) {
      atomicOr(&bitmap[p >> 5], 1u << (p & 31));
      B.fetch_slot[bu * G.k + s] = s;
      B.fetch_pos[bu * G.k + s] = p;
    }
    B.sel[bu * G.k + s] = p;
  }
  if (threadIdx.x == 0) B.newcnt[bu] = npos;
}

void launch_set_pins(const Geo& G, const LayerBufs& B, int seq, int unit, const int32_t* pos,
                     int npos, cudaStream_t st) {
  k_set_pins<<<1, 256, 0, st>>>(G, B, seq, unit, pos, npos);
}

// K5: PCIe gather of the new pins (zero-copy loads from the pinned host tier).
// Few CTAs (a resident prefetch CTA costs its SM a K2 slot for the whole
// PCIe-bound gather), each thread keeping kPfUnroll independent 16-byte host
// loads of K and V in flight.  Rows of a unit's heads are contiguous in the host
// tier ([pos][H][d]).

template <int kPfUnroll>
__global__ void __launch_bounds__(kSideThreads, kSideMinBlocks) k_prefetch(Geo G, LayerBufs B, const uint4* host_k,
                                                  const uint4* host_v, int seq0, int unit0, int one) {
  const int bu_i = one ? 0 : blockIdx.y;
  const int u = one ? unit0 : bu_i % G.U, b = one ? seq0 : bu_i / G.U;
  const size_t bu = (size_t)b * G.U + u;
  const int nnew = B.newcnt[bu];
  const int h0 = G.scope ? u : 0;
  if (G.d % 8) {  // small / odd head dims: element copies
    const __nv_bfloat16* hk = reinterpret_cast<const __nv_bfloat16*>(host_k);
    const __nv_bfloat16* hv = reinterpret_cast<const __nv_bfloat16*>(host_v);
    const int row = G.Hu * G.d;
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < nnew * row; x += gridDim.x * blockDim.x) {
      const int i = x / row, e = x - i * row;
      const int slot = B.fetch_slot[bu * G.k + i], pos = B.fetch_pos[bu * G.k + i];
      const size_t src = (((size_t)b * G.L + pos) * G.H + h0) * G.d + e;
      const size_t dst = ((bu * G.k + slot) * G.Hu) * G.d + e;
      B.pool_k[dst] = hk[src];
      B.pool_v[dst] = hv[src];
    }
    return;
  }
  // the unit's (slot, position) list into shared memory first: the gather loop's
  // host loads then depend on a shared-memory read, not on an HBM round trip
  // each (k <= 1024 new pins: 8 KB)
  __shared__ int2 s_sp[1024];
  for (int i = threadIdx.x; i < nnew; i += blockDim.x)
    s_sp[i] = make_int2(B.fetch_slot[bu * G.k + i], B.fetch_pos[bu * G.k + i]);
  __syncthreads();
  const int vec = G.Hu * G.d / 8;  // uint4 per row
  const int total = nnew * vec;
  uint4* pk = reinterpret_cast<uint4*>(B.pool_k);
  uint4* pv = reinterpret_cast<uint4*>(B.pool_v);
  const int stride = gridDim.x * blockDim.x;
  for (int x0 = blockIdx.x * blockDim.x + threadIdx.x; x0 < total; x0 += stride * kPfUnroll) {
    uint4 rk[kPfUnroll], rv[kPfUnroll];
    size_t dst[kPfUnroll];
#pragma unroll
    for (int u2 = 0; u2 < kPfUnroll; ++u2) {
      const int x = x0 + u2 * stride;
      if (x < total) {
        const int i = x / vec, e = x - i * vec;
        const int2 sp = s_sp[i];
        const size_t src = (((size_t)b * G.L + sp.y) * G.H + h0) * G.d / 8 + e;
        dst[u2] = ((bu * G.k + sp.x) * G.Hu) * G.d / 8 + e;
        rk[u2] = host_k[src];
        rv[u2] = host_v[src];
      }
    }
#pragma unroll
    for (int u2 = 0; u2 < kPfUnroll; ++u2) {
      if (x0 + u2 * stride < total) {
        pk[dst[u2]] = rk[u2];
        pv[dst[u2]] = rv[u2];
      }
    }
  }
}

// Sysmem reads in flight = grid CTAs * 256 threads * depth * 32 B (K + V).  PCIe
// only needs its bandwidth-delay product (~150-250 KB); anything beyond queues in
// the memory system and slows every concurrent HBM client (measured: K2 -4%,
// cuBLAS GEMMs / small kernels up to 10x with 2 MB in flight).  So the grid and
// depth are sized from a byte budget, independent of batch size.
static void launch_pf(int64_t inflight, int units, const Geo& G, const LayerBufs& B, const __nv_bfloat16* host_k,
                      const __nv_bfloat16* host_v, int seq, int unit, int one, cudaStream_t st) {
  const uint4* hk = reinterpret_cast<const uint4*>(host_k);
  const uint4* hv = reinterpret_cast<const uint4*>(host_v);
  const int64_t per = inflight / units;            // bytes per (seq, unit)
  const int64_t cta2 = kSideThreads * 32 * 2;      // one CTA at depth 2
  if (per >= cta2) {
    const int ctas = (int)(per / cta2 < 16 ? per / cta2 : 16);
    k_prefetch<2><<<dim3(ctas, one ? 1 : units), kSideThreads, 0, st>>>(G, B, hk, hv, seq, unit, one);
  } else {
    k_prefetch<1><<<dim3(1, one ? 1 : units), kSideThreads, 0, st>>>(G, B, hk, hv, seq, unit, one);
  }
}

void launch_prefetch(const Geo& G, const LayerBufs& B, const __nv_bfloat16* host_k,
                     const __nv_bfloat16* host_v, int64_t inflight, cudaStream_t st) {
  launch_pf(inflight, G.U * G.batch, G, B, host_k, host_v, 0, 0, 0, st);
}

void launch_prefetch_one(const Geo& G, const LayerBufs& B, int seq, int unit,
                         const __nv_bfloat16* host_k, const __nv_bfloat16* host_v, cudaStream_t st) {
  launch_pf(int64_t(256) << 10, 1, G, B, host_k, host_v, seq, unit, 1, st);
}

// Host-link peak probe (spc_h2d_peak): a zero-copy read of a contiguous pinned
// buffer by `ctas` CTAs x 256 threads, 4 independent 16-byte loads per thread.
__global__ void __launch_bounds__(256) k_h2d_probe(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += 4 * stride) {
    uint4 r[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i + u * stride < n) r[u] = src[i + u * stride];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i + u * stride < n) dst[i + u * stride] = r[u];
  }
}

void launch_h2d_probe(const void* src, void* dst, size_t bytes, int ctas, cudaStream_t st) {
  k_h2d_probe<<<ctas, 256, 0, st>>>(reinterpret_cast<const uint4*>(src), reinterpret_cast<uint4*>(dst), bytes / 16);
}

// pin() with caller-supplied rows: device bf16 [npos][Hu][d] -> slots 0..npos-1
__global__ void k_copy_pins(Geo G, LayerBufs B, int seq, int unit, const __nv_bfloat16* kr,
                            const __nv_bfloat16* vr) {
  const int s = blockIdx.x;
  const size_t dst = ((((size_t)seq * G.U + unit) * G.k + s) * G.Hu) * G.d;
  const size_t src = (size_t)s * G.Hu * G.d;
  for (int x = threadIdx.x; x < G.Hu * G.d; x += blockDim.x) {
    B.pool_k[dst + x] = kr[src + x];
    B.pool_v[dst + x] = vr[src + x];
  }
}

void launch_copy_pins(const Geo& G, const LayerBufs& B, int seq, int unit, const __nv_bfloat16* k_rows,
                      const __nv_bfloat16* v_rows, int npos, cudaStream_t st) {
  if (npos > 0) k_copy_pins<<<npos, 256, 0, st>>>(G, B, seq, unit, k_rows, v_rows);
}

// K6a: append row 0 at position n to the residual ring (compute stream; the
// ring slot n % (r+g) is not read by this step's attention).
// One thread per 16-byte chunk (8 bf16) of the (seq, head, channel) row, grid
// (ceil(H*d/8 / 128), batch): a single wide pass instead of a 2-byte loop.
__global__ void k_ring_append(Geo G, LayerBufs B, const __nv_bfloat16* kr, const __nv_bfloat16* vr,
                              long long seq_stride, int n) {
  const int b = blockIdx.y, x = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (x >= G.H * G.d) return;
  const int slot = n % G.ring, h = x / G.d, c = x - h * G.d;
  const size_t ro = (((size_t)b * G.H + h) * G.ring + slot) * G.d + c;
  *reinterpret_cast<uint4*>(B.ring_k + ro) = *reinterpret_cast<const uint4*>(kr + (size_t)b * seq_stride + x);
  *reinterpret_cast<uint4*>(B.ring_v + ro) = *reinterpret_cast<const uint4*>(vr + (size_t)b * seq_stride + x);
}

// K6b: persist the row to the slow tier (pinned host, zero-copy 16-byte stores)
// from its ring slot (copy stream).
__global__ void k_host_append(Geo G, LayerBufs B, int n, __nv_bfloat16* host_k, __nv_bfloat16* host_v) {
  const int b = blockIdx.y, x = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (x >= G.H * G.d) return;
  const int slot = n % G.ring, h = x / G.d, c = x - h * G.d;
  const size_t ro = (((size_t)b * G.H + h) * G.ring + slot) * G.d + c;
  const size_t ho = (((size_t)b * G.L + n) * G.H + h) * G.d + c;
  *reinterpret_cast<uint4*>(host_k + ho) = *reinterpret_cast<const uint4*>(B.ring_k + ro);
  *reinterpret_cast<uint4*>(host_v + ho) = *reinterpret_cast<const uint4*>(B.ring_v + ro);
}

static bool rows_vectorizable(const Geo& G, long long seq_stride, const void* a, const void* b) {
  return G.d % 8 == 0 && seq_stride % 8 == 0 && ((uintptr_t)a & 15) == 0 && ((uintptr_t)b & 15) == 0;
}

__global__ void k_ring_append_scalar(Geo G, LayerBufs B, const __nv_bfloat16* kr, const __nv_bfloat16* vr,
                                     long long seq_stride, int n) {
  const int b = blockIdx.x;
  const int slot = n % G.ring;
  for (int x = threadIdx.x; x < G.H * G.d; x += blockDim.x) {
    const int h = x / G.d, c = x - h * G.d;
    const size_t ro = (((size_t)b * G.H + h) * G.ring + slot) * G.d + c;
    B.ring_k[ro] = kr[(size_t)b * seq_stride + x];
    B.ring_v[ro] = vr[(size_t)b * seq_stride + x];
  }
}

__global__ void k_host_append_scalar(Geo G, LayerBufs B, int n, __nv_bfloat16* host_k, __nv_bfloat16* host_v) {
  const int b = blockIdx.x;
  const int slot = n % G.ring;
  for (int x = threadIdx.x; x < G.H * G.d; x += blockDim.x) {
    const int h = x / G.d, c = x - h * G.d;
    const size_t ro = (((size_t)b * G.H + h) * G.ring + slot) * G.d + c;
    const size_t ho = (((size_t)b * G.L + n) * G.H + h) * G.d + c;
    host_k[ho] = B.ring_k[ro];
    host_v[ho] = B.ring_v[ro];
  }
}

void launch_ring_append(const Geo& G, const LayerBufs& B, const __nv_bfloat16* k_rows,
                        const __nv_bfloat16* v_rows, long long seq_stride, int n, cudaStream_t st) {
  if (rows_vectorizable(G, seq_stride, k_rows, v_rows)) {
    const int chunks = G.H * G.d / 8;
    k_ring_append<<<dim3((chunks + 127) / 128, G.batch), 128, 0, st>>>(G, B, k_rows, v_rows, seq_stride, n);
  } else {
    k_ring_append_scalar<<<G.batch, 256, 0, st>>>(G, B, k_rows, v_rows, seq_stride, n);
  }
}

void launch_host_append(const Geo& G, const LayerBufs& B, int n, __nv_bfloat16* host_k,
                        __nv_bfloat16* host_v, cudaStream_t st) {
  if (G.d % 8 == 0) {
    const int chunks = G.H * G.d / 8;
    k_host_append<<<dim3((chunks + 127) / 128, G.batch), 128, 0, st>>>(G, B, n, host_k, host_v);
  } else {
    k_host_append_scalar<<<G.batch, 256, 0, st>>>(G, B, n, host_k, host_v);
  }
}

// Prefill: residual rows [f, n) of K/V [b][n][H][d] into the ring.
__global__ void k_ring_fill(Geo G, LayerBufs B, const __nv_bfloat16* K, const __nv_bfloat16* V,
                            int n, int f) {
  const int pos = f + blockIdx.x, b = blockIdx.y;
  const int slot = pos % G.ring;
  for (int x = threadIdx.x; x < G.H * G.d; x += blockDim.x) {
    int h = x / G.d, c = x - h * G.d;
    size_t src = (((size_t)b * n + pos) * G.H + h) * G.d + c;
    size_t ro = (((size_t)b * G.H + h) * G.ring + slot) * G.d + c;
    B.ring_k[ro] = K[src];
    B.ring_v[ro] = V[src];
  }
}

void launch_ring_fill(const Geo& G, const LayerBufs& B, const __nv_bfloat16* K,
                      const __nv_bfloat16* V, int n, int f, cudaStream_t st) {
  if (n > f) k_ring_fill<<<dim3(n - f, G.batch), 256, 0, st>>>(G, B, K, V, n, f);
}

}  // namespace spc
