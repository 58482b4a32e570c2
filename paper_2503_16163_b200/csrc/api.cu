// api.cu -- the C ABI (include/specache.h): cache object, allocation, streams,
// per-layer ticket protocol, and the K1..K6 launch sequence of one decode layer.
//
// Stream structure per layer l (SURVEY.md 8(b) "Threading"):
//   compute stream     : [wait ev_pf(l)] K2 attend (+K3 combine) -> K6a ring
//                        append -> record ev_att(l)
//   select stream l % 2: [wait ev_att(l)] K3 cross-head aggregate -> K4 top-k +
//   (lowest priority)    pin diff -> record ev_sel(l)
//   copy stream l % 2  : [wait ev_sel(l)] K5 PCIe prefetch -> K6b slow-tier write
//   (high priority)      (+K1 migration) -> record ev_pf(l)
// The selection CTAs (a 1184-CTA aggregate, 1024-thread top-k CTAs) would
// otherwise take every SM slot a retiring K2 CTA leaves; at low priority they
// fill K2's gaps instead, while the PCIe gather keeps its slots.
// Only attention sits on the caller's stream; the selection, the PCIe gather
// and the slow-tier write for step t+1 overlap the next layers' attention.
// decode_layer(l, t+1) waits on ev_pf(l) -- the device form of
// SimulatedChannel.await_layer (transfer.py:96-100).  Spill buffers are per
// layer so the aggregate can lag the compute stream.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/specache.h"
#include "common.cuh"
#include "kernels.h"

using namespace spc;

namespace {
thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
}  // namespace

namespace spc {
int set_error(int code, const char* msg) {
  g_err = msg;
  return code;
}
}  // namespace spc

namespace {
#define CUDA_TRY(expr)                                                               \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess)                                                           \
      return fail(SPC_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));    \
  } while (0)

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
int64_t frontier_of(int64_t n, int r, int g) { return n < r ? 0 : (int64_t)g * ((n - r) / g); }
constexpr int kSplitCap = 128;
// Measurement only: SPC_DEBUG_SKIP bitmask skips side kernels of the decode
// layer (1 = K3b aggregate, 2 = K4 top-k, 4 = K5 PCIe gather) to price their
// interference with K2 in the layer loop.  Results are invalid when set.
int debug_skip() {
  static const int v = [] {
    const char* e = getenv("SPC_DEBUG_SKIP");
    return e ? atoi(e) : 0;
  }();
  return v;
}
constexpr int kNumSMs = 148;
}  // namespace

struct spc_cache {
  Geo G{};
  int device = 0;
  int impl = 0;  // 0 auto, 1 generic exact, 2 fast
  int agg_mode = 0;  // 0 spill (K2 writes the speculative logits), 1 recompute (K3r)
  int64_t pf_inflight = int64_t(256) << 10;  // K5 sysmem bytes in flight (spc_set_prefetch_inflight)
  std::vector<LayerBufs> L;
  std::vector<void*> dev_allocs;
  __nv_bfloat16* host_k = nullptr;
  __nv_bfloat16* host_v = nullptr;
  size_t host_bytes = 0, dev_bytes = 0, slab_elems = 0;
  std::vector<int64_t> n, f;
  std::vector<int> ticket;  // pending ticket step per layer (-1 none)
  cudaStream_t copy_stream = nullptr, copy_stream2 = nullptr;
  // selection streams (K3 aggregate + K4 top-k): the copy streams themselves,
  // or separate lower-priority streams (SPC_COPY_PRIO=split) so that the
  // selection CTAs only take SM slots K2 leaves free while the PCIe gather keeps
  // its high priority
  cudaStream_t sel_stream = nullptr, sel_stream2 = nullptr;
  std::vector<cudaEvent_t> ev_agg, ev_pf, ev_sel;
  cudaStream_t cstream(int layer) const { return (layer & 1) ? copy_stream2 : copy_stream; }
  cudaStream_t sstream(int layer) const {
    return sel_stream ? ((layer & 1) ? sel_stream2 : sel_stream) : cstream(layer);
  }
  float *part_o = nullptr, *part_ml = nullptr, *pin_ml = nullptr, *spill = nullptr, *mz = nullptr;
  float* dbg_out = nullptr;  // spc_debug_output_f32: [layers][b][2][Hq][d] fp32 outputs
  int32_t* staging = nullptr;
  unsigned long long* pf_rows = nullptr;
  int context_length = 0;
  // live profiling of the dominant kernel (K2) and the copy-stream work (K4+K5)
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_attn, prof_sel, prof_wait, prof_pf;
  cudaEvent_t prof_base = nullptr;  // recorded when profiling starts: common origin of the intervals
  double last_pf_wall_ms = 0;
  int64_t launches = 0;
  double last_wait_ms = 0, last_pf_ms = 0;
  int64_t last_pf_rows = 0;
  // head-sharded layer scope (spc_set_agg_reduce): the ticket tail waits for the
  // caller's cross-rank reduction of agg, enqueued on the copy stream
  bool agg_ext = false;
  struct Pending {
    bool on = false, append = false;
    int f = 0, n_before = 0;
    cudaEvent_t p0 = nullptr;
  };
  std::vector<Pending> pend;
  // step graphs (spc_graph_begin / spc_graph_launch): the decode calls between
  // them are captured from the caller's stream, then replayed as one graph
  bool capturing = false, capture_failed = false;
  cudaStream_t cap_stream = nullptr;
  cudaGraphExec_t gexec[2] = {nullptr, nullptr};
  int gexec_last = 0;
  cudaEvent_t ev_join[4] = {nullptr, nullptr, nullptr, nullptr};
  int64_t graph_updates = 0, graph_instantiations = 0;
};

namespace {
int dalloc(spc_cache* c, void** p, size_t bytes) {
  bytes = std::max<size_t>(bytes, 256);
  cudaError_t e = cudaMalloc(p, bytes);
  if (e != cudaSuccess)
    return fail(SPC_ENOMEM, std::string("cudaMalloc(") + std::to_string(bytes) + "): " + cudaGetErrorString(e));
  c->dev_allocs.push_back(*p);
  c->dev_bytes += bytes;
  return SPC_OK;
}

__nv_bfloat16* host_slab(spc_cache* c, __nv_bfloat16* base, int layer) {
  return base + (size_t)(layer % c->G.host_layers) * c->slab_elems;
}

int check_layer(const spc_cache* c, int layer) {
  if (!c) return fail(SPC_EINVAL, "null cache");
  if (layer < 0 || layer >= c->G.layers) return fail(SPC_EINVAL, "layer out of range");
  return SPC_OK;
}

int no_capture(const spc_cache* c) {
  if (c->capturing)
    return fail(SPC_EPROTO, "only spc_decode_layer may be called between spc_graph_begin and spc_graph_launch");
  return SPC_OK;
}

int check_not_pending(const spc_cache* c, int layer, bool capture_ok = false) {
  if (!capture_ok)
    if (int rc = no_capture(c)) return rc;
  if (c->pend[layer].on)
    return fail(SPC_EPROTO, "layer " + std::to_string(layer) +
                                ": the aggregate awaits its cross-rank reduction (call spc_finish_layer)");
  return SPC_OK;
}

void choose_splits(const spc_cache* c, int f, int* nsplit, int* bps) {
  const Geo& G = c->G;
  int nblk = f / G.tb;
  if (nblk <= 0) {
    *nsplit = 1;
    *bps = 1;
    return;
  }
  int want = (2 * kNumSMs + G.H * G.batch - 1) / (G.H * G.batch);
  want = std::max(1, std::min(want, std::min(kSplitCap, nblk)));
  *bps = (nblk + want - 1) / want;
  *nsplit = (nblk + *bps - 1) / *bps;
}

int migrate(spc_cache* c, int layer, cudaStream_t st) {
  const Geo& G = c->G;
  QuantSrc S{c->L[layer].ring_k, c->L[layer].ring_v, (long long)G.H * G.ring * G.d, (long long)G.d,
             (long long)G.ring * G.d, G.ring};
  // ring layout is [b][H][ring][d]: row stride d, head stride ring*d
  launch_quantize(G, c->L[layer], S, (int)(c->f[layer] / G.g), 1, st);
  CUDA_TRY(cudaGetLastError());
  c->launches += 1;
  c->f[layer] += G.g;
  return SPC_OK;
}

// append_verified on one stream: ring + slow tier + migration (kvcache.py:162-171)
int append_rows(spc_cache* c, int layer, const void* kr, const void* vr, int64_t seq_stride,
                cudaStream_t st) {
  const Geo& G = c->G;
  if (c->n[layer] >= c->context_length)
    return fail(SPC_EINVAL, "context_length exceeded");
  launch_ring_append(G, c->L[layer], (const __nv_bfloat16*)kr, (const __nv_bfloat16*)vr,
                     seq_stride ? seq_stride : (int64_t)G.H * G.d, (int)c->n[layer], st);
  launch_host_append(G, c->L[layer], (int)c->n[layer], host_slab(c, c->host_k, layer),
                     host_slab(c, c->host_v, layer), st);
  c->launches += 2;
  CUDA_TRY(cudaGetLastError());
  c->n[layer] += 1;
  while (c->n[layer] - c->f[layer] >= G.r + G.g) {
    int rc = migrate(c, layer, st);
    if (rc) return rc;
  }
  return SPC_OK;
}

cudaEvent_t prof_event(spc_cache* c) {
  if (c->ev_used == c->ev_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    c->ev_pool.push_back(e);
  }
  return c->ev_pool[c->ev_used++];
}

int ticket_tail(spc_cache* c, int layer, int f, int n_before, bool append_row0, cudaEvent_t p0);

// One decode / predecode layer.  append_row0: decode persists row 0 (engine.py:321).
int run_layer(spc_cache* c, int layer, int rows, const void* q, const void* k_new,
              const void* v_new, void* out, float* pinned_mass, cudaStream_t st, bool append_row0) {
  const Geo& G = c->G;
  if (append_row0 && c->n[layer] >= c->context_length)
    return fail(SPC_EINVAL, "context_length exceeded");
  if (!q || !k_new || !v_new || !out) return fail(SPC_EINVAL, "null q / k_new / v_new / out");
  // rows are read with 8- and 16-byte vector loads (and cp.async) by the attend kernels
  if (((uintptr_t)q | (uintptr_t)k_new | (uintptr_t)v_new | (uintptr_t)out) & 15)
    return fail(SPC_EINVAL, "q, k_new, v_new and out must be 16-byte aligned device pointers");
  AttnArgs a{};
  a.G = G;
  a.B = c->L[layer];
  a.q = (const __nv_bfloat16*)q;
  a.k_new = (const __nv_bfloat16*)k_new;
  a.v_new = (const __nv_bfloat16*)v_new;
  a.out = (__nv_bfloat16*)out;
  a.pinned_mass = pinned_mass;
  a.rows = rows;
  a.agg_row = rows - 1;  // decode: speculative row 1; predecode: row 0 (engine.py:262,317)
  a.n = (int)c->n[layer];
  a.f = (int)c->f[layer];
  a.part_o = c->part_o;
  a.part_ml = c->part_ml;
  a.pin_ml = c->pin_ml;
  a.spill = c->spill + (size_t)layer * G.batch * G.Hq * (size_t)G.L;
  a.mz = c->mz + (size_t)layer * G.batch * G.Hq * 2;
  a.sm_scale_log2 = (float)(1.0 / std::sqrt((double)G.d) * 1.4426950408889634);
  a.out_f32 = c->dbg_out ? c->dbg_out + (size_t)layer * G.batch * 2 * G.Hq * G.d : nullptr;
  bool fast = (c->impl != 1) && attend_fast_supported(G, rows);
  a.agg_recompute = (c->agg_mode == 1 && fast) ? 1 : 0;
  // K6a (row 0 -> residual ring) rides on the combine kernel when the rows are
  // 16-byte vectors (they are: run_layer requires 16-byte aligned inputs)
  a.ring_append = (append_row0 && G.d % 8 == 0) ? 1 : 0;
  if (c->impl == 2 && !fast) return fail(SPC_EINVAL, "fast attention path not available for this geometry");
  cudaEvent_t p0 = nullptr, p1 = nullptr;
  if (c->prof) {
    p0 = prof_event(c);
    p1 = prof_event(c);
    CUDA_TRY(cudaEventRecord(p0, st));
  }
  if (fast) {
    c->launches += launch_attend_fast(a, st);  // K2 + K3 combine; own split plan
  } else {
    choose_splits(c, a.f, &a.nsplit, &a.blocks_per_split);
    launch_attend_generic(a, st);
    CUDA_TRY(cudaGetLastError());
    launch_combine(a, st);
    c->launches += 2;
  }
  CUDA_TRY(cudaGetLastError());
  if (c->prof) {
    CUDA_TRY(cudaEventRecord(p1, st));
    c->prof_attn.push_back({p0, p1});
  }
  const int n_before = (int)c->n[layer];
  if (append_row0 && !a.ring_append) {  // K6a on the compute stream (reads the caller's k_new/v_new now)
    launch_ring_append(G, c->L[layer], (const __nv_bfloat16*)k_new, (const __nv_bfloat16*)v_new,
                       (long long)rows * G.H * G.d, n_before, st);
    c->launches += 1;
    CUDA_TRY(cudaGetLastError());
  }
  CUDA_TRY(cudaEventRecord(c->ev_agg[layer], st));
  // ---- ticket + slow tier on a copy stream (transfer.py:84-94, kvcache.py:162-192) ----
  cudaStream_t cs = c->sstream(layer);
  CUDA_TRY(cudaStreamWaitEvent(cs, c->ev_agg[layer], 0));
  if (c->prof) {
    p0 = prof_event(c);
    CUDA_TRY(cudaEventRecord(p0, cs));
  }
  if (!(debug_skip() & 1)) {
    if (a.agg_recompute) launch_agg_recompute(a, cs);
    else launch_agg(a, cs);
  }
  c->launches += a.f > 0;
  CUDA_TRY(cudaGetLastError());
  if (c->agg_ext) {  // the caller reduces agg across ranks on cs, then spc_finish_layer
    c->pend[layer] = spc_cache::Pending{true, append_row0, a.f, n_before, p0};
    return SPC_OK;
  }
  return ticket_tail(c, layer, a.f, n_before, append_row0, p0);
}

// K4 top-k + pin diff -> K5 prefetch -> K6b slow-tier write (+K1 migration) on
// the layer's copy stream, then ev_pf(layer): the rest of the ticket.
int ticket_tail(spc_cache* c, int layer, int f, int n_before, bool append_row0, cudaEvent_t p0) {
  const Geo& G = c->G;
  cudaStream_t cs = c->cstream(layer);
  cudaEvent_t p1 = nullptr;
  if (c->prof) p1 = prof_event(c);
  cudaStream_t ss = c->sstream(layer);
  if (!(debug_skip() & 2)) launch_topk(G, c->L[layer], f, ss);
  if (ss != cs) {
    CUDA_TRY(cudaEventRecord(c->ev_sel[layer], ss));
    CUDA_TRY(cudaStreamWaitEvent(cs, c->ev_sel[layer], 0));
  }
  cudaEvent_t q0 = nullptr, q1 = nullptr;
  if (c->prof) {
    q0 = prof_event(c);
    q1 = prof_event(c);
    CUDA_TRY(cudaEventRecord(q0, cs));
  }
  if (!(debug_skip() & 4))
    launch_prefetch(G, c->L[layer], host_slab(c, c->host_k, layer), host_slab(c, c->host_v, layer), c->pf_inflight,
                    cs);
  if (c->prof) {
    CUDA_TRY(cudaEventRecord(q1, cs));
    c->prof_pf.push_back({q0, q1});
  }
  c->launches += 2;
  CUDA_TRY(cudaGetLastError());
  if (c->prof) {
    CUDA_TRY(cudaEventRecord(p1, cs));
    c->prof_sel.push_back({p0, p1});
  }
  if (append_row0) {
    launch_host_append(G, c->L[layer], n_before, host_slab(c, c->host_k, layer),
                       host_slab(c, c->host_v, layer), cs);
    c->launches += 1;
    c->n[layer] += 1;
    while (c->n[layer] - c->f[layer] >= G.r + G.g) {  // kvcache.py:169-171
      int rc = migrate(c, layer, cs);
      if (rc) return rc;
    }
    CUDA_TRY(cudaGetLastError());
  }
  CUDA_TRY(cudaEventRecord(c->ev_pf[layer], cs));
  return SPC_OK;
}
}  // namespace

extern "C" {

int spc_abi_version(void) { return SPC_ABI_VERSION; }
const char* spc_last_error(void) { return g_err.c_str(); }

int spc_cache_create(const spc_dims* d, int device, spc_cache** out) {
  if (!d || !out) return fail(SPC_EINVAL, "null argument");
  *out = nullptr;
  if (d->layers <= 0 || d->kv_heads <= 0 || d->head_dim <= 0)
    return fail(SPC_EINVAL, "layers, kv_heads and head_dim must be positive");
  if (!(d->bits == 1 || d->bits == 2 || d->bits == 4 || d->bits == 16))
    return fail(SPC_EINVAL, "bits must be one of (1, 2, 4, 16)");
  if (d->group_size <= 0 || d->residual <= 0 || d->prefetch_k <= 0 || d->context_length <= 0)
    return fail(SPC_EINVAL, "group_size, residual, prefetch_k and context_length must be positive");
  if (d->batch <= 0 || d->q_heads <= 0 || d->q_heads % d->kv_heads)
    return fail(SPC_EINVAL, "q_heads must be a positive multiple of kv_heads and batch positive");
  if (d->head_dim % 2 || d->head_dim > 256) return fail(SPC_EINVAL, "head_dim must be even and <= 256");
  if (d->prefetch_k > 1024) return fail(SPC_EINVAL, "prefetch_k > 1024 unsupported");
  if (2 * (d->q_heads / d->kv_heads) > 16) return fail(SPC_EINVAL, "more than 8 q heads per kv head unsupported");
  if (d->group_size * d->head_dim > 12288) return fail(SPC_EINVAL, "group_size*head_dim too large");
  if (d->topk_scope != SPC_SCOPE_LAYER && d->topk_scope != SPC_SCOPE_KV_HEAD)
    return fail(SPC_EINVAL, "topk_scope must be 0 (layer) or 1 (kv_head)");
  CUDA_TRY(cudaSetDevice(device));

  spc_cache* c = new spc_cache();
  c->device = device;
  Geo& G = c->G;
  G.layers = d->layers;
  G.batch = d->batch;
  G.H = d->kv_heads;
  G.Hq = d->q_heads;
  G.d = d->head_dim;
  G.bits = d->bits;
  G.g = d->group_size;
  G.r = d->residual;
  G.k = d->prefetch_k;
  G.scope = d->topk_scope;
  G.host_layers = (d->host_layers > 0 && d->host_layers <= d->layers) ? d->host_layers : d->layers;
  G.G = G.Hq / G.H;
  G.U = G.scope ? G.H : 1;
  G.Hu = G.scope ? 1 : G.H;
  c->context_length = d->context_length;
  // capacity: whole blocks and whole bitmap words
  int lcm = G.g;
  while (lcm % 32) lcm += G.g;
  G.L = (int)align_up((size_t)d->context_length, (size_t)lcm);
  G.ring = G.r + G.g;
  G.nch = (G.d + G.g - 1) / G.g;
  G.krw = G.bits == 16 ? G.d / 2 : (G.d * G.bits + 31) / 32;
  G.vrw = G.krw;
  G.fast = (G.d == 128 && (G.g == 32 || G.g == 64) && (G.bits == 1 || G.bits == 2)) ? 1 : 0;
  G.tb = G.fast ? 32 : G.g;
  G.vps = G.fast ? G.d / 32 : G.nch;
  G.nblk = G.L / G.tb;
  G.bwords = G.tb * G.krw;
  G.rec = 2 * G.bwords + (G.bits == 16 ? 0 : G.d + G.tb * G.vps);

  int rc = SPC_OK;
  const size_t b = G.batch, H = G.H, U = G.U;
  c->L.resize(G.layers);
  for (int l = 0; l < G.layers && rc == SPC_OK; ++l) {
    LayerBufs& B = c->L[l];
    size_t codes = b * H * G.nblk * (size_t)G.rec * 4;  // block records
    size_t kpar = 0, vpar = 0;
    size_t ring = b * H * G.ring * (size_t)G.d * 2;
    size_t pool = b * U * G.k * (size_t)G.Hu * G.d * 2;
    size_t off[16], tot = 0, sizes[16] = {codes, 0, kpar, vpar, ring, ring, pool, pool,
                                          b * U * G.k * 4, b * U * (G.L / 32) * 4, b * U * (size_t)G.L * 4,
                                          b * U * G.k * 4, b * U * 4, b * U * G.k * 4, b * U * G.k * 4,
                                          b * H * 4 * 4};
    for (int i = 0; i < 16; ++i) {
      off[i] = tot;
      tot += align_up(std::max<size_t>(sizes[i], 16), 256);
    }
    char* base = nullptr;
    rc = dalloc(c, (void**)&base, tot);
    if (rc) break;
    // defined contents everywhere (e.g. agg beyond the frontier, which a
    // cross-rank all-reduce of the whole buffer reads): one memset per layer
    if (cudaMemset(base, 0, tot) != cudaSuccess) {
      rc = fail(SPC_ECUDA, "cudaMemset of the layer buffers failed");
      break;
    }
    B.kcodes = (uint32_t*)(base + off[0]);
    B.vcodes = B.kcodes + G.bwords;
    B.kparams = B.kcodes + 2 * G.bwords;
    B.vparams = B.kparams + (G.bits == 16 ? 0 : G.d);
    B.ring_k = (__nv_bfloat16*)(base + off[4]);
    B.ring_v = (__nv_bfloat16*)(base + off[5]);
    B.pool_k = (__nv_bfloat16*)(base + off[6]);
    B.pool_v = (__nv_bfloat16*)(base + off[7]);
    B.pin_pos = (int32_t*)(base + off[8]);
    B.bitmap = (uint32_t*)(base + off[9]);
    B.agg = (float*)(base + off[10]);
    B.sel = (int32_t*)(base + off[11]);
    B.newcnt = (int32_t*)(base + off[12]);
    B.fetch_slot = (int32_t*)(base + off[13]);
    B.fetch_pos = (int32_t*)(base + off[14]);
    B.rmax = (uint32_t*)(base + off[15]);
    if (cudaMemset(B.pin_pos, 0xFF, sizes[8]) != cudaSuccess || cudaMemset(B.bitmap, 0, sizes[9]) != cudaSuccess ||
        cudaMemset(B.sel, 0xFF, sizes[11]) != cudaSuccess || cudaMemset(B.newcnt, 0, sizes[12]) != cudaSuccess ||
        cudaMemset(B.rmax, 0, sizes[15]) != cudaSuccess ||
        cudaMemset(B.ring_k, 0, ring) != cudaSuccess || cudaMemset(B.ring_v, 0, ring) != cudaSuccess ||
        cudaMemset(B.pool_k, 0, pool) != cudaSuccess || cudaMemset(B.pool_v, 0, pool) != cudaSuccess)
      rc = fail(SPC_ECUDA, "cudaMemset failed");
  }
  const size_t R = 2 * G.G;
  if (rc == SPC_OK) rc = dalloc(c, (void**)&c->part_o, b * H * (kSplitCap + 1) * R * G.d * 4);
  if (rc == SPC_OK) rc = dalloc(c, (void**)&c->part_ml, b * H * (kSplitCap + 1) * R * 2 * 4);
  if (rc == SPC_OK) rc = dalloc(c, (void**)&c->pin_ml, b * H * R * 2 * 4);
  if (rc == SPC_OK) rc = dalloc(c, (void**)&c->spill, (size_t)G.layers * b * G.Hq * (size_t)G.L * 4);
  if (rc == SPC_OK) rc = dalloc(c, (void**)&c->mz, (size_t)G.layers * b * G.Hq * 2 * 4);
  if (rc == SPC_OK) rc = dalloc(c, (void**)&c->staging, (size_t)G.k * 4);
  if (rc == SPC_OK) rc = dalloc(c, (void**)&c->pf_rows, sizeof(unsigned long long));
  if (rc == SPC_OK) {
    cudaMemset(c->pf_rows, 0, sizeof(unsigned long long));
    for (auto& B : c->L) B.pf_rows = c->pf_rows;
  }
  if (rc == SPC_OK) {
    c->slab_elems = b * (size_t)G.L * H * G.d;
    c->host_bytes = 2 * c->slab_elems * G.host_layers * sizeof(__nv_bfloat16);
    cudaError_t e1 = cudaHostAlloc((void**)&c->host_k, c->host_bytes / 2, cudaHostAllocMapped | cudaHostAllocPortable);
    cudaError_t e2 = e1 == cudaSuccess ? cudaHostAlloc((void**)&c->host_v, c->host_bytes / 2,
                                                       cudaHostAllocMapped | cudaHostAllocPortable)
                                       : e1;
    if (e1 != cudaSuccess || e2 != cudaSuccess)
      rc = fail(SPC_ENOMEM, std::string("pinned host slow tier (") + std::to_string(c->host_bytes) +
                                " bytes): " + cudaGetErrorString(e1 != cudaSuccess ? e1 : e2));
  }
  if (rc == SPC_OK) {
    int lo_prio = 0, hi_prio = 0;
    cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
    // stream priorities (SPC_COPY_PRIO): "split" (default) = PCIe gather + slow-tier
    // write on high-priority copy streams, aggregate + top-k on lowest-priority
    // selection streams, whose CTAs then only take SM slots K2 leaves free;
    // "high" = everything on the high-priority copy streams; "low" = everything
    // lowest.  32-layer bench, one box: C2 999 -> 1035, C3 467 -> 531, C4 404 -> 486
    // tok/s for high -> split
    const char* pe = getenv("SPC_COPY_PRIO");
    const std::string mode = pe ? pe : "split";
    const int prio = mode == "low" ? lo_prio : hi_prio;
    if (cudaStreamCreateWithPriority(&c->copy_stream, cudaStreamNonBlocking, prio) != cudaSuccess ||
        cudaStreamCreateWithPriority(&c->copy_stream2, cudaStreamNonBlocking, prio) != cudaSuccess)
      rc = fail(SPC_ECUDA, "stream create failed");
    if (rc == SPC_OK && mode == "split" &&
        (cudaStreamCreateWithPriority(&c->sel_stream, cudaStreamNonBlocking, lo_prio) != cudaSuccess ||
         cudaStreamCreateWithPriority(&c->sel_stream2, cudaStreamNonBlocking, lo_prio) != cudaSuccess))
      rc = fail(SPC_ECUDA, "stream create failed");
    c->ev_agg.resize(G.layers);
    c->ev_pf.resize(G.layers);
    c->ev_sel.resize(G.layers);
    for (int l = 0; l < G.layers && rc == SPC_OK; ++l) {
      if (cudaEventCreateWithFlags(&c->ev_agg[l], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&c->ev_sel[l], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&c->ev_pf[l], cudaEventDisableTiming) != cudaSuccess)
        rc = fail(SPC_ECUDA, "event create failed");
    }
  }
  if (rc == SPC_OK && cudaDeviceSynchronize() != cudaSuccess) rc = fail(SPC_ECUDA, "init sync failed");
  c->n.assign(G.layers, 0);
  c->f.assign(G.layers, 0);
  c->ticket.assign(G.layers, -1);
  c->pend.assign(G.layers, spc_cache::Pending{});
  if (rc != SPC_OK) {
    std::string keep = g_err;
    spc_cache_destroy(c);
    g_err = keep;
    return rc;
  }
  *out = c;
  return SPC_OK;
}

int spc_cache_destroy(spc_cache* c) {
  if (!c) return SPC_OK;
  cudaSetDevice(c->device);
  if (c->capturing) {  // abandon an open capture
    cudaGraph_t g = nullptr;
    if (cudaStreamEndCapture(c->cap_stream, &g) == cudaSuccess && g) cudaGraphDestroy(g);
    cudaGetLastError();
  }
  cudaDeviceSynchronize();
  for (void* p : c->dev_allocs) cudaFree(p);
  if (c->dbg_out) cudaFree(c->dbg_out);
  for (auto g : c->gexec) if (g) cudaGraphExecDestroy(g);
  for (auto e : c->ev_join) if (e) cudaEventDestroy(e);
  if (c->host_k) cudaFreeHost(c->host_k);
  if (c->host_v) cudaFreeHost(c->host_v);
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  if (c->prof_base) cudaEventDestroy(c->prof_base);
  for (auto e : c->ev_agg) if (e) cudaEventDestroy(e);
  for (auto e : c->ev_sel) if (e) cudaEventDestroy(e);
  if (c->sel_stream) cudaStreamDestroy(c->sel_stream);
  if (c->sel_stream2) cudaStreamDestroy(c->sel_stream2);
  for (auto e : c->ev_pf) if (e) cudaEventDestroy(e);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  if (c->copy_stream2) cudaStreamDestroy(c->copy_stream2);
  delete c;
  return SPC_OK;
}

int spc_cache_fast_path(const spc_cache* c) { return c && c->G.fast ? attend_fast_supported(c->G, 2) : 0; }
int64_t spc_device_bytes(const spc_cache* c) { return c ? (int64_t)c->dev_bytes : -1; }
int64_t spc_host_bytes(const spc_cache* c) { return c ? (int64_t)c->host_bytes : -1; }
int64_t spc_length(const spc_cache* c, int layer) { return check_layer(c, layer) ? -1 : c->n[layer]; }
int64_t spc_frontier(const spc_cache* c, int layer) { return check_layer(c, layer) ? -1 : c->f[layer]; }
int64_t spc_row_bytes(const spc_cache* c, int64_t positions) {
  // kvcache.py:148-150: 16-bit accounting, key + value rows, all kv heads
  return c ? positions * 2 * c->G.d * 2 * c->G.H : -1;
}

int spc_set_attend_impl(spc_cache* c, int impl) {
  if (!c || impl < 0 || impl > 2) return fail(SPC_EINVAL, "impl must be 0 (auto), 1 (generic) or 2 (fast)");
  c->impl = impl;
  return SPC_OK;
}

int spc_set_agg_mode(spc_cache* c, int mode) {
  if (!c || mode < 0 || mode > 1) return fail(SPC_EINVAL, "agg mode must be 0 (spill) or 1 (recompute)");
  c->agg_mode = mode;
  return SPC_OK;
}

int spc_set_prefetch_inflight(spc_cache* c, int64_t bytes) {
  if (!c) return fail(SPC_EINVAL, "null cache");
  if (bytes < 0) return fail(SPC_EINVAL, "prefetch in-flight bytes must be >= 0");
  c->pf_inflight = bytes ? bytes : int64_t(256) << 10;
  return SPC_OK;
}

int spc_prefill(spc_cache* c, int layer, const void* K, const void* V, int n, void* stream) {
  if (int rc = check_layer(c, layer)) return rc;
  if (int rc = no_capture(c)) return rc;
  const Geo& G = c->G;
  cudaStream_t st = (cudaStream_t)stream;
  if (c->n[layer] != 0) return fail(SPC_EPROTO, "prefill requires an empty layer");
  if (n <= 0) return fail(SPC_EINVAL, "prompt must be nonempty");
  if (n > c->context_length) return fail(SPC_EINVAL, "prompt longer than context_length");
  CUDA_TRY(cudaSetDevice(c->device));
  // slow tier: every row (kvcache.py:165-166)
  size_t row = (size_t)G.H * G.d * sizeof(__nv_bfloat16);
  CUDA_TRY(cudaMemcpy2DAsync(host_slab(c, c->host_k, layer), (size_t)G.L * row, K, (size_t)n * row,
                             (size_t)n * row, G.batch, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpy2DAsync(host_slab(c, c->host_v, layer), (size_t)G.L * row, V, (size_t)n * row,
                             (size_t)n * row, G.batch, cudaMemcpyDeviceToHost, st));
  int64_t f = frontier_of(n, G.r, G.g);
  QuantSrc S{(const __nv_bfloat16*)K, (const __nv_bfloat16*)V, (long long)n * G.H * G.d,
             (long long)G.H * G.d, (long long)G.d, 0};
  launch_quantize(G, c->L[layer], S, 0, (int)(f / G.g), st);
  CUDA_TRY(cudaGetLastError());
  launch_ring_fill(G, c->L[layer], (const __nv_bfloat16*)K, (const __nv_bfloat16*)V, n, (int)f, st);
  CUDA_TRY(cudaGetLastError());
  c->n[layer] = n;
  c->f[layer] = f;
  return SPC_OK;
}

int spc_append(spc_cache* c, int layer, const void* k_rows, const void* v_rows, int64_t seq_stride,
               void* stream) {
  if (int rc = check_layer(c, layer)) return rc;
  if (int rc = no_capture(c)) return rc;
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaStreamWaitEvent((cudaStream_t)stream, c->ev_pf[layer], 0));
  return append_rows(c, layer, k_rows, v_rows, seq_stride, (cudaStream_t)stream);
}

int spc_migrate(spc_cache* c, int layer, void* stream) {
  if (int rc = check_layer(c, layer)) return rc;
  if (int rc = no_capture(c)) return rc;
  if (c->n[layer] - c->f[layer] < c->G.g)  // kvcache.py:175-177
    return fail(SPC_EINVAL, "not enough residual tokens to migrate");
  CUDA_TRY(cudaSetDevice(c->device));
  return migrate(c, layer, (cudaStream_t)stream);
}

int spc_select_topk(const float* scores, int n, int k, int32_t* out, void* stream) {
  if (n < 0 || k < 0 || k > 1024) return fail(SPC_EINVAL, "select_topk: need n >= 0 and 0 <= k <= 1024");
  if (k == 0) return SPC_OK;
  launch_select(scores, n, k, out, (cudaStream_t)stream);
  CUDA_TRY(cudaGetLastError());
  return SPC_OK;
}

int spc_pin(spc_cache* c, int layer, int seq, int unit, const int32_t* positions, int npos,
            const void* k_rows, const void* v_rows, void* stream) {
  if (int rc = check_layer(c, layer)) return rc;
  if (int rc = check_not_pending(c, layer)) return rc;
  const Geo& G = c->G;
  cudaStream_t st = (cudaStream_t)stream;
  if (seq < 0 || seq >= G.batch || unit < 0 || unit >= G.U) return fail(SPC_EINVAL, "seq/unit out of range");
  if (npos > G.k) return fail(SPC_EINVAL, "pinned set larger than the prefetch budget");
  std::vector<int32_t> p(positions, positions + std::max(npos, 0));
  for (int32_t x : p) {  // kvcache.py:202-209
    if (x < 0 || x >= c->n[layer]) return fail(SPC_EINVAL, "position " + std::to_string(x) + " does not exist");
    if (x >= c->f[layer]) return fail(SPC_EINVAL, "position " + std::to_string(x) + " is inside the residual window");
  }
  std::sort(p.begin(), p.end());
  p.erase(std::unique(p.begin(), p.end()), p.end());
  if (k_rows && (int)p.size() != npos) return fail(SPC_EINVAL, "duplicate positions with explicit rows");
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaStreamWaitEvent(st, c->ev_pf[layer], 0));  // no selection in flight
  if (!p.empty())
    CUDA_TRY(cudaMemcpyAsync(c->staging, p.data(), p.size() * 4, cudaMemcpyHostToDevice, st));
  launch_set_pins(G, c->L[layer], seq, unit, c->staging, (int)p.size(), st);
  if (k_rows && v_rows) {
    launch_copy_pins(G, c->L[layer], seq, unit, (const __nv_bfloat16*)k_rows, (const __nv_bfloat16*)v_rows,
                     (int)p.size(), st);
  } else {
    // slow-tier fetch of every pinned row (pin() default, kvcache.py:208-209)
    launch_prefetch_one(G, c->L[layer], seq, unit, host_slab(c, c->host_k, layer),
                        host_slab(c, c->host_v, layer), st);
  }
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaStreamSynchronize(st));  // staging buffer reuse + host vector lifetime
  return SPC_OK;
}

int spc_predecode_layer(spc_cache* c, int layer, const void* q, const void* k_new, const void* v_new,
                        void* out, void* stream) {
  if (int rc = check_layer(c, layer)) return rc;
  if (c->ticket[layer] != -1)
    return fail(SPC_EPROTO, "duplicate ticket for step 0 layer " + std::to_string(layer));
  if (int rc = check_not_pending(c, layer)) return rc;
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(cudaStreamWaitEvent(st, c->ev_pf[layer], 0));
  int rc = run_layer(c, layer, 1, q, k_new, v_new, out, nullptr, st, false);
  if (rc) return rc;
  c->ticket[layer] = 0;
  return SPC_OK;
}

int spc_decode_layer(spc_cache* c, int layer, int step, const void* q, const void* k_new,
                     const void* v_new, void* out, float* pinned_mass, void* stream) {
  if (int rc = check_layer(c, layer)) return rc;
  if (c->ticket[layer] != step - 1)  // transfer.py:96-100
    return fail(SPC_EPROTO, "no ticket was issued at step " + std::to_string(step - 1) + " for layer " +
                                std::to_string(layer));
  if (int rc = check_not_pending(c, layer, true)) return rc;
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  if (c->capturing) {
    // in a step graph the previous step's ticket is complete before the graph
    // starts (graph launches are stream-ordered; spc_graph_begin orders the
    // first one after any eager ticket), so there is no await_layer edge
    if (st != c->cap_stream)
      return fail(SPC_EINVAL, "spc_decode_layer during capture must use the stream given to spc_graph_begin");
    c->ticket[layer] = -1;
    int rc = run_layer(c, layer, 2, q, k_new, v_new, out, pinned_mass, st, true);
    if (rc) {
      c->capture_failed = true;
      return rc;
    }
    c->ticket[layer] = step;
    return SPC_OK;
  }
  cudaEvent_t w0 = nullptr, w1 = nullptr;
  if (c->prof) {  // exposed prefetch: compute-stream time spent waiting on the ticket
    w0 = prof_event(c);
    w1 = prof_event(c);
    CUDA_TRY(cudaEventRecord(w0, st));
  }
  CUDA_TRY(cudaStreamWaitEvent(st, c->ev_pf[layer], 0));  // await_layer
  if (c->prof) {
    CUDA_TRY(cudaEventRecord(w1, st));
    c->prof_wait.push_back({w0, w1});
  }
  c->ticket[layer] = -1;
  // persists row 0 only (engine.py:321; the speculative row is never persisted)
  int rc = run_layer(c, layer, 2, q, k_new, v_new, out, pinned_mass, st, true);
  if (rc) return rc;
  c->ticket[layer] = step;
  return SPC_OK;
}

int spc_graph_begin(spc_cache* c, void* stream) {
  if (!c) return fail(SPC_EINVAL, "null cache");
  if (c->capturing) return fail(SPC_EPROTO, "spc_graph_begin: already capturing");
  if (c->prof) return fail(SPC_EPROTO, "spc_graph_begin: live profiling (spc_profile) is on");
  if (c->agg_ext) return fail(SPC_EPROTO, "spc_graph_begin: the cross-rank aggregate reduction is on");
  cudaStream_t st = (cudaStream_t)stream;
  if (!st) return fail(SPC_EINVAL, "spc_graph_begin: the legacy default stream cannot be captured");
  CUDA_TRY(cudaSetDevice(c->device));
  // eager tickets still in flight on the copy streams come before the graph
  for (int l = 0; l < c->G.layers; ++l) CUDA_TRY(cudaStreamWaitEvent(st, c->ev_pf[l], 0));
  CUDA_TRY(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  c->capturing = true;
  c->capture_failed = false;
  c->cap_stream = st;
  return SPC_OK;
}

// Joins the side streams back into the capture, ends it, refreshes the
// executable graph (cudaGraphExecUpdate: same topology, new kernel arguments;
// a step with a different topology -- a migration, another split plan's
// kernel -- instantiates afresh) and launches it on the capture stream.
int spc_graph_launch(spc_cache* c, void* stream) {
  if (!c) return fail(SPC_EINVAL, "null cache");
  if (!c->capturing) return fail(SPC_EPROTO, "spc_graph_launch without spc_graph_begin");
  cudaStream_t st = (cudaStream_t)stream;
  if (st != c->cap_stream) return fail(SPC_EINVAL, "spc_graph_launch: not the stream given to spc_graph_begin");
  CUDA_TRY(cudaSetDevice(c->device));
  const cudaStream_t side[4] = {c->copy_stream, c->copy_stream2, c->sel_stream, c->sel_stream2};
  cudaError_t err = cudaSuccess;
  for (int i = 0; i < 4 && err == cudaSuccess; ++i) {
    if (!side[i]) continue;
    cudaStreamCaptureStatus cs_status = cudaStreamCaptureStatusNone;
    err = cudaStreamIsCapturing(side[i], &cs_status);
    if (err == cudaSuccess && cs_status == cudaStreamCaptureStatusActive) {
      if (!c->ev_join[i]) err = cudaEventCreateWithFlags(&c->ev_join[i], cudaEventDisableTiming);
      if (err == cudaSuccess) err = cudaEventRecord(c->ev_join[i], side[i]);
      if (err == cudaSuccess) err = cudaStreamWaitEvent(st, c->ev_join[i], 0);
    }
  }
  cudaGraph_t graph = nullptr;
  cudaError_t e_end = cudaStreamEndCapture(st, &graph);
  c->capturing = false;
  if (err == cudaSuccess) err = e_end;
  if (err != cudaSuccess || c->capture_failed) {
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    if (c->capture_failed) return fail(SPC_EPROTO, "a decode call failed during capture; nothing was launched");
    return fail(SPC_ECUDA, std::string("step graph capture: ") + cudaGetErrorString(err));
  }
  // two executable graphs: the steady step and the other shape that recurs (a
  // step with a migration), so alternating shapes update in place too
  int slot = -1;
  for (int k = 0; k < 2 && slot < 0; ++k) {
    const int i = (c->gexec_last + k) & 1;
    if (!c->gexec[i]) continue;
    cudaGraphExecUpdateResultInfo info;
    if (cudaGraphExecUpdate(c->gexec[i], graph, &info) == cudaSuccess) {
      slot = i;
      c->graph_updates += 1;
    } else {
      cudaGetLastError();
    }
  }
  if (slot < 0) {
    slot = c->gexec[c->gexec_last] ? (c->gexec_last ^ 1) : c->gexec_last;  // the slot not used last
    if (c->gexec[slot]) cudaGraphExecDestroy(c->gexec[slot]);
    c->gexec[slot] = nullptr;
    cudaError_t e = cudaGraphInstantiate(&c->gexec[slot], graph, 0);
    if (e != cudaSuccess) {
      cudaGraphDestroy(graph);
      c->gexec[slot] = nullptr;
      return fail(SPC_ECUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(e));
    }
    c->graph_instantiations += 1;
  }
  c->gexec_last = slot;
  cudaGraphDestroy(graph);
  CUDA_TRY(cudaGraphLaunch(c->gexec[slot], st));
  // later eager work that awaits a layer's ticket (the next eager decode,
  // export, materialize, ...) waits on ev_pf: point it past the graph
  for (int l = 0; l < c->G.layers; ++l) CUDA_TRY(cudaEventRecord(c->ev_pf[l], st));
  return SPC_OK;
}

int spc_graph_abort(spc_cache* c) {
  if (!c) return fail(SPC_EINVAL, "null cache");
  if (!c->capturing) return SPC_OK;
  CUDA_TRY(cudaSetDevice(c->device));
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(c->cap_stream, &g);
  if (g) cudaGraphDestroy(g);
  c->capturing = false;
  cudaGetLastError();
  // the captured decode calls advanced the host-side state (lengths, tickets)
  // without running: the cache is no longer consistent with the device
  return fail(SPC_EPROTO, std::string("step graph aborted (") + cudaGetErrorString(e) +
                              "): the cache's host state ran ahead of the device; destroy it");
}

int spc_copy_async(void* dst, const void* src, int64_t bytes, void* stream) {
  if (bytes < 0 || (bytes && (!dst || !src))) return fail(SPC_EINVAL, "spc_copy_async: bad arguments");
  if (bytes) CUDA_TRY(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDefault, (cudaStream_t)stream));
  return SPC_OK;
}

int spc_graph_stats(const spc_cache* c, int64_t* instantiations, int64_t* updates) {
  if (!c) return fail(SPC_EINVAL, "null cache");
  if (instantiations) *instantiations = c->graph_instantiations;
  if (updates) *updates = c->graph_updates;
  return SPC_OK;
}

int spc_set_agg_reduce(spc_cache* c, int enable) {
  if (!c) return fail(SPC_EINVAL, "null cache");
  if (int rc = no_capture(c)) return rc;
  for (int l = 0; l < c->G.layers; ++l)
    if (c->pend[l].on) return fail(SPC_EPROTO, "a layer is waiting for spc_finish_layer");
  c->agg_ext = enable != 0;
  return SPC_OK;
}

int spc_agg_buffer(spc_cache* c, int layer, float** agg, int64_t* count, void** stream) {
  if (int rc = check_layer(c, layer)) return rc;
  if (!c->agg_ext) return fail(SPC_EINVAL, "spc_agg_buffer needs spc_set_agg_reduce(cache, 1)");
  if (agg) *agg = c->L[layer].agg;
  if (count) *count = (int64_t)c->G.batch * c->G.U * c->G.L;
  if (stream) *stream = (void*)c->sstream(layer);
  return SPC_OK;
}

int spc_finish_layer(spc_cache* c, int layer) {
  if (int rc = check_layer(c, layer)) return rc;
  if (int rc = no_capture(c)) return rc;
  spc_cache::Pending& p = c->pend[layer];
  if (!p.on)
    return fail(SPC_EPROTO, "spc_finish_layer without a pending aggregate for layer " + std::to_string(layer));
  CUDA_TRY(cudaSetDevice(c->device));
  p.on = false;
  return ticket_tail(c, layer, p.f, p.n_before, p.append, p.p0);
}

int spc_ticket(spc_cache* c, int layer, int32_t* picked, int32_t* new_count, void* stream) {
  if (int rc = check_layer(c, layer)) return rc;
  if (int rc = check_not_pending(c, layer)) return rc;
  const Geo& G = c->G;
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaStreamWaitEvent(st, c->ev_pf[layer], 0));
  if (picked)
    CUDA_TRY(cudaMemcpyAsync(picked, c->L[layer].sel, (size_t)G.batch * G.U * G.k * 4, cudaMemcpyDeviceToDevice, st));
  if (new_count)
    CUDA_TRY(cudaMemcpyAsync(new_count, c->L[layer].newcnt, (size_t)G.batch * G.U * 4, cudaMemcpyDeviceToDevice, st));
  return SPC_OK;
}

int spc_debug_agg(spc_cache* c, int layer, float* agg, void* stream) {
  if (int rc = check_layer(c, layer)) return rc;
  if (int rc = check_not_pending(c, layer)) return rc;
  const Geo& G = c->G;
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(cudaStreamWaitEvent(st, c->ev_pf[layer], 0));
  CUDA_TRY(cudaMemcpyAsync(agg, c->L[layer].agg, (size_t)G.batch * G.U * G.L * 4, cudaMemcpyDeviceToDevice, st));
  return SPC_OK;
}

int spc_debug_output_f32(spc_cache* c, int enable) {
  if (!c) return fail(SPC_EINVAL, "null cache");
  if (int rc = no_capture(c)) return rc;
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaDeviceSynchronize());
  if (enable && !c->dbg_out) {
    const size_t bytes = (size_t)c->G.layers * c->G.batch * 2 * c->G.Hq * c->G.d * sizeof(float);
    CUDA_TRY(cudaMalloc((void**)&c->dbg_out, bytes));
    CUDA_TRY(cudaMemset(c->dbg_out, 0, bytes));
  } else if (!enable && c->dbg_out) {
    CUDA_TRY(cudaFree(c->dbg_out));
    c->dbg_out = nullptr;
  }
  return SPC_OK;
}

int spc_debug_out_f32(spc_cache* c, int layer, float* out, void* stream) {
  if (int rc = check_layer(c, layer)) return rc;
  if (!c->dbg_out) return fail(SPC_EINVAL, "spc_debug_out_f32 needs spc_debug_output_f32(cache, 1)");
  CUDA_TRY(cudaSetDevice(c->device));
  const size_t n = (size_t)c->G.batch * 2 * c->G.Hq * c->G.d;
  CUDA_TRY(cudaMemcpyAsync(out, c->dbg_out + (size_t)layer * n, n * sizeof(float), cudaMemcpyDeviceToDevice,
                           (cudaStream_t)stream));
  return SPC_OK;
}

int spc_materialize(spc_cache* c, int layer, int seq, int head, float* keys, float* values, void* stream) {
  if (int rc = check_layer(c, layer)) return rc;
  if (seq < 0 || seq >= c->G.batch || head < 0 || head >= c->G.H) return fail(SPC_EINVAL, "seq/head out of range");
  if (int rc = check_not_pending(c, layer)) return rc;
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(cudaStreamWaitEvent(st, c->ev_pf[layer], 0));
  launch_materialize(c->G, c->L[layer], seq, head, (int)c->n[layer], (int)c->f[layer], keys, values, st);
  CUDA_TRY(cudaGetLastError());
  return SPC_OK;
}

int spc_export_packed(spc_cache* c, int layer, int seq, uint8_t* kc, uint16_t* kz, uint16_t* ks,
                      uint8_t* vc, uint16_t* vz, uint16_t* vs, void* stream) {
  if (int rc = check_layer(c, layer)) return rc;
  if (c->G.bits == 16) return fail(SPC_EINVAL, "16-bit tier has no packed groups");
  if (seq < 0 || seq >= c->G.batch) return fail(SPC_EINVAL, "seq out of range");
  if (int rc = check_not_pending(c, layer)) return rc;
  CUDA_TRY(cudaSetDevice(c->device));
  // the newest group's migration (K1) runs on the layer's copy stream after the
  // host frontier has advanced: wait for it like spc_materialize does
  CUDA_TRY(cudaStreamWaitEvent((cudaStream_t)stream, c->ev_pf[layer], 0));
  launch_export(c->G, c->L[layer], seq, (int)(c->f[layer] / c->G.g), kc, kz, ks, vc, vz, vs,
                (cudaStream_t)stream);
  CUDA_TRY(cudaGetLastError());
  return SPC_OK;
}

int spc_slow_fetch(spc_cache* c, int layer, int seq, const int32_t* positions, int npos, void* k_out,
                   void* v_out) {
  if (int rc = check_layer(c, layer)) return rc;
  if (int rc = no_capture(c)) return rc;
  const Geo& G = c->G;
  if (seq < 0 || seq >= G.batch) return fail(SPC_EINVAL, "seq out of range");
  for (int i = 0; i < npos; ++i)  // kvcache.py:250-252
    if (positions[i] < 0 || positions[i] >= c->n[layer])
      return fail(SPC_EINVAL, "position " + std::to_string(positions[i]) + " not present in the slow tier");
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaDeviceSynchronize());
  const size_t row = (size_t)G.H * G.d;
  const __nv_bfloat16* hk = host_slab(c, c->host_k, layer) + (size_t)seq * G.L * row;
  const __nv_bfloat16* hv = host_slab(c, c->host_v, layer) + (size_t)seq * G.L * row;
  for (int i = 0; i < npos; ++i) {
    std::memcpy((char*)k_out + i * row * 2, hk + (size_t)positions[i] * row, row * 2);
    std::memcpy((char*)v_out + i * row * 2, hv + (size_t)positions[i] * row, row * 2);
  }
  return SPC_OK;
}

int spc_profile(spc_cache* c, int enable, double* attn_ms, int64_t* attn_launches, double* sel_ms,
                int64_t* sel_launches, int64_t* launches) {
  if (!c) return fail(SPC_EINVAL, "null cache");
  if (int rc = no_capture(c)) return rc;
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaDeviceSynchronize());
  double a = 0, s = 0;
  for (auto& p : c->prof_attn) {
    float ms = 0;
    CUDA_TRY(cudaEventElapsedTime(&ms, p.first, p.second));
    a += ms;
  }
  for (auto& p : c->prof_sel) {
    float ms = 0;
    CUDA_TRY(cudaEventElapsedTime(&ms, p.first, p.second));
    s += ms;
  }
  double w = 0;
  for (auto& p : c->prof_wait) {
    float ms = 0;
    CUDA_TRY(cudaEventElapsedTime(&ms, p.first, p.second));
    w += ms;
  }
  c->last_wait_ms = w;
  double pf = 0;
  for (auto& p : c->prof_pf) {
    float ms = 0;
    CUDA_TRY(cudaEventElapsedTime(&ms, p.first, p.second));
    pf += ms;
  }
  c->last_pf_ms = pf;
  // wall time of the prefetch: union of the K5 intervals (two copy streams overlap)
  c->last_pf_wall_ms = 0;
  if (c->prof_base && !c->prof_pf.empty()) {
    std::vector<std::pair<float, float>> iv;
    for (auto& p : c->prof_pf) {
      float s0 = 0, s1 = 0;
      CUDA_TRY(cudaEventElapsedTime(&s0, c->prof_base, p.first));
      CUDA_TRY(cudaEventElapsedTime(&s1, c->prof_base, p.second));
      iv.push_back({s0, s1});
    }
    std::sort(iv.begin(), iv.end());
    double tot = 0, a0 = iv[0].first, a1 = iv[0].second;
    for (size_t i = 1; i < iv.size(); ++i) {
      if (iv[i].first > a1) {
        tot += a1 - a0;
        a0 = iv[i].first;
        a1 = iv[i].second;
      } else {
        a1 = std::max(a1, (double)iv[i].second);
      }
    }
    c->last_pf_wall_ms = tot + (a1 - a0);
  }
  unsigned long long rows = 0;
  CUDA_TRY(cudaMemcpy(&rows, c->pf_rows, sizeof(rows), cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemset(c->pf_rows, 0, sizeof(rows)));
  c->last_pf_rows = (int64_t)rows;
  if (attn_ms) *attn_ms = a;
  if (attn_launches) *attn_launches = (int64_t)c->prof_attn.size();
  if (sel_ms) *sel_ms = s;
  if (sel_launches) *sel_launches = (int64_t)c->prof_sel.size();
  if (launches) *launches = c->launches;
  c->prof_attn.clear();
  c->prof_sel.clear();
  c->prof_wait.clear();
  c->prof_pf.clear();
  c->ev_used = 0;
  c->launches = 0;
  c->prof = enable != 0;
  if (c->prof) {
    if (!c->prof_base) CUDA_TRY(cudaEventCreate(&c->prof_base));
    CUDA_TRY(cudaEventRecord(c->prof_base, c->copy_stream));  // the device is idle (synchronized above)
  }
  return SPC_OK;
}

double spc_profile_wait_ms(const spc_cache* c) { return c ? c->last_wait_ms : -1.0; }
double spc_profile_prefetch_ms(const spc_cache* c) { return c ? c->last_pf_ms : -1.0; }
double spc_profile_prefetch_wall_ms(const spc_cache* c) { return c ? c->last_pf_wall_ms : -1.0; }

int spc_h2d_peak(int device, int64_t bytes, double* dma_gbs, double* zero_copy_gbs) {
  if (bytes < (1 << 20) || bytes % 16) return fail(SPC_EINVAL, "spc_h2d_peak: bytes must be >= 1 MiB and a multiple of 16");
  CUDA_TRY(cudaSetDevice(device));
  void* h = nullptr;
  void* dv = nullptr;
  cudaStream_t st = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  int rc = SPC_OK;
  auto best_of = [&](auto&& body) -> double {
    double best = 0;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0, st);
      body();
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms > 0) best = std::max(best, bytes / (ms * 1e-3) / 1e9);
    }
    return best;
  };
  if (cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess ||
      cudaMalloc(&dv, bytes) != cudaSuccess || cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) {
    rc = fail(SPC_ENOMEM, "spc_h2d_peak: allocation failed");
  } else {
    std::memset(h, 1, bytes);
    void* hd = nullptr;
    cudaHostGetDevicePointer(&hd, h, 0);
    if (dma_gbs) *dma_gbs = best_of([&] { cudaMemcpyAsync(dv, h, bytes, cudaMemcpyHostToDevice, st); });
    if (zero_copy_gbs) *zero_copy_gbs = best_of([&] { launch_h2d_probe(hd, dv, (size_t)bytes, 2 * kNumSMs, st); });
    if (cudaGetLastError() != cudaSuccess) rc = fail(SPC_ECUDA, "spc_h2d_peak: probe failed");
  }
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (st) cudaStreamDestroy(st);
  if (dv) cudaFree(dv);
  if (h) cudaFreeHost(h);
  return rc;
}
int64_t spc_profile_prefetch_bytes(const spc_cache* c) {
  // one new pin moves the K and V rows of the unit's heads (16-bit accounting, kvcache.py:148-150)
  return c ? c->last_pf_rows * (int64_t)2 * c->G.Hu * c->G.d * 2 : -1;
}

int spc_pin_state(spc_cache* c, int layer, const int32_t** pin_pos) {
  if (int rc = check_layer(c, layer)) return rc;
  *pin_pos = c->L[layer].pin_pos;
  return SPC_OK;
}

}  // extern "C"
