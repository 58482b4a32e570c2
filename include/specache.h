/*
 * specache.h -- C ABI of the B200-native SpeCache decode hot path.
 *
 * The reference (SpeCache, arXiv 2503.16163; /root/reference/pkg/src/speckv)
 * has no FFI: its boundary is the Python object API of TwoTierCache and the
 * per-layer body of SpeculativeDecoder.  Each entry point below replaces one
 * piece of that API (file:line relative to pkg/src/speckv).  Plain pointers
 * and sizes only: device pointers are CUDA device addresses, `stream` is a
 * cudaStream_t passed as void*.  No exceptions cross this boundary; every
 * function returns an spc_status (0 = ok).  The Python binding
 * (paper_2503_16163_b200/_lib.py) maps SPC_EINVAL -> ValueError and
 * SPC_EPROTO -> ProtocolError, matching the reference's error convention
 * (kvcache.py:40-44,156-157,202-209; transfer.py:31-32,86-87,98-99).
 *
 * Data types: rows / queries / outputs are bf16 (uint16 bit patterns),
 * accumulation is fp32, quantizer parameters are exact fp64 functions of the
 * group's bf16 (min, max) which the cache stores.
 */
#ifndef SPECACHE_H_
#define SPECACHE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPC_ABI_VERSION 1

#if defined(__GNUC__)
#define SPC_API __attribute__((visibility("default")))
#else
#define SPC_API
#endif

typedef enum spc_status {
  SPC_OK = 0,
  SPC_EINVAL = -22,  /* ValueError in the reference                          */
  SPC_EPROTO = -71,  /* ProtocolError (phase / ticket misuse)                 */
  SPC_ENOMEM = -12,  /* device or pinned-host allocation failed               */
  SPC_ECUDA = -5     /* CUDA runtime error (message in spc_last_error())      */
} spc_status;

typedef enum spc_topk_scope {
  SPC_SCOPE_LAYER = 0,   /* reference: one set per (seq, layer), agg over all q heads (engine.py:317) */
  SPC_SCOPE_KV_HEAD = 1  /* north-star extension: one set per (seq, layer, kv head)                    */
} spc_topk_scope;

/* Cache geometry; replaces CacheBudget (kvcache.py:29-44) + the TwoTierCache
 * constructor arguments (kvcache.py:116-118), batched over `batch` sequences
 * that advance in lockstep. */
typedef struct spc_dims {
  int32_t layers;
  int32_t batch;
  int32_t kv_heads;
  int32_t q_heads;
  int32_t head_dim;
  int32_t bits;            /* 1, 2, 4 or 16 (kvcache.py:25-26)               */
  int32_t group_size;      /* g                                              */
  int32_t residual;        /* r                                              */
  int32_t prefetch_k;      /* k                                              */
  int32_t context_length;  /* L: per-sequence capacity in positions          */
  int32_t topk_scope;      /* spc_topk_scope                                 */
  int32_t host_layers;     /* distinct pinned-host slow-tier slabs; layer l uses
                              slab l % host_layers (0 -> layers).  Aliased layers
                              must be fed identical KV.                       */
} spc_dims;

typedef struct spc_cache spc_cache;

/* -- library -------------------------------------------------------------- */
SPC_API int spc_abi_version(void);
/* Message for the last non-OK status on this thread. */
SPC_API const char* spc_last_error(void);

/* -- construction: TwoTierCache.__init__ (kvcache.py:116-129) --------------- */
SPC_API int spc_cache_create(const spc_dims* dims, int device, spc_cache** out);
SPC_API int spc_cache_destroy(spc_cache* cache);
/* 1 when the tensor-core fast path serves this geometry (d=128, g=32, bits 1/2). */
SPC_API int spc_cache_fast_path(const spc_cache* cache);
/* Attention implementation: 0 auto (fast when supported), 1 generic exact, 2 fast (error if unsupported). */
SPC_API int spc_set_attend_impl(spc_cache* cache, int impl);
/* K5 (PCIe prefetch gather) sysmem bytes kept in flight, summed over the
 * batch (0 -> default 256 KiB).  Enough to cover PCIe's bandwidth-delay
 * product; more only queues in the memory system and slows concurrent kernels
 * (a full decoder step with GEMMs prefers 128 KiB). */
SPC_API int spc_set_prefetch_inflight(spc_cache* cache, int64_t bytes);
SPC_API int64_t spc_device_bytes(const spc_cache* cache);
SPC_API int64_t spc_host_bytes(const spc_cache* cache);

/* -- bookkeeping: length / quantized_frontier / row_bytes (kvcache.py:133-150) */
SPC_API int64_t spc_length(const spc_cache* cache, int layer);
SPC_API int64_t spc_frontier(const spc_cache* cache, int layer);
SPC_API int64_t spc_row_bytes(const spc_cache* cache, int64_t positions);

/* -- writes ----------------------------------------------------------------- */
/* Bulk prefill of an empty layer: equivalent to n x append_verified
 * (kvcache.py:162-171, called at engine.py:234-235).  K, V: device bf16
 * [batch][n][kv_heads][head_dim].  Writes the slow tier (pinned host),
 * quantizes [0, f(n)) and stores the residual window [f(n), n). */
SPC_API int spc_prefill(spc_cache* cache, int layer, const void* K, const void* V, int n, void* stream);
/* append_verified (kvcache.py:162-171): one row per sequence.  k_rows, v_rows:
 * device bf16 [batch][kv_heads][head_dim] at element stride `seq_stride`
 * between sequences (0 -> kv_heads*head_dim).  Migrates when the residual
 * reaches r+g (migrate_residual, kvcache.py:173-192). */
SPC_API int spc_append(spc_cache* cache, int layer, const void* k_rows, const void* v_rows,
               int64_t seq_stride, void* stream);
/* migrate_residual (kvcache.py:173-192): quantize the oldest g residual rows;
 * SPC_EINVAL when fewer than g are resident. */
SPC_API int spc_migrate(spc_cache* cache, int layer, void* stream);
/* pin (kvcache.py:194-218) for one (seq, unit): replaces the pinned set.
 * positions: HOST int32 [npos]; rows default to a slow-tier fetch when
 * k_rows/v_rows are NULL, else device bf16 [npos][heads_per_unit][head_dim]. */
SPC_API int spc_pin(spc_cache* cache, int layer, int seq, int unit, const int32_t* positions,
            int npos, const void* k_rows, const void* v_rows, void* stream);

/* -- the hot path ------------------------------------------------------------ */
/* q, k_new, v_new and out of both calls must be 16-byte aligned device
 * pointers (vector loads / cp.async); SPC_EINVAL otherwise. */
/* Pre-decoding (engine.py:245-268): q device bf16 [batch][1][q_heads][d],
 * k_new/v_new [batch][1][kv_heads][d].  out: device bf16 [batch][1][q_heads][d].
 * Issues ticket (step 0, layer) -- top-k + prefetch on the cache's copy stream. */
SPC_API int spc_predecode_layer(spc_cache* cache, int layer, const void* q, const void* k_new,
                        const void* v_new, void* out, void* stream);
/* Dual-token decode step, one layer (engine.py:299-321): awaits ticket
 * (step-1, layer) (transfer.py:96-100 -> cudaStreamWaitEvent), attends rows
 * 0 (verified) and 1 (speculative) over packed + pinned + residual + in-step
 * rows, writes out [batch][2][q_heads][d] bf16 and pinned_mass [batch][q_heads]
 * fp32 (device), issues ticket (step, layer) and appends row 0. */
SPC_API int spc_decode_layer(spc_cache* cache, int layer, int step, const void* q, const void* k_new,
                     const void* v_new, void* out, float* pinned_mass, void* stream);
/* Step graphs (no reference counterpart: the launch side of engine.py:286-339's
 * per-step layer loop).  spc_graph_begin starts capturing `stream`; the
 * spc_decode_layer calls that follow (same stream; no other entry point until
 * spc_graph_launch, SPC_EPROTO otherwise) are recorded with their copy- and
 * selection-stream work instead of launched; spc_graph_launch joins those
 * streams, refreshes the cache's executable graph with the new kernel
 * arguments (cudaGraphExecUpdate; a step of another shape -- a migration, a
 * different split plan -- is instantiated afresh) and launches it on `stream`.
 * Results equal the eager calls'.  Not with spc_profile on or with
 * spc_set_agg_reduce(c, 1). */
SPC_API int spc_graph_begin(spc_cache* cache, void* stream);
SPC_API int spc_graph_launch(spc_cache* cache, void* stream);
/* Ends an open capture without launching.  The decode calls already captured
 * have advanced the cache's lengths and tickets, so it returns SPC_EPROTO and
 * the cache must be destroyed. */
SPC_API int spc_graph_abort(spc_cache* cache);
/* A step's host I/O (the engine's inputs in, outputs out): cudaMemcpyAsync
 * of `bytes`, direction from the pointers (pinned host or device), on
 * `stream`; inside a step graph it is captured with the decode calls. */
SPC_API int spc_copy_async(void* dst, const void* src, int64_t bytes, void* stream);
/* Instantiations and in-place updates of the step graph so far. */
SPC_API int spc_graph_stats(const spc_cache* cache, int64_t* instantiations, int64_t* updates);
/* The last ticket of `layer` (PrefetchTicket, transfer.py:50-55): picked
 * positions device int32 [batch][units][k] (-1 padded, ascending) and new-pin
 * counts device int32 [batch][units].  Ordered after the selection on `stream`. */
SPC_API int spc_ticket(spc_cache* cache, int layer, int32_t* picked, int32_t* new_count, void* stream);
/* select_topk (engine.py:75-84) over eligible [0, n): device fp32 scores (>= 0),
 * device int32 out[k] ascending, -1 padded; ties to the lower position. */
SPC_API int spc_select_topk(const float* scores, int n, int k, int32_t* out, void* stream);
/* Debug: speculative-row aggregate of `layer`, device fp32 [batch][units][context_length]. */
SPC_API int spc_debug_agg(spc_cache* cache, int layer, float* agg, void* stream);
/* Debug (parity tests): when enabled, every decode / predecode layer also keeps its
 * attention output in fp32 before the bf16 rounding (the north star's tolerance
 * applies to the fp32-accumulated result; bf16 I/O adds one RN rounding). */
SPC_API int spc_debug_output_f32(spc_cache* cache, int enable);
/* The speculative-row aggregate of the top-k (engine.py:317; SURVEY hard part
 * (b)): 0 = spill (default: the attention kernel writes the speculative rows'
 * log2 logits, K3b normalises and sums them), 1 = recompute (no spill of
 * packed positions; K3r re-reads the key codes and recomputes the scores).
 * The fast path only; the exact kernel always spills. */
SPC_API int spc_set_agg_mode(spc_cache* cache, int mode);
/* Wall time (ms) of the K5 prefetch kernels of the last profiled window: the
 * union of their intervals on the two copy streams. */
SPC_API double spc_profile_prefetch_wall_ms(const spc_cache* cache);
/* Host-link roofline: best of 5 pinned host -> device transfers of `bytes`, by
 * DMA (cudaMemcpyAsync) and by a zero-copy read kernel (K5's mechanism), GB/s. */
SPC_API int spc_h2d_peak(int device, int64_t bytes, double* dma_gbs, double* zero_copy_gbs);
/* The last fp32 output of `layer`: device fp32 [batch][rows][q_heads][head_dim]
 * (rows = 1 after predecode, 2 after decode; room for 2 rows is copied). */
SPC_API int spc_debug_out_f32(spc_cache* cache, int layer, float* out, void* stream);

/* -- KV-head sharding with layer-scope top-k (collective (2)) -----
 * A rank that owns kv heads [h0, h1) of every sequence builds its cache with
 * kv_heads = h1 - h0 (q_heads likewise).  engine.py:317 sums the speculative
 * row's probabilities over ALL q heads of the layer, so the ranks' partial
 * aggregates must be summed before the top-k.  With spc_set_agg_reduce(c, 1),
 * spc_decode_layer / spc_predecode_layer stop after the partial aggregate; the
 * caller sums spc_agg_buffer's fp32 [batch][1][L] across ranks in place (e.g.
 * an NCCL all-reduce) on the returned stream (the layer's selection stream),
 * then spc_finish_layer enqueues the rest of the ticket: top-k + pin diff on
 * that stream, then the PCIe prefetch and slow-tier append on the layer's copy
 * stream (ordered by an event).  Every rank then selects the same positions.  Until
 * spc_finish_layer, the next decode/predecode, spc_ticket, spc_debug_agg and
 * spc_pin of that layer return SPC_EPROTO.  kv_head scope needs no exchange
 * and no reduction. */
SPC_API int spc_set_agg_reduce(spc_cache* cache, int enable);
/* agg: device fp32 [batch][units][L] of `layer` (count elements); stream: the
 * cudaStream_t the reduction must be enqueued on. */
SPC_API int spc_agg_buffer(spc_cache* cache, int layer, float** agg, int64_t* count, void** stream);
SPC_API int spc_finish_layer(spc_cache* cache, int layer);

/* -- reads / parity ------------------------------------------------------------ */
/* materialize (kvcache.py:222-243) for one (seq, head): device fp32 [n][d] x2,
 * bit-identical to the reference's float32 dequantization. */
SPC_API int spc_materialize(spc_cache* cache, int layer, int seq, int head, float* keys, float* values,
                    void* stream);
/* Normative fast-tier export (snapshot(), kvcache.py:270-281 / quant.py:150-160)
 * for one (layer, seq), device buffers:
 *   key_codes uint8 [f/g][H][d][nb], key_zero/key_scale fp16 bits [f/g][H][d]
 *   val_codes uint8 [f][H][nchunk][nb], val_zero/val_scale fp16 bits [f][H][nchunk]
 * nb = ceil(g*bits/8), nchunk = ceil(d/g). */
SPC_API int spc_export_packed(spc_cache* cache, int layer, int seq, uint8_t* key_codes,
                      uint16_t* key_zero, uint16_t* key_scale, uint8_t* val_codes,
                      uint16_t* val_zero, uint16_t* val_scale, void* stream);
/* slow_fetch (kvcache.py:245-259) from the pinned host tier: HOST int32
 * positions, HOST bf16 outputs [npos][kv_heads][d].  Synchronous. */
SPC_API int spc_slow_fetch(spc_cache* cache, int layer, int seq, const int32_t* positions, int npos,
                   void* k_out, void* v_out);
/* Live profiling: synchronizes, returns the CUDA-event time summed over the
 * K2 attention launches (compute stream) and the K4+K5 ticket work (copy
 * stream) recorded since the previous call, the number of recorded launches,
 * and the count of kernels the library launched; then resets and turns
 * recording on (enable=1) or off. */
SPC_API int spc_profile(spc_cache* cache, int enable, double* attn_ms, int64_t* attn_launches,
                        double* sel_ms, int64_t* sel_launches, int64_t* launches);
/* Exposed prefetch of the last spc_profile window: summed compute-stream time
 * (ms) between reaching a decode layer and its ticket's prefetch event. */
SPC_API double spc_profile_wait_ms(const spc_cache* cache);
/* K5 (PCIe prefetch gather) kernel time of the last spc_profile window (ms). */
SPC_API double spc_profile_prefetch_ms(const spc_cache* cache);
/* Bytes the K5 gathers moved over PCIe in the last spc_profile window. */
SPC_API int64_t spc_profile_prefetch_bytes(const spc_cache* cache);
/* Device pointer + element count of the pin state of (layer): pin_pos int32
 * [batch][units][k] (-1 = empty slot). */
SPC_API int spc_pin_state(spc_cache* cache, int layer, const int32_t** pin_pos);

/* -- decoder layer around the path ---------------------------
 * The elementwise pieces of the reference's decoder layer (engine.py:35-72),
 * fused; the GEMMs are plain cuBLAS bf16 GEMMs on the caller's side.  All
 * pointers are device pointers; bf16 as uint16 bit patterns. */
/* x[rows][hidden] fp32 += delta (bf16, may be NULL); out = bf16(x * gain /
 * sqrt(mean(x^2) + eps)) -- rmsnorm, numerics.py:42-51.  hidden % 8 == 0. */
SPC_API int spc_add_rmsnorm(float* x, const void* delta, const float* gain, void* out, int rows, int hidden,
                            float eps, void* stream);
/* table [rows][d/2] of fp32 (cos, sin) pairs of positions[r] * base^(-2i/d),
 * angles in fp64 -- rope_apply's angles, numerics.py:54-63.  Positions are
 * shared by all layers of a step: build once, use in every spc_qkv_rope. */
SPC_API int spc_rope_table(const int32_t* positions, int rows, int head_dim, double rope_base, float* table,
                           void* stream);
/* Split fused QKV GEMM rows [rows][(Hq + 2 Hkv) * d] into q [rows][Hq][d],
 * k, v [rows][Hkv][d], rotating q and k pairs (2i, 2i+1) by the table --
 * _qkv + rope_apply, engine.py:39-48, numerics.py:64-70. */
SPC_API int spc_qkv_rope(const void* qkv, const float* rope_table, int rows, int q_heads, int kv_heads,
                         int head_dim, void* q, void* k, void* v, void* stream);
/* g = g / (1 + exp(-g)) in place over n bf16 values (n % 8 == 0) -- _silu, engine.py:35-36. */
SPC_API int spc_silu(void* g, int64_t n, void* stream);
/* out[r] = argmax of bf16 row r, ties to the lowest index -- argmax_row, numerics.py:73-78. */
SPC_API int spc_argmax_rows(const void* x, int rows, int cols, int32_t* out, void* stream);

/* -- hit-rate study on the device -----------------------------
 * A trace row (sequence s, query step t) starts at rows + s*seq_ld + t*row_ld
 * and holds lens[t] fp32 probabilities; a sequence is one (layer, q head) of
 * AttentionTrace.sequences() (hitrate.py:23-25).  lens is a DEVICE int32
 * array of `steps` entries, max_len its maximum.  Rates are float64 and
 * bit-identical to hitrate.py on the same rows (see csrc/hitrate.cu). */
/* Exact fp32 attention of one decode step over a full cache (the full-cache
 * decoder's _attend, engine.py:51-63): q [q_heads][d], k/v [n][kv_heads][d]
 * fp32; writes out [q_heads][d] and the probability row of q head h to
 * probs + h*probs_ld (the trace row of that step). */
SPC_API int spc_full_attend(const float* q, const float* k, const float* v, int n, int q_heads, int kv_heads,
                            int head_dim, float scale, float* out, float* probs, int64_t probs_ld, void* stream);
/* sums[s*steps + t] = float32 np.sum of the row -- AttentionTrace.validate, hitrate.py:27-31. */
SPC_API int spc_trace_row_sums(const float* rows, int64_t seq_ld, int64_t row_ld, const int32_t* lens, int nseq,
                               int steps, int max_len, double* sums, void* stream);
/* rates[s*steps + t] = mass of the k largest entries -- topk_hitrate, hitrate.py:34-43. */
SPC_API int spc_topk_hitrate(const float* rows, int64_t seq_ld, int64_t row_ld, const int32_t* lens, int nseq,
                             int steps, int max_len, int k, double* rates, void* stream);
/* rates[s*steps + t] = greedy cumulative-score eviction at budget k -- eviction_hitrate, hitrate.py:46-77. */
SPC_API int spc_eviction_hitrate(const float* rows, int64_t seq_ld, int64_t row_ld, const int32_t* lens, int nseq,
                                 int steps, int max_len, int k, double* rates, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPECACHE_H_ */
