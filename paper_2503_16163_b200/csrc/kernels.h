// kernels.h -- internal launch interface between the C-ABI layer (api.cu) and
// the kernel translation units.  Not part of the public ABI.
#pragma once
#include "common.cuh"

namespace spc {

// K1 source: bf16 rows at element offset b*seq_stride + row*tok_stride +
// h*head_stride + c, where row = pos (prefill input) or pos % ring (ring).
struct QuantSrc {
  const __nv_bfloat16* k;
  const __nv_bfloat16* v;
  long long seq_stride, tok_stride, head_stride;
  int ring;
};

struct AttnArgs {
  Geo G;
  LayerBufs B;
  const __nv_bfloat16* q;      // [b][rows][Hq][d]
  const __nv_bfloat16* k_new;  // [b][rows][H][d]
  const __nv_bfloat16* v_new;
  __nv_bfloat16* out;          // [b][rows][Hq][d]
  float* pinned_mass;          // [b][Hq] or null
  int rows;                    // 1 predecode, 2 decode
  int agg_row;                 // row feeding the top-k aggregate
  int n, f;                    // length / frontier before this step's append
  int nsplit;                  // packed splits; split == nsplit is the exact segment
  int blocks_per_split;
  float* part_o;               // [b][H][nsplit+1][R][d]
  float* part_ml;              // [b][H][nsplit+1][R][2]
  float* pin_ml;               // [b][H][R][2]
  float* spill;                // [b][Hq][L] agg-row logits, log2 domain
  float* mz;                   // [b][Hq][2] agg-row (max, sum), log2 domain
  float sm_scale_log2;         // d^-0.5 * log2(e)
  float* out_f32;              // debug (spc_debug_output_f32): the combine's fp32 O before bf16 rounding
  int agg_recompute;           // 1: K2 spills no packed-position logits; K3r recomputes them (spc_set_agg_mode)
  int ring_append;             // 1: the combine also writes row 0's K/V into the residual ring (K6a fused)
};

size_t quantize_smem_bytes(const Geo& G);
void launch_h2d_probe(const void* src, void* dst, size_t bytes, int ctas, cudaStream_t st);
void launch_quantize(const Geo& G, const LayerBufs& B, const QuantSrc& S, int blk0, int nblocks,
                     cudaStream_t st);
void launch_export(const Geo& G, const LayerBufs& B, int seq, int nblocks, uint8_t* kc,
                   uint16_t* kz, uint16_t* ks, uint8_t* vc, uint16_t* vz, uint16_t* vs,
                   cudaStream_t st);
void launch_materialize(const Geo& G, const LayerBufs& B, int b, int h, int n, int f, float* keys,
                        float* values, cudaStream_t st);

// K2 (generic exact path and the tensor-core fast path) + K3 combine / agg
void launch_attend_generic(const AttnArgs& a, cudaStream_t st);
int attend_fast_supported(const Geo& G, int rows);
int launch_attend_fast(const AttnArgs& a, cudaStream_t st);  // returns kernels launched
void launch_combine(const AttnArgs& a, cudaStream_t st);
void launch_agg(const AttnArgs& a, cudaStream_t st);
void launch_agg_recompute(const AttnArgs& a, cudaStream_t st);

// K4 select + pin diff, K5 prefetch gather (zero-copy from pinned host), K6 append
void launch_topk(const Geo& G, const LayerBufs& B, int f, cudaStream_t st);
void launch_select(const float* scores, int n, int k, int32_t* out, cudaStream_t st);
void launch_set_pins(const Geo& G, const LayerBufs& B, int seq, int unit, const int32_t* pos,
                     int npos, cudaStream_t st);
void launch_prefetch(const Geo& G, const LayerBufs& B, const __nv_bfloat16* host_k,
                     const __nv_bfloat16* host_v, int64_t inflight_bytes, cudaStream_t st);
void launch_prefetch_one(const Geo& G, const LayerBufs& B, int seq, int unit,
                         const __nv_bfloat16* host_k, const __nv_bfloat16* host_v, cudaStream_t st);
void launch_copy_pins(const Geo& G, const LayerBufs& B, int seq, int unit, const __nv_bfloat16* k_rows,
                      const __nv_bfloat16* v_rows, int npos, cudaStream_t st);
void launch_ring_append(const Geo& G, const LayerBufs& B, const __nv_bfloat16* k_rows,
                        const __nv_bfloat16* v_rows, long long seq_stride, int n, cudaStream_t st);
void launch_host_append(const Geo& G, const LayerBufs& B, int n, __nv_bfloat16* host_k,
                        __nv_bfloat16* host_v, cudaStream_t st);
void launch_ring_fill(const Geo& G, const LayerBufs& B, const __nv_bfloat16* K,
                      const __nv_bfloat16* V, int n, int f, cudaStream_t st);

// spc_last_error() text for entry points outside api.cu (layer.cu)
int set_error(int code, const char* msg);

}  // namespace spc
