// quant.cu -- K1: group quantizer + bit packing on device, and the two parity
// readers (normative export, exact materialize).
//
// Reference: quant.py:59-190 (params, codes, LSB-first packing, per-channel key
// groups, per-token value groups), kvcache.py:173-192 (migrate_residual),
// kvcache.py:222-243 (materialize), kvcache.py:270-281 (snapshot).
#include "common.cuh"
#include "kernels.h"

namespace spc {

// One CTA quantizes one g-token block of one (seq, kv head).  The block is
// staged in shared memory as fp32 (exact copies of the bf16 inputs), group
// (min, max) are reduced there, codes are computed in float64 exactly as the
// reference does and OR-ed into the block's packed words in shared memory,
// then the words stream out coalesced.
__global__ void __launch_bounds__(256) k_quantize(Geo G, LayerBufs B, QuantSrc S, int blk0) {
  const int blk = blk0 + blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int g = G.g, d = G.d, tid = threadIdx.x, nt = blockDim.x;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* sk = reinterpret_cast<float*>(smem_raw);            // [g][d]
  float* sv = sk + g * d;                                    // [g][d]
  uint32_t* wk = reinterpret_cast<uint32_t*>(sv + g * d);    // [g*krw]
  uint32_t* wv = wk + G.bwords;                              // [g*vrw]
  double* kz = reinterpret_cast<double*>(wv + G.bwords + (G.bwords & 1));  // [d]
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
  const size_t bi = blk_index(G, b, h, blk);

  if (G.bits == 16) {  // verbatim full-precision tier (kvcache.py:185-187)
    __nv_bfloat16* okc = reinterpret_cast<__nv_bfloat16*>(B.kcodes + bi * (size_t)G.rec);
    __nv_bfloat16* ovc = reinterpret_cast<__nv_bfloat16*>(B.vcodes + bi * (size_t)G.rec);
    for (int i = tid; i < g * d; i += nt) {
      okc[i] = __float2bfloat16_rn(sk[i]);
      ovc[i] = __float2bfloat16_rn(sv[i]);
    }
    return;
  }

  __shared__ float s_rk, s_rv;
  if (tid == 0) {
    s_rk = 0.f;
    s_rv = 0.f;
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
    B.kparams[bi * G.rec + kpi(G, c)] = float_to_bf16_bits_exact(lo) | (float_to_bf16_bits_exact(hi) << 16);
    atomicMax(reinterpret_cast<unsigned*>(&s_rk), __float_as_uint(hi - lo));
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
    B.vparams[bi * (size_t)G.rec + vpi(G, t, j)] =
        float_to_bf16_bits_exact(lo) | (float_to_bf16_bits_exact(hi) << 16);
    atomicMax(reinterpret_cast<unsigned*>(&s_rv), __float_as_uint(hi - lo));
    GroupParams p = params_from_minmax((double)lo, (double)hi, G.bits);
    vz[i] = p.zero;
    vs[i] = p.scale;
  }
  for (int i = tid; i < G.bwords; i += nt) {
    wk[i] = 0u;
    wv[i] = 0u;
  }
  __syncthreads();
  if (tid == 0) {  // per-(seq, head) range maxima: exponent choice of the MMA path
    atomicMax(&B.rmax[((size_t)b * G.H + h) * 2 + 0], __float_as_uint(s_rk));
    atomicMax(&B.rmax[((size_t)b * G.H + h) * 2 + 1], __float_as_uint(s_rv));
  }
  for (int i = tid; i < g * d; i += nt) {
    int t = i / d, c = i - t * d, w, bit;
    GroupParams pk{kz[c], ks[c]};
    uint32_t ck = quantize_code(sk[i], pk, G.bits);
    kloc(G, t, c, &w, &bit);
    if (ck) atomicOr(&wk[w], ck << bit);
    int j = c / g;
    GroupParams pv{vz[t * G.nch + j], vs[t * G.nch + j]};
    uint32_t cv = quantize_code(sv[i], pv, G.bits);
    vloc(G, t, c, &w, &bit);
    if (cv) atomicOr(&wv[w], cv << bit);
  }
  __syncthreads();
  uint32_t* okc = B.kcodes + bi * (size_t)G.rec;
  uint32_t* ovc = B.vcodes + bi * (size_t)G.rec;
  for (int i = tid; i < G.bwords; i += nt) {
    okc[i] = wk[i];
    ovc[i] = wv[i];
  }
}

size_t quantize_smem_bytes(const Geo& G) {
  size_t s = 2 * sizeof(float) * G.g * G.d;
  s += sizeof(uint32_t) * (2 * G.bwords + 2);
  s += sizeof(double) * (2 * G.d + 2 * G.g * G.nch);
  return s;
}

void launch_quantize(const Geo& G, const LayerBufs& B, const QuantSrc& S, int blk0, int nblocks,
                     cudaStream_t st) {
  if (nblocks <= 0) return;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_quantize, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    configured = true;
  }
  dim3 grid(nblocks, G.H, G.batch);
  k_quantize<<<grid, 256, quantize_smem_bytes(G), st>>>(G, B, S, blk0);
}

// ---------------------------------------------------------------------------------
// Normative export of one (layer, seq): the arrays TwoTierCache.snapshot() would
// serialise (kvcache.py:270-281), codes LSB-first per group (quant.py:96-109),
// fp16 zero/scale as a direct float64 -> fp16 rounding (quant.py:150-160).
__global__ void k_export(Geo G, LayerBufs B, int seq, int nblocks, uint8_t* kcodes,
                         uint16_t* kzero, uint16_t* kscale, uint8_t* vcodes, uint16_t* vzero,
                         uint16_t* vscale) {
  const int blk = blockIdx.x, h = blockIdx.y, tid = threadIdx.x;
  const int g = G.g, d = G.d, bits = G.bits, nb = (g * bits + 7) / 8;
  const size_t bi = blk_index(G, seq, h, blk);
  const uint32_t* kw = B.kcodes + bi * (size_t)G.rec;
  const uint32_t* vw = B.vcodes + bi * (size_t)G.rec;
  const int per = 8 / bits;
  // key groups [nblocks][H][d][nb]
  for (int i = tid; i < d * nb; i += blockDim.x) {
    int c = i / nb, byte = i - c * nb;
    uint32_t v = 0;
    for (int j = 0; j < per; ++j) {
      int t = byte * per + j;
      if (t >= g) break;
      int w, bit;
      kloc(G, t, c, &w, &bit);
      v |= read_code(kw, w, bit, bits) << (j * bits);
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
      vloc(G, t, c, &w, &bit);
      v |= read_code(vw, w, bit, bits) << (jj * bits);
    }
    vcodes[((((size_t)blk * g + t) * G.H + h) * G.nch + j) * nb + byte] = (uint8_t)v;
  }
  for (int i = tid; i < g * G.nch; i += blockDim.x) {
    int t = i / G.nch, j = i - t * G.nch;
    GroupParams p = params_from_word(B.vparams[bi * (size_t)G.rec + vpi(G, t, j)], bits);
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
  int blk = pos / G.g, t = pos - blk * G.g;
  size_t bi = blk_index(G, b, h, blk);
  if (G.bits == 16)
    return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(B.kcodes + bi * (size_t)G.rec)[t * G.d + c]);
  int w, bit;
  kloc(G, t, c, &w, &bit);
  uint32_t code = read_code(B.kcodes + bi * (size_t)G.rec, w, bit, G.bits);
  return dequant_exact(code, params_from_word(B.kparams[bi * G.rec + kpi(G, c)], G.bits));
}
__device__ inline float packed_val(const Geo& G, const LayerBufs& B, int b, int h, int pos, int c) {
  int blk = pos / G.g, t = pos - blk * G.g;
  size_t bi = blk_index(G, b, h, blk);
  if (G.bits == 16)
    return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(B.vcodes + bi * (size_t)G.rec)[t * G.d + c]);
  int w, bit;
  vloc(G, t, c, &w, &bit);
  uint32_t code = read_code(B.vcodes + bi * (size_t)G.rec, w, bit, G.bits);
  return dequant_exact(code, params_from_word(B.vparams[bi * (size_t)G.rec + vpi(G, t, c / G.g)], G.bits));
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
