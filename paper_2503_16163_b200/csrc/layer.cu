// Decoder-layer glue around the hot path: the elementwise
// pieces of the reference's layer (engine.py:35-72) as fused sm_100a kernels.
// The GEMMs (Wqkv, Wo, W1, W2, head) are plain cuBLAS bf16 GEMMs issued by the
// host (decoder.py); the attention is spc_decode_layer.
//
//   spc_add_rmsnorm  x += delta; out = bf16(rmsnorm(x) * gain)   numerics.py:42-51
//   spc_rope_table   (cos, sin) per (row, pair), once per step    numerics.py:54-63
//   spc_qkv_rope     split fused QKV rows, rotate q/k pairs       numerics.py:64-70
//   spc_silu         g / (1 + exp(-g)) in place                   engine.py:35-36
//   spc_argmax_rows  argmax per row, ties to the lowest index     numerics.py:73-78
//
// The residual stream x stays fp32 (rows x hidden, a few hundred KB); every
// GEMM operand is bf16 with fp32 accumulation.  All of these are HBM/latency
// bound at decode sizes (rows = 2 x batch): one CTA per row, 16-byte accesses.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/specache.h"
#include "kernels.h"

namespace {

__device__ __forceinline__ float bf2f(uint16_t u) { return __uint_as_float(uint32_t(u) << 16); }

constexpr int kNormThreads = 256;

// one CTA per row; hidden % 8 == 0
__global__ void __launch_bounds__(kNormThreads) k_add_rmsnorm(float* __restrict__ x,
                                                              const uint16_t* __restrict__ delta,
                                                              const float* __restrict__ gain,
                                                              uint16_t* __restrict__ out, int hidden,
                                                              float eps) {
  const int r = blockIdx.x;
  float* xr = x + (size_t)r * hidden;
  const uint16_t* dr = delta ? delta + (size_t)r * hidden : nullptr;
  float ss = 0.f;
  for (int c = threadIdx.x * 8; c < hidden; c += kNormThreads * 8) {
    float4 a = *reinterpret_cast<const float4*>(xr + c), b = *reinterpret_cast<const float4*>(xr + c + 4);
    if (dr) {
      const uint4 d = *reinterpret_cast<const uint4*>(dr + c);
      a.x += __uint_as_float(d.x << 16), a.y += __uint_as_float(d.x & 0xFFFF0000u);
      a.z += __uint_as_float(d.y << 16), a.w += __uint_as_float(d.y & 0xFFFF0000u);
      b.x += __uint_as_float(d.z << 16), b.y += __uint_as_float(d.z & 0xFFFF0000u);
      b.z += __uint_as_float(d.w << 16), b.w += __uint_as_float(d.w & 0xFFFF0000u);
      *reinterpret_cast<float4*>(xr + c) = a;
      *reinterpret_cast<float4*>(xr + c + 4) = b;
    }
    ss += a.x * a.x + a.y * a.y + a.z * a.z + a.w * a.w + b.x * b.x + b.y * b.y + b.z * b.z + b.w * b.w;
  }
  __shared__ float red[kNormThreads / 32];
#pragma unroll
  for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
#pragma unroll
  for (int w = 0; w < kNormThreads / 32; ++w) tot += red[w];
  const float inv = 1.f / __fsqrt_rn(tot / (float)hidden + eps);
  uint16_t* orow = out + (size_t)r * hidden;
  for (int c = threadIdx.x * 8; c < hidden; c += kNormThreads * 8) {
    const float4 a = *reinterpret_cast<const float4*>(xr + c), b = *reinterpret_cast<const float4*>(xr + c + 4);
    const float4 g0 = *reinterpret_cast<const float4*>(gain + c), g1 = *reinterpret_cast<const float4*>(gain + c + 4);
    __nv_bfloat162 o0 = __floats2bfloat162_rn(a.x * g0.x * inv, a.y * g0.y * inv);
    __nv_bfloat162 o1 = __floats2bfloat162_rn(a.z * g0.z * inv, a.w * g0.w * inv);
    __nv_bfloat162 o2 = __floats2bfloat162_rn(b.x * g1.x * inv, b.y * g1.y * inv);
    __nv_bfloat162 o3 = __floats2bfloat162_rn(b.z * g1.z * inv, b.w * g1.w * inv);
    uint4 pk;
    pk.x = *reinterpret_cast<uint32_t*>(&o0);
    pk.y = *reinterpret_cast<uint32_t*>(&o1);
    pk.z = *reinterpret_cast<uint32_t*>(&o2);
    pk.w = *reinterpret_cast<uint32_t*>(&o3);
    *reinterpret_cast<uint4*>(orow + c) = pk;
  }
}

// table[r][i] = (cos, sin) of positions[r] * base^(-2i/d): angles in fp64 like
// numerics.py:62, cos/sin rounded to fp32.  Once per step (positions are shared by
// every layer), so the fp64 work is off the per-layer path.
__global__ void k_rope_table(const int32_t* __restrict__ pos, int rows, int half, double base,
                             float2* __restrict__ table) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= rows * half) return;
  const int r = t / half, i = t - r * half;
  const double ang = (double)pos[r] * pow(base, -2.0 * i / (2 * half));
  double sd, cd;
  sincos(ang, &sd, &cd);
  table[t] = make_float2((float)cd, (float)sd);
}

// grid (rows, Hq + 2 Hkv), block d/2: thread i rotates pair (2i, 2i+1) of one head
__global__ void k_qkv_rope(const uint16_t* __restrict__ qkv, const float2* __restrict__ table, int Hq, int Hkv,
                           int d, uint16_t* __restrict__ q, uint16_t* __restrict__ k, uint16_t* __restrict__ v) {
  const int r = blockIdx.x, h = blockIdx.y, i = threadIdx.x;
  const int width = (Hq + 2 * Hkv) * d;
  const uint16_t* src = qkv + (size_t)r * width + (size_t)h * d;
  const uint32_t w = *reinterpret_cast<const uint32_t*>(src + 2 * i);
  uint16_t* dst;
  if (h < Hq) dst = q + ((size_t)r * Hq + h) * d;
  else if (h < Hq + Hkv) dst = k + ((size_t)r * Hkv + (h - Hq)) * d;
  else {
    *reinterpret_cast<uint32_t*>(v + ((size_t)r * Hkv + (h - Hq - Hkv)) * d + 2 * i) = w;
    return;
  }
  const float2 cs = table[(size_t)r * (d / 2) + i];
  const float x0 = __uint_as_float(w << 16), x1 = __uint_as_float(w & 0xFFFF0000u);
  __nv_bfloat162 o = __floats2bfloat162_rn(x0 * cs.x - x1 * cs.y, x0 * cs.y + x1 * cs.x);
  *reinterpret_cast<__nv_bfloat162*>(dst + 2 * i) = o;
}

__global__ void k_silu(uint16_t* __restrict__ g, size_t n8) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n8; i += (size_t)gridDim.x * blockDim.x) {
    uint4 w = reinterpret_cast<uint4*>(g)[i];
    uint32_t* p = &w.x;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float a = __uint_as_float(p[j] << 16), b = __uint_as_float(p[j] & 0xFFFF0000u);
      __nv_bfloat162 o = __floats2bfloat162_rn(a / (1.f + __expf(-a)), b / (1.f + __expf(-b)));
      p[j] = *reinterpret_cast<uint32_t*>(&o);
    }
    reinterpret_cast<uint4*>(g)[i] = w;
  }
}

constexpr int kArgThreads = 1024;

__global__ void __launch_bounds__(kArgThreads) k_argmax_rows(const uint16_t* __restrict__ x, int cols,
                                                             int32_t* __restrict__ out) {
  const uint16_t* row = x + (size_t)blockIdx.x * cols;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  for (int c = threadIdx.x; c < cols; c += kArgThreads) {
    const float v = bf2f(row[c]);
    if (v > best) best = v, bi = c;  // strided scan: first hit is this thread's lowest index
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) best = ov, bi = oi;
  }
  __shared__ float sv[kArgThreads / 32];
  __shared__ int si[kArgThreads / 32];
  if ((threadIdx.x & 31) == 0) sv[threadIdx.x >> 5] = best, si[threadIdx.x >> 5] = bi;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kArgThreads / 32; ++w)
      if (sv[w] > best || (sv[w] == best && si[w] < bi)) best = sv[w], bi = si[w];
    out[blockIdx.x] = bi == 0x7fffffff ? 0 : bi;  // all-NaN row -> 0
  }
}

int cuda_status(cudaError_t e) {
  return e == cudaSuccess ? SPC_OK : spc::set_error(SPC_ECUDA, cudaGetErrorString(e));
}

int bad(const char* what) { return spc::set_error(SPC_EINVAL, what); }

}  // namespace

extern "C" {

int spc_add_rmsnorm(float* x, const void* delta, const float* gain, void* out, int rows, int hidden, float eps,
                    void* stream) {
  if (!x || !gain || !out || rows < 0) return bad("add_rmsnorm: null pointer or negative rows");
  if (hidden <= 0 || hidden % 8) return bad("add_rmsnorm: hidden must be a positive multiple of 8");
  if (!(eps > 0.f)) return bad("eps must be positive");
  if (rows == 0) return SPC_OK;
  k_add_rmsnorm<<<rows, kNormThreads, 0, (cudaStream_t)stream>>>(x, (const uint16_t*)delta, gain, (uint16_t*)out,
                                                                 hidden, eps);
  return cuda_status(cudaGetLastError());
}

int spc_rope_table(const int32_t* positions, int rows, int head_dim, double rope_base, float* table,
                   void* stream) {
  if (!positions || !table || rows < 0) return bad("rope_table: null pointer or negative rows");
  if (head_dim <= 0 || head_dim % 2 || head_dim > 2048) return bad("head_dim must be even (rotary pairs)");
  if (!(rope_base > 0)) return bad("rope_base must be positive");
  if (rows == 0) return SPC_OK;
  const int n = rows * (head_dim / 2);
  k_rope_table<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(positions, rows, head_dim / 2, rope_base,
                                                                  (float2*)table);
  return cuda_status(cudaGetLastError());
}

int spc_qkv_rope(const void* qkv, const float* rope_table, int rows, int q_heads, int kv_heads, int head_dim,
                 void* q, void* k, void* v, void* stream) {
  if (!qkv || !rope_table || !q || !k || !v || rows < 0) return bad("qkv_rope: null pointer or negative rows");
  if (q_heads <= 0 || kv_heads <= 0) return bad("qkv_rope: head counts must be positive");
  if (head_dim <= 0 || head_dim % 2 || head_dim > 2048) return bad("head_dim must be even (rotary pairs)");
  if (rows == 0) return SPC_OK;
  k_qkv_rope<<<dim3(rows, q_heads + 2 * kv_heads), head_dim / 2, 0, (cudaStream_t)stream>>>(
      (const uint16_t*)qkv, (const float2*)rope_table, q_heads, kv_heads, head_dim, (uint16_t*)q, (uint16_t*)k,
      (uint16_t*)v);
  return cuda_status(cudaGetLastError());
}

int spc_silu(void* g, int64_t n, void* stream) {
  if (!g || n < 0 || n % 8) return bad("silu: n must be a non-negative multiple of 8");
  if (n == 0) return SPC_OK;
  const size_t n8 = (size_t)n / 8;
  const int blocks = (int)((n8 + 255) / 256 < 148 * 8 ? (n8 + 255) / 256 : 148 * 8);
  k_silu<<<blocks, 256, 0, (cudaStream_t)stream>>>((uint16_t*)g, n8);
  return cuda_status(cudaGetLastError());
}

int spc_argmax_rows(const void* x, int rows, int cols, int32_t* out, void* stream) {
  if (!x || !out || rows < 0) return bad("argmax_rows: null pointer or negative rows");
  if (cols <= 0) return bad("argmax of an empty row");
  if (rows == 0) return SPC_OK;
  k_argmax_rows<<<rows, kArgThreads, 0, (cudaStream_t)stream>>>((const uint16_t*)x, cols, out);
  return cuda_status(cudaGetLastError());
}

}  // extern "C"
