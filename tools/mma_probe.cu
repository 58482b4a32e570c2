// mma_probe.cu -- the legacy tensor-core ceiling of K2 on B200: throughput of
// independent mma.sync.m16n8k16 f16 x f16 -> f32 (the SASS HMMA.16816.F32 K2
// issues), all SMs, several warps per SM, 8 independent accumulators per warp.
// K2 at the GQA-4 1-bit geometry (C3/C4) issues 68 of these per 32-token block
// of 2 KB (scores hi + lo, P.V hi + lo, the z and C_j MMAs), so at the HBM roof
// it would need blocks/s x 68 x 4096 x 2 flop; this probe gives the rate the
// mma.sync path can deliver at all.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/mma_probe.cu -o tools/mma_probe
//   tools/mma_probe            (prints one JSON line)
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__global__ void __launch_bounds__(256) k_hmma(float* out, int iters) {
  float d[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) d[i][0] = d[i][1] = d[i][2] = d[i][3] = 0.f;
  uint32_t a0 = 0x3c003c00u ^ threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 + 4, b1 = a0 + 5;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};\n"
          : "+f"(d[i][0]), "+f"(d[i][1]), "+f"(d[i][2]), "+f"(d[i][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1] + d[i][2] + d[i][3];
  if (s == 12345.f) out[threadIdx.x] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, 1024 * sizeof(float));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  std::printf("{\"probe\": \"mma.sync.m16n8k16.f32.f16.f16.f32\", \"sms\": %d, \"points\": [", sms);
  bool first = true;
  for (int wps : {4, 8, 16, 32}) {  // warps per SM
    const int ctas = sms * (wps / 4 > 0 ? wps / 4 : 1), threads = wps >= 4 ? 128 : 32 * wps;
    k_hmma<<<ctas, threads>>>(out, 64);
    cudaEventRecord(e0);
    k_hmma<<<ctas, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double mmas = (double)ctas * (threads / 32) * iters * 8;
    const double tflops = mmas * 16 * 8 * 16 * 2 / (ms * 1e-3) / 1e12;
    std::printf("%s{\"warps_per_sm\": %d, \"ms\": %.3f, \"hmma_per_sm_per_clk_at_1965\": %.3f, \"tflops\": %.1f}",
                first ? "" : ", ", wps, ms, mmas / sms / (ms * 1e-3 * 1.965e9), tflops);
    first = false;
  }
  std::printf("]}\n");
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
