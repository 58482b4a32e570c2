// h2d_probe.cu -- SURVEY 7 step 6: the K5 prefetch design choice, measured.
// Gathers `rows` randomly chosen rows of `row_bytes` from a pinned host slab
// into device memory three ways and reports GB/s:
//   (a) zero-copy gather kernel (K5's approach: 16-byte loads through the
//       mapped host pointer, in-flight bytes bounded by the grid);
//   (b) one cudaMemcpyAsync per row.
// (A batched-descriptor copy arm was measured in r1, profiles/r1_20_*; that
// API is closed on this GPU pool and the arm was removed.)
// Also the contiguous pinned H2D peak (one cudaMemcpyAsync of the same bytes).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/h2d_probe.cu -o tools/h2d_probe
//   tools/h2d_probe [row_bytes rows [slab_rows]]   (default: the C2 and C3 per-layer gathers)
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));                 \
      std::exit(1);                                                                 \
    }                                                                               \
  } while (0)

__global__ void gather(const uint4* __restrict__ host, uint4* __restrict__ dev, const int* __restrict__ pos,
                       int rows, int chunks_per_row) {
  const long long total = (long long)rows * chunks_per_row;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(i / chunks_per_row), c = (int)(i % chunks_per_row);
    dev[i] = host[(long long)pos[r] * chunks_per_row + c];
  }
}

static float time_ms(cudaStream_t st, cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  CK(cudaEventSynchronize(b));
  CK(cudaEventElapsedTime(&ms, a, b));
  return ms;
}

static void run(size_t row_bytes, int rows, size_t slab_rows) {
  const size_t slab = slab_rows * row_bytes, bytes = (size_t)rows * row_bytes;
  char* h = nullptr;
  CK(cudaHostAlloc((void**)&h, slab, cudaHostAllocMapped));
  for (size_t i = 0; i < slab; i += 4096) h[i] = (char)i;
  char* hd = nullptr;
  CK(cudaHostGetDevicePointer((void**)&hd, h, 0));
  char* d = nullptr;
  CK(cudaMalloc((void**)&d, bytes));
  std::vector<int> pos(rows);  // row index < 2^31
  std::mt19937 rng(7);
  std::uniform_int_distribution<long long> U(0, (long long)slab_rows - 1);
  for (int& p : pos) p = U(rng);
  int* dpos = nullptr;
  CK(cudaMalloc((void**)&dpos, rows * sizeof(int)));
  CK(cudaMemcpy(dpos, pos.data(), rows * sizeof(int), cudaMemcpyHostToDevice));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int reps = 20;
  auto best = [&](auto&& fn) {
    fn();
    CK(cudaStreamSynchronize(st));
    float b = 1e30f;
    for (int i = 0; i < reps; ++i) {
      CK(cudaEventRecord(e0, st));
      fn();
      CK(cudaEventRecord(e1, st));
      b = std::min(b, time_ms(st, e0, e1));
    }
    return bytes / (b / 1e3) / 1e9;
  };
  // (0) contiguous peak
  const double peak = best([&] { CK(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st)); });
  // (a) zero-copy gather, ~256 KiB in flight (16 CTAs x 256 threads x 4 x 16 B) and wider
  const int cpr = (int)(row_bytes / 16);
  double zc[3];
  const int grids[3] = {16, 64, 296};
  for (int g = 0; g < 3; ++g)
    zc[g] = best([&] { gather<<<grids[g], 256, 0, st>>>((const uint4*)hd, (uint4*)d, dpos, rows, cpr); });
  std::vector<void*> dsts(rows), srcs(rows);
  for (int r = 0; r < rows; ++r) {
    dsts[r] = d + (size_t)r * row_bytes;
    srcs[r] = h + (size_t)pos[r] * row_bytes;
  }
  // (b) one cudaMemcpyAsync per row
  const double per_row = best([&] {
    for (int r = 0; r < rows; ++r)
      CK(cudaMemcpyAsync(dsts[r], srcs[r], row_bytes, cudaMemcpyHostToDevice, st));
  });
  std::printf("{\"row_bytes\": %zu, \"rows\": %d, \"MB\": %.2f, \"contiguous_peak_gbs\": %.1f, "
              "\"zero_copy_gbs\": {\"16_ctas\": %.1f, \"64_ctas\": %.1f, \"296_ctas\": %.1f}, "
              "\"memcpy_per_row_gbs\": %.1f}\n",
              row_bytes, rows, bytes / 1e6, peak, zc[0], zc[1], zc[2], per_row);
  CK(cudaFree(dpos));
  CK(cudaFree(d));
  CK(cudaFreeHost(h));
  CK(cudaStreamDestroy(st));
}

int main(int argc, char** argv) {
  if (argc >= 3) {  // row_bytes rows [slab_rows]
    run((size_t)std::atoll(argv[1]), std::atoi(argv[2]), argc > 3 ? (size_t)std::atoll(argv[3]) : 65536);
    return 0;
  }
  // C2 per layer-step: 16 seqs x ~47 new pins (73% of k=64) x (K, V) rows of H*d*2 = 8 KiB
  run(8192, 16 * 47 * 2, 65536);
  // C3 per layer-step: 8 seqs x ~100 new pins (78% of 128) x (K, V) rows of 8 heads * 128 * 2 = 2 KiB
  run(2048, 8 * 100 * 2, 262144);
  // a larger batch of copies
  run(8192, 8192, 65536);
  return 0;
}
