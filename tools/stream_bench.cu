// Microbenchmark (tools only): HBM weight-streaming rate of one resident CTA
// per SM pulling 16 KB tiles through an 8-deep TMA ring, as K7 / K8 do, for
// two weight layouts:
//   2d  : row-major W [N][K] bf16, each tile = a 128-row x 64-col box
//         (128 separate 128-B row segments, 2*K bytes apart) -- today's layout
//   1d  : the same tiles stored contiguously (a pre-tiled copy), each fetched
//         by one cp.async.bulk of 16 KB
// Prints GB/s for a weight matrix streamed by all SMs (N x K = the Llama-3.1-8B
// gate|up and qkv shapes), best of 5, CUDA events.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2410_01228_b200/csrc \
//        tools/stream_bench.cu -o tools/stream_bench
#include <cuda.h>

#include <cstdio>
#include <vector>

#include "common.cuh"
#include "tc.cuh"

using namespace csk;

constexpr int kTile = 16384;
constexpr int kRing = 8;

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   tc::smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(tc::smem_u32(bar))
               : "memory");
}

// tiles t = blockIdx.x, +gridDim.x, ...; tile t = (n_tile = t / kc, k_chunk = t % kc)
template <bool kBulk>
__global__ void __launch_bounds__(64, 1)
    stream_kernel(const __grid_constant__ CUtensorMap wmap, const uint8_t* tiled, int n_tiles, int kc, float* sink) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kRing * kTile);
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kRing; ++i) tc::mbar_init(&full[i], 1);
    tc::fence_mbar_init();
  }
  __syncthreads();
  const int mine = (n_tiles - static_cast<int>(blockIdx.x) + static_cast<int>(gridDim.x) - 1) / static_cast<int>(gridDim.x);
  float acc = 0.f;
  if (warp == 0 && tc::elect_one_sync()) {
    // producer and consumer in one thread: keep kRing tiles in flight
    auto issue = [&](int i) {
      const int t = static_cast<int>(blockIdx.x) + i * static_cast<int>(gridDim.x);
      const int st = i % kRing;
      tc::mbar_expect_tx(&full[st], kTile);
      if (kBulk) {
        bulk_load(smem + st * kTile, tiled + static_cast<size_t>(t) * kTile, kTile, &full[st]);
      } else {
        tc::tma_load_2d(smem + st * kTile, &wmap, &full[st], (t % kc) * 64, (t / kc) * 128);
      }
    };
    for (int i = 0; i < kRing && i < mine; ++i) issue(i);
    for (int i = 0; i < mine; ++i) {
      const int st = i % kRing;
      tc::mbar_wait(&full[st], (i / kRing) & 1);
      acc += reinterpret_cast<const float*>(smem + st * kTile)[i & 1023];
      if (i + kRing < mine) issue(i + kRing);
    }
  }
  if (acc == 12345.f) sink[0] = acc;  // keep the loads observable
}

static bool make_map(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols) {
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q{};
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (!fn) return false;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {cols * 2};
  const cuuint32_t box[2] = {64, 128};
  const cuuint32_t es[2] = {1, 1};
  return reinterpret_cast<EncodeFn>(fn)(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                                        strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = kRing * kTile + 1024 + 256;
  cudaFuncSetAttribute(stream_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(stream_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  float* sink;
  cudaMalloc(&sink, 4);
  struct Shape { const char* name; int N, K; };
  const Shape shapes[] = {{"gate_up", 28672, 4096}, {"qkv", 6144, 4096}, {"o_proj", 4096, 4096}, {"down", 4096, 14336}};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (const Shape& sh : shapes) {
    const size_t bytes = static_cast<size_t>(sh.N) * sh.K * 2;
    // 4 copies (>= 4 x 32 MB > L2) rotated so every launch streams from HBM
    const int copies = static_cast<int>(std::max<size_t>(2, (512u << 20) / bytes));
    uint8_t *w, *t;
    cudaMalloc(&w, bytes * copies);
    cudaMalloc(&t, bytes * copies);
    cudaMemset(w, 1, bytes * copies);
    cudaMemset(t, 1, bytes * copies);
    std::vector<CUtensorMap> maps(copies);
    for (int c = 0; c < copies; ++c) make_map(&maps[c], w + bytes * c, sh.N, sh.K);
    const int kc = sh.K / 64, n_tiles = (sh.N / 128) * kc;
    for (int mode = 0; mode < 2; ++mode) {
      float best = 1e30f;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        for (int c = 0; c < copies; ++c) {
          if (mode)
            stream_kernel<true><<<sms, 64, smem>>>(maps[c], t + bytes * c, n_tiles, kc, sink);
          else
            stream_kernel<false><<<sms, 64, smem>>>(maps[c], t + bytes * c, n_tiles, kc, sink);
        }
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        best = std::min(best, ms / copies);
      }
      std::printf("{\"shape\": \"%s\", \"layout\": \"%s\", \"MB\": %.1f, \"us\": %.2f, \"GBs\": %.1f}\n", sh.name,
                  mode ? "tiled_1d_bulk" : "rowmajor_2d_tma", bytes / 1e6, best * 1e3, bytes / (best * 1e-3) / 1e9);
    }
    cudaFree(w);
    cudaFree(t);
  }
  const cudaError_t err = cudaDeviceSynchronize();
  std::printf("{\"status\": \"%s\"}\n", cudaGetErrorString(err));
  return 0;
}
