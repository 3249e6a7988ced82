// Microbenchmark: cycles per tcgen05.mma (kind::f16, bf16 -> f32, cta_group::1)
// for the operand modes/shapes K2 uses. One CTA per SM, one elected lane
// issues `reps` back-to-back UMMAs into TMEM, commit + wait, clock64 delta.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2410_01228_b200/csrc \
//        tools/umma_bench.cu -o tools/umma_bench
#include <cstdio>

#include "common.cuh"
#include "tc.cuh"

using namespace csk;

template <int N, bool TS>
__global__ void umma_bench(long long* out, int reps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  // operands: A [128][64] bf16 (16 KB), B [N][64] (N*128 B); contents irrelevant
  for (int i = threadIdx.x; i < (16384 + N * 128) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  tc::fence_async_smem();
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc<512>(&tslot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 0) {
    const uint32_t a = tc::smem_u32(smem), b = a + 16384;
    constexpr uint32_t idesc = tc::idesc_bf16_f32(128, N, false, false);
    long long t0 = clock64();
    if (tc::elect_one_sync()) {
      for (int r = 0; r < reps; ++r) {
        const int ks = r & 3;
        if (TS)
          tc::umma_bf16_ts(tmem + 256, tmem + ks * 8, tc::sdesc_sw128(b + ks * 32, 16, 1024), idesc, 1);
        else
          tc::umma_bf16_ss(tmem, tc::sdesc_sw128(a + ks * 32, 16, 1024), tc::sdesc_sw128(b + ks * 32, 16, 1024),
                           idesc, 1);
      }
      tc::umma_commit(&bar);
    }
    __syncwarp();
    tc::mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

template <int N, bool TS>
void run(const char* name, int blocks) {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * blocks);
  const int smem = 16384 + N * 128 + 1024;
  cudaFuncSetAttribute(umma_bench<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int reps = 4096;
  umma_bench<N, TS><<<blocks, 128, smem>>>(d, reps);  // warm
  umma_bench<N, TS><<<blocks, 128, smem>>>(d, reps);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[256];
  cudaMemcpy(h, d, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < blocks; ++i) avg += h[i];
  avg /= blocks;
  const double cyc = avg / reps;
  const double macs = 128.0 * N * 16;
  printf("%-22s blocks=%3d  %7.1f cyc/UMMA  %7.0f MAC/cyc/SM  (%s)\n", name, blocks, cyc, macs / cyc,
         cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  for (int blocks : {1, 148}) {
    run<64, false>("SS M128 N64 K16", blocks);
    run<128, false>("SS M128 N128 K16", blocks);
    run<256, false>("SS M128 N256 K16", blocks);
    run<64, true>("TS M128 N64 K16", blocks);
    run<128, true>("TS M128 N128 K16", blocks);
    run<256, true>("TS M128 N256 K16", blocks);
  }
  return 0;
}
