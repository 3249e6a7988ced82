// Micro-benchmark: host-link paths for KV checkpoint/restore on B200.
//  (1) cudaMemcpyAsync pinned D2H/H2D (DMA, the reference number)
//  (2) zero-copy kernel STORES into mapped pinned memory (gather-to-host)
//  (3) zero-copy kernel LOADS from mapped pinned memory (scatter-from-host)
//  segment sizes 256 B .. 64 KiB scattered randomly over a 4 GiB device pool.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void gather_to_host(const int4* __restrict__ dev, int4* host, const int64_t* seg_src, int nseg, int seg_vec) {
  // one warp per segment chunk
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int s = warp; s < nseg; s += nwarps) {
    const int4* src = dev + seg_src[s] * seg_vec;
    int4* dst = host + (int64_t)s * seg_vec;
    for (int i = lane; i < seg_vec; i += 32) dst[i] = __ldg(src + i);
  }
}
__global__ void scatter_from_host(int4* __restrict__ dev, const int4* host, const int64_t* seg_dst, int nseg, int seg_vec) {
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int s = warp; s < nseg; s += nwarps) {
    int4* dst = dev + seg_dst[s] * seg_vec;
    const int4* src = host + (int64_t)s * seg_vec;
    int4 v[4]; int n = 0;
    for (int i = lane; i < seg_vec; i += 32 * 4) {
      #pragma unroll
      for (int u = 0; u < 4; ++u) if (i + u * 32 < seg_vec) v[u] = src[i + u * 32];
      #pragma unroll
      for (int u = 0; u < 4; ++u) if (i + u * 32 < seg_vec) dst[i + u * 32] = v[u];
      n++;
    }
  }
}
int main() {
  const size_t pool = 4ull << 30, hostsz = 1ull << 30;
  void *d, *h, *hd;
  CK(cudaMalloc(&d, pool));
  CK(cudaHostAlloc(&h, hostsz, cudaHostAllocMapped));
  CK(cudaHostGetDevicePointer(&hd, h, 0));
  cudaStream_t st; CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  for (int dir = 0; dir < 2; ++dir) {
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0, st);
      if (dir == 0) cudaMemcpyAsync(h, d, hostsz, cudaMemcpyDeviceToHost, st); else cudaMemcpyAsync(d, h, hostsz, cudaMemcpyHostToDevice, st);
      cudaEventRecord(e1, st); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms);
    }
    printf("memcpyAsync %s 1GiB: %.1f GB/s\n", dir ? "H2D" : "D2H", hostsz / (best * 1e-3) / 1e9);
  }
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int seg : {256, 512, 1024, 4096, 16384, 65536, 2 << 20}) {
    int seg_vec = seg / 16;
    int nseg = (int)(hostsz / seg);
    int64_t nslots = pool / seg;
    std::vector<int64_t> idx(nseg);
    std::mt19937_64 rng(1);
    for (auto& x : idx) x = rng() % nslots;
    int64_t* didx; CK(cudaMalloc(&didx, nseg * 8)); CK(cudaMemcpy(didx, idx.data(), nseg * 8, cudaMemcpyHostToDevice));
    for (int grid_mult : {1, 4, 16}) {
      int grid = sms * grid_mult;
      for (int dir = 0; dir < 2; ++dir) {
        float best = 1e9;
        for (int r = 0; r < 4; ++r) {
          cudaEventRecord(e0, st);
          if (dir == 0) gather_to_host<<<grid, 512, 0, st>>>((const int4*)d, (int4*)hd, didx, nseg, seg_vec);
          else scatter_from_host<<<grid, 512, 0, st>>>((int4*)d, (const int4*)hd, didx, nseg, seg_vec);
          cudaEventRecord(e1, st); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms);
        }
        printf("zero-copy %s seg=%7d B grid=%4d: %.1f GB/s\n", dir ? "load(H2D)" : "store(D2H)", seg, grid, hostsz / (best * 1e-3) / 1e9);
      }
    }
    cudaFree(didx);
  }
  // per-page DMA copies (2 MiB), many calls
  {
    int npages = 256; size_t pb = 2 << 20;
    float best = 1e9;
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(e0, st);
      for (int i = 0; i < npages; ++i) cudaMemcpyAsync((char*)d + (size_t)((i * 7919) % 2000) * pb, (char*)h + i * pb, pb, cudaMemcpyHostToDevice, st);
      cudaEventRecord(e1, st); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms);
    }
    printf("per-page DMA H2D 256 x 2MiB: %.1f GB/s\n", npages * pb / (best * 1e-3) / 1e9);
  }
  return 0;
}
