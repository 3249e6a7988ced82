// K7: the decode-step projections (qkv, o_proj, gate|up, down, lm_head for
// M <= 256 token rows) as a weight-streaming GEMM on the 5th-generation
// tensor cores. At these M the GEMM is an HBM stream of the weights (436 MB
// per Llama-3.1-8B layer) and cuBLAS leaves 20-55% of the bandwidth idle
// (profiles/r1: o_proj 2.9 TB/s, down 3.9 TB/s at M = 128).
//
// Swap-AB: D[128 features, Mp tokens] = W_tile[128, K] . X[Mp, K]^T, so the
// weight tile is the UMMA A operand (M = 128) and the few token rows are the
// N dimension (Mp = M rounded up to 16, <= 256); both operands K-major,
// 128-B swizzled, loaded by TMA (64 K-elements per stage). One CTA = one
// 128-feature tile x one K range; the K ranges of a feature tile form a
// thread-block cluster (<= 8 CTAs) whose fp32 partials are reduced through
// distributed shared memory -- no global workspace, no atomics, no second
// kernel. Warp roles (128 threads): warp 0 TMA producer, warp 1 UMMA issuer
// (one elected lane each, warp-wide loops), then all four warps drain TMEM
// (warp w owns lanes / features 32w .. 32w+31).
#include <cstdlib>

#include "common.cuh"
#include "tc.cuh"

namespace csk {

namespace {

constexpr int kFeat = 128;        // UMMA M: output features per CTA
constexpr int kKc = 64;           // K elements per stage (one 128-B swizzled row)
constexpr int kWBytes = kFeat * kKc * 2;  // 16 KB weight tile per stage
constexpr int kGemmThreads = 128;
constexpr int kMaxStages = 8;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cta address of this CTA -> the same offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t map_peer(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ float4 ld_dsmem_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}

}  // namespace

struct WgemmArgs {
  void* y;            // [M, N] bf16 (or fp32 when f32_out)
  int32_t M, Mp, N, K;
  int32_t splits;     // cluster size along K (1..8) = gridDim.y
  int32_t chunks;     // 64-element K chunks per split
  int32_t f32_out;
  int32_t stages;     // smem ring depth (<= kMaxStages)
};

__global__ void __launch_bounds__(kGemmThreads, 1)
    wgemm_tc_kernel(const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap xmap,
                    WgemmArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int Mp = a.Mp;
  const uint32_t stage_bytes = kWBytes + static_cast<uint32_t>(Mp) * 128;  // multiple of 2 KB
  const int S = a.stages;
  const uint32_t ring_bytes = S * stage_bytes;
  const uint32_t red_bytes = static_cast<uint32_t>(Mp) * kFeat * 4;        // fp32 partial [Mp][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (ring_bytes > red_bytes ? ring_bytes : red_bytes));
  uint64_t* full = bars;                 // [stages]
  uint64_t* empty = bars + kMaxStages;   // [stages]
  uint64_t* done = bars + 2 * kMaxStages;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * kFeat;
  const int split = blockIdx.y;
  const int c_begin = split * a.chunks;
  const int nc = min(a.chunks, a.K / kKc - c_begin);

  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&empty[i], 1);
    }
    tc::mbar_init(done, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&wmap);
    tc::prefetch_tmap(&xmap);
  }
  if (warp == 1) tc::tmem_alloc<256>(tslot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tslot;

  const int rot = static_cast<int>(blockIdx.x) % max(nc, 1);
  if (warp == 0) {
    // ------------------------------------------------------ TMA producer --
    // The weights do not depend on the previous kernel: the first ring's
    // worth is requested before griddepcontrol.wait (PDL launch), the
    // activations only after it.
    const int pre = min(S, nc);
    if (tc::elect_one_sync()) {
      for (int i = 0; i < pre; ++i) {
        const int kc = (c_begin + (i + rot) % nc) * kKc;
        tc::mbar_expect_tx(&full[i], stage_bytes);
        tc::tma_load_2d(smem + i * stage_bytes, &wmap, &full[i], kc, n0);
      }
    }
    __syncwarp();
    pdl_wait();
    for (int i = 0; i < nc; ++i) {
      const int st = i % S;
      if (i >= S) tc::mbar_wait(&empty[st], ((i / S) - 1) & 1);
      if (tc::elect_one_sync()) {
        uint8_t* sw = smem + st * stage_bytes;
        // feature tiles start their K loop at different chunks: the X tile
        // every CTA of a split needs is not fetched by all of them at once
        const int kc = (c_begin + (i + rot) % nc) * kKc;
        if (i >= pre) {
          tc::mbar_expect_tx(&full[st], stage_bytes);
          tc::tma_load_2d(sw, &wmap, &full[st], kc, n0);
        }
        tc::tma_load_2d(sw + kWBytes, &xmap, &full[st], kc, 0);
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // -------------------------------------------------------- MMA issuer --
    const uint32_t idesc = tc::idesc_bf16_f32(kFeat, Mp, false, false);
    const uint32_t base = tc::smem_u32(smem);
    for (int i = 0; i < nc; ++i) {
      const int st = i % S;
      tc::mbar_wait(&full[st], (i / S) & 1);
      tc::tc_fence_after();
      if (tc::elect_one_sync()) {
        const uint32_t wa = base + st * stage_bytes, xa = wa + kWBytes;
#pragma unroll
        for (int ks = 0; ks < kKc / 16; ++ks)
          tc::umma_bf16_ss(tmem, tc::sdesc_sw128(wa + ks * 32, 16, 1024), tc::sdesc_sw128(xa + ks * 32, 16, 1024),
                           idesc, (i > 0 || ks > 0) ? 1u : 0u);
        tc::umma_commit(&empty[st]);
        if (i == nc - 1) tc::umma_commit(done);
      }
      __syncwarp();
    }
  }

  // ---------------------------------------------------------- epilogue --
  // TMEM lane f = feature n0 + f, column c = token c. Partial -> own smem as
  // red[c][f] (the ring is idle once `done` fired), cluster barrier, then CTA
  // r of the cluster sums rows c = r, r + splits, ... over every peer's red
  // and writes them (16-B stores along the features).
  tc::mbar_wait(done, 0);
  tc::tc_fence_after();
  pdl_wait();  // (returns at once: the producer's wait already saw the previous grid complete)
  float* red = reinterpret_cast<float*>(smem);
  const int f = warp * 32 + lane;
  const uint32_t tl = tmem + (static_cast<uint32_t>(warp * 32) << 16);
  for (int c0 = 0; c0 < Mp; c0 += 32) {
    float v[32];
    tc::tmem_ld32(tl + c0, v);
    tc::tmem_wait_ld();
    tc::reg_fence<32>(v);
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (c0 + i < Mp) red[(c0 + i) * kFeat + f] = v[i];
  }
  tc::tc_fence_before();
  if (a.splits > 1) {
    cluster_sync();
  } else {
    __syncthreads();
  }
  const uint32_t my_rank = a.splits > 1 ? cluster_rank() : 0;
  const uint32_t red_s = tc::smem_u32(red);
  // 32 threads per row (4 features each), 4 rows per pass
  const int fq = (threadIdx.x & 31) * 4;
  for (int c = static_cast<int>(my_rank) * 4 + (threadIdx.x >> 5); c < a.M; c += a.splits * 4) {
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    const uint32_t off = static_cast<uint32_t>((c * kFeat + fq) * 4);
    for (int q = 0; q < a.splits; ++q) {
      const float4 t = a.splits > 1 ? ld_dsmem_f4(map_peer(red_s + off, q))
                                    : *reinterpret_cast<const float4*>(red + c * kFeat + fq);
      s.x += t.x;
      s.y += t.y;
      s.z += t.z;
      s.w += t.w;
    }
    const size_t o = static_cast<size_t>(c) * a.N + n0 + fq;
    if (a.f32_out) {
      *reinterpret_cast<float4*>(static_cast<float*>(a.y) + o) = s;
    } else {
      *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(a.y) + o) = make_uint2(pack_bf16(s.x, s.y), pack_bf16(s.z, s.w));
    }
  }
  if (a.splits > 1) cluster_sync();  // peers keep their smem until every reader is done
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 1) tc::tmem_dealloc<256>(tmem);
}

// ------------------------------------------------------ K7 stream-K mode --
// Same swap-AB operands as above, but ONE persistent CTA per SM walks an
// equal contiguous range of the flattened (feature tile, 64-wide K chunk)
// units, so every SM streams the same number of weight bytes whatever N / 128
// is (gate|up 224 tiles, qkv 48, o/down 32 on 148 SMs), and the TMA ring runs
// on across tile boundaries. The accumulator is double-buffered in TMEM:
// the epilogue of one tile segment overlaps the next segment's main loop. A
// tile cut by range boundaries leaves an fp32 partial per covering CTA in a
// global workspace (slot 0 = the CTA's first segment, slot 1 = its last);
// the last covering CTA to finish (per-tile counter, self-resetting) folds
// them. Roles (192 threads): warp 0 TMA, warp 1 UMMA issuer + TMEM owner,
// warps 2-5 epilogue (warp w drains TMEM lanes 32 (w % 4) .. +31 = features).
struct WskArgs {
  void* y;
  float* ws;        // [gridDim.x][2][Mp][128] fp32 partials
  int32_t* cnt;     // [N / 128] arrival counters (zero between launches)
  int32_t M, Mp, N, K;
  int32_t f32_out;
  int32_t stages;
};

__device__ __forceinline__ void epi_bar_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

__global__ void __launch_bounds__(192, 1)
    wgemm_sk_kernel(const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap xmap, WskArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int Mp = a.Mp;
  const uint32_t stage_bytes = kWBytes + static_cast<uint32_t>(Mp) * 128;
  const int S = a.stages;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * stage_bytes);
  uint64_t* full = bars;                       // [S]
  uint64_t* empty = bars + kMaxStages;         // [S]
  uint64_t* acc_full = bars + 2 * kMaxStages;  // [2]
  uint64_t* acc_empty = acc_full + 2;          // [2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  int* s_last = reinterpret_cast<int*>(tslot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int C = a.K / kKc;          // K chunks per tile
  const int U = (a.N / kFeat) * C;  // units
  const int W = (U + static_cast<int>(gridDim.x) - 1) / static_cast<int>(gridDim.x);
  const int u0 = static_cast<int>(blockIdx.x) * W;
  const int u1 = min(U, u0 + W);
  const int n = max(0, u1 - u0);

  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&acc_full[i], 1);
      tc::mbar_init(&acc_empty[i], 128);
    }
    tc::fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&wmap);
    tc::prefetch_tmap(&xmap);
  }
  if (warp == 1) {
    if (Mp <= 64) tc::tmem_alloc<128>(tslot);
    else if (Mp <= 128) tc::tmem_alloc<256>(tslot);
    else tc::tmem_alloc<512>(tslot);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer --
    // weights first (independent of the previous kernel: before the PDL wait)
    const int pre = min(S, n);
    if (tc::elect_one_sync()) {
      for (int i = 0; i < pre; ++i) {
        const int u = u0 + i;
        tc::mbar_expect_tx(&full[i], stage_bytes);
        tc::tma_load_2d(smem + i * stage_bytes, &wmap, &full[i], (u % C) * kKc, (u / C) * kFeat);
      }
    }
    __syncwarp();
    pdl_wait();
    for (int i = 0; i < n; ++i) {
      const int st = i % S;
      const int u = u0 + i;
      if (i >= S) tc::mbar_wait(&empty[st], ((i / S) - 1) & 1);
      if (tc::elect_one_sync()) {
        uint8_t* sw = smem + st * stage_bytes;
        if (i >= pre) {
          tc::mbar_expect_tx(&full[st], stage_bytes);
          tc::tma_load_2d(sw, &wmap, &full[st], (u % C) * kKc, (u / C) * kFeat);
        }
        tc::tma_load_2d(sw + kWBytes, &xmap, &full[st], (u % C) * kKc, 0);
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // -------------------------------------------------------- MMA issuer --
    const uint32_t idesc = tc::idesc_bf16_f32(kFeat, Mp, false, false);
    const uint32_t base = tc::smem_u32(smem);
    int seg = 0;
    for (int i = 0; i < n; ++i) {
      const int st = i % S;
      const int u = u0 + i;
      const bool first = i == 0 || u % C == 0;
      const bool last = i == n - 1 || u % C == C - 1;
      const int b = seg & 1;
      if (first && seg >= 2) tc::mbar_wait(&acc_empty[b], ((seg >> 1) - 1) & 1);
      tc::mbar_wait(&full[st], (i / S) & 1);
      tc::tc_fence_after();
      if (tc::elect_one_sync()) {
        const uint32_t wa = base + st * stage_bytes, xa = wa + kWBytes;
        const uint32_t d = tmem + static_cast<uint32_t>(b * Mp);
#pragma unroll
        for (int ks = 0; ks < kKc / 16; ++ks)
          tc::umma_bf16_ss(d, tc::sdesc_sw128(wa + ks * 32, 16, 1024), tc::sdesc_sw128(xa + ks * 32, 16, 1024),
                           idesc, (!first || ks > 0) ? 1u : 0u);
        tc::umma_commit(&empty[st]);
        if (last) tc::umma_commit(&acc_full[b]);
      }
      __syncwarp();
      if (last) ++seg;
    }
  } else {
    // ---------------------------------------------------------- epilogue --
    const int f = (warp & 3) * 32 + lane;  // feature row of the tile = TMEM lane
    const uint32_t tl = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    int seg = 0;
    int u = u0;
    while (u < u1) {
      const int t = u / C;
      const int c_lo = u % C;
      const int seg_end = min(u1, (t + 1) * C);
      const bool full_tile = c_lo == 0 && seg_end == (t + 1) * C;
      const bool first_seg = u == u0;
      u = seg_end;
      const int b = seg & 1;
      tc::mbar_wait(&acc_full[b], (seg >> 1) & 1);
      tc::tc_fence_after();
      const int n0 = t * kFeat;
      float* part = a.ws + ((static_cast<size_t>(blockIdx.x) * 2 + (first_seg ? 0 : 1)) * Mp) * kFeat;
      for (int c0 = 0; c0 < Mp; c0 += 32) {
        float v[32];
        tc::tmem_ld32(tl + static_cast<uint32_t>(b * Mp + c0), v);
        tc::tmem_wait_ld();
        tc::reg_fence<32>(v);
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const int tok = c0 + k;
          if (tok >= a.M) break;
          if (full_tile) {
            const size_t o = static_cast<size_t>(tok) * a.N + n0 + f;
            if (a.f32_out) static_cast<float*>(a.y)[o] = v[k];
            else static_cast<__nv_bfloat16*>(a.y)[o] = __float2bfloat16(v[k]);
          } else {
            __stcg(part + static_cast<size_t>(tok) * kFeat + f, v[k]);
          }
        }
      }
      tc::tc_fence_before();
      tc::mbar_arrive(&acc_empty[b]);
      ++seg;
      if (!full_tile) {
        // the last CTA covering tile t folds its partials
        const int c_first = (t * C) / W, c_last = ((t + 1) * C - 1) / W;
        __threadfence();
        epi_bar_sync();
        if (threadIdx.x == 64) *s_last = atomicAdd(a.cnt + t, 1) == c_last - c_first;
        epi_bar_sync();
        if (*s_last) {
          __threadfence();
          // 16 tokens per pass: the partial loads of a pass are independent
          // (in flight together) instead of one L2 round trip per token
          for (int t0 = 0; t0 < a.M; t0 += 16) {
            float acc[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) acc[k] = 0.f;
            for (int cc = c_first; cc <= c_last; ++cc) {
              const int slot = cc * W >= t * C ? 0 : 1;
              const float* pp = a.ws + ((static_cast<size_t>(cc) * 2 + slot) * Mp + t0) * kFeat + f;
              float v[16];
#pragma unroll
              for (int k = 0; k < 16; ++k) v[k] = t0 + k < Mp ? __ldcg(pp + k * kFeat) : 0.f;
#pragma unroll
              for (int k = 0; k < 16; ++k) acc[k] += v[k];
            }
#pragma unroll
            for (int k = 0; k < 16; ++k) {
              if (t0 + k >= a.M) break;
              const size_t o = static_cast<size_t>(t0 + k) * a.N + n0 + f;
              if (a.f32_out) static_cast<float*>(a.y)[o] = acc[k];
              else static_cast<__nv_bfloat16*>(a.y)[o] = __float2bfloat16(acc[k]);
            }
          }
          if (threadIdx.x == 64) a.cnt[t] = 0;
        }
        epi_bar_sync();  // s_last is rewritten by the next cut tile
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 1) {
    if (Mp <= 64) tc::tmem_dealloc<128>(tmem);
    else if (Mp <= 128) tc::tmem_dealloc<256>(tmem);
    else tc::tmem_dealloc<512>(tmem);
  }
}

size_t wgemm_sk_smem_bytes(int Mp, int stages) {
  return static_cast<size_t>(stages) * (kWBytes + static_cast<size_t>(Mp) * 128) + 256 + 1024;
}

int wgemm_sk_stages(int Mp) {
  int s = kMaxStages;
  while (s > 2 && wgemm_sk_smem_bytes(Mp, s) > 220 * 1024) --s;
  return s;
}

// Stream-K launch: grid = `ctas` (<= SMs, one resident CTA each), ws >= ctas x
// 2 x Mp x 128 floats, cnt >= N / 128 zeroed ints.
void wgemm_sk(const CUtensorMap* wmap, const CUtensorMap* xmap, void* y, float* ws, int32_t* cnt, int M, int Mp,
              int N, int K, bool f32_out, int ctas, cudaStream_t s) {
  smem_attr_once(reinterpret_cast<const void*>(wgemm_sk_kernel), 227 * 1024);
  WskArgs a{};
  a.y = y;
  a.ws = ws;
  a.cnt = cnt;
  a.M = M;
  a.Mp = Mp;
  a.N = N;
  a.K = K;
  a.f32_out = f32_out ? 1 : 0;
  a.stages = wgemm_sk_stages(Mp);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(ctas, 1, 1);
  cfg.blockDim = dim3(192, 1, 1);
  cfg.dynamicSmemBytes = wgemm_sk_smem_bytes(Mp, a.stages);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL: weights stream during the producer's tail
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, wgemm_sk_kernel, *wmap, *xmap, a);
}

size_t wgemm_smem_bytes(int Mp, int stages) {
  const size_t stage = kWBytes + static_cast<size_t>(Mp) * 128;
  const size_t ring = stages * stage, red = static_cast<size_t>(Mp) * kFeat * 4;
  return (ring > red ? ring : red) + 256 + 1024;
}

// Ring depth that fits `budget` bytes of shared memory (>= 2).
int wgemm_stages(int Mp, size_t budget) {
  const size_t stage = kWBytes + static_cast<size_t>(Mp) * 128;
  int s = kMaxStages;
  while (s > 2 && wgemm_smem_bytes(Mp, s) > budget) --s;
  return s;
}

bool wgemm_supported(int M, int N, int K) { return M >= 1 && M <= 256 && N % kFeat == 0 && K % kKc == 0; }

// Y[M, N] = X[M, K] . W[N, K]^T. wmap: W as [N rows][K] (box 64 x 128);
// xmap: X as [rows][K] (box 64 x Mp). splits x chunks covers K / 64; the K
// splits of a feature tile are one cluster.
void wgemm_tc(const CUtensorMap* wmap, const CUtensorMap* xmap, void* y, int M, int Mp, int N, int K, int splits,
              int stages, bool f32_out, cudaStream_t s) {
  smem_attr_once(reinterpret_cast<const void*>(wgemm_tc_kernel), 227 * 1024);
  WgemmArgs a{};
  a.y = y;
  a.M = M;
  a.Mp = Mp;
  a.N = N;
  a.K = K;
  const int total = K / kKc;
  a.chunks = (total + splits - 1) / splits;
  a.splits = (total + a.chunks - 1) / a.chunks;
  a.f32_out = f32_out ? 1 : 0;
  a.stages = stages;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(N / kFeat, a.splits, 1);
  cfg.blockDim = dim3(kGemmThreads, 1, 1);
  cfg.dynamicSmemBytes = wgemm_smem_bytes(Mp, stages);
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 1;
  at[0].val.clusterDim.y = a.splits;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL: see the producer
  at[1].val.programmaticStreamSerializationAllowed = 1;
  // PDL off by default: in a decode graph the early-resident K7 CTAs (one per
  // SM, 227 KB of smem) hold SMs the producer's last CTAs need, which cost
  // more than the weight prefetch won (39 x 4.2K step 7.144 -> 7.093 ms
  // without it, profiles/r2/SUMMARY.md); CS_K7_PDL=1 re-enables it
  static const bool no_pdl = [] {
    const char* v = std::getenv("CS_K7_PDL");
    return !(v && v[0] == '1');
  }();
  cfg.attrs = at;
  cfg.numAttrs = no_pdl ? 1 : 2;
  cudaLaunchKernelEx(&cfg, wgemm_tc_kernel, *wmap, *xmap, a);
}

// Clusters of `splits` CTAs (each `smem` bytes) that can be resident at once.
int wgemm_max_clusters(int Mp, int stages, int splits) {
  smem_attr_once(reinterpret_cast<const void*>(wgemm_tc_kernel), 227 * 1024);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(1, splits, 1);
  cfg.blockDim = dim3(kGemmThreads, 1, 1);
  cfg.dynamicSmemBytes = wgemm_smem_bytes(Mp, stages);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 1;
  at[0].val.clusterDim.y = splits;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, wgemm_tc_kernel, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

}  // namespace csk
