// K8: the token-parallel projections of a layer (qkv, o_proj, gate|up, down)
// at prefill-sized M on the 5th-generation tensor cores, replacing the cuBLAS
// GEMMs that were 64% of the co-serving step (reference
// stand-in: the k1*P linear term of oracle_latency, proj/src/perf_model.cpp:
// 56-65).
//
//   Y[M, N] = X[M, K] . W[N, K]^T      bf16 in, fp32 accumulate, bf16 (or fp32) out
//
// CTA pair (cluster of 2, tcgen05 cta_group::2): one 256 x 256 output tile
// per pair and step; each CTA stages 128 rows of X and 128 rows of W per
// 64-element K block (TMA, 128-B swizzle), the leader's single issuing lane
// runs UMMA M=256 N=256 K=16 over both CTAs' shared memory, and each CTA's
// TMEM receives its 128 rows x 256 fp32 columns. Two accumulators (512 TMEM
// columns) let the epilogue of tile i overlap the main loop of tile i+1.
// Persistent: one pair per two SMs walks tiles t = pair, pair + pairs, ...
// M-fastest, so the X panel stays in L2 while W streams once.
//
// M is read on the device (IterDesc.n_tok_cur when `m_dev` is given): a
// layer-wise preemption that truncates the batch to its online prefix on the
// device (safepoint kernel) shrinks every later GEMM of the same forward
// without the host -- tiles past the live rows are never computed.
//
// Warp roles (192 threads per CTA): warp 0 TMA producer (both CTAs, elected
// lane), warp 1 MMA issuer (leader CTA, elected lane) + TMEM owner, warps 2-5
// epilogue (warp w drains TMEM lanes 32*(w%4) .. +31: one thread = one row).
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "tc.cuh"

namespace csk {

namespace {

constexpr int kPfRows = 128;                       // rows of X per CTA (UMMA M = 256 per pair)
constexpr int kPfN = 256;                          // UMMA N (output columns per pair tile)
constexpr int kPfBk = 64;                          // K elements per stage
constexpr int kPfStages = 6;
constexpr int kPfABytes = kPfRows * kPfBk * 2;     // 16 KB
constexpr int kPfBBytes = (kPfN / 2) * kPfBk * 2;  // 16 KB (this CTA's half of the N rows)
constexpr int kPfStageBytes = kPfABytes + kPfBBytes;
constexpr int kPfThreads = 192;
constexpr int kPfSmem = kPfStages * kPfStageBytes + 256 + 1024;

struct PfArgs {
  void* y;
  const int32_t* m_dev;  // device row count (IterDesc.n_tok_cur) or null
  int32_t M, N, K;       // M: host upper bound (rows of the X tensor map)
  int32_t f32_out;
  int32_t band;          // m-tiles per raster band (L2 reuse of the X and W panels)
  int32_t swiglu;        // W = gate|up interleaved in 128-row blocks: y = silu(gate) * up [M, N / 2]
  PfExtra ex;            // fused residual add / RoPE + KV append (common.cuh)
};

// Tile t -> (m tile, n tile): bands of `band` m-tiles, m fastest inside a
// band, bands in order. The ~74 tiles in flight then touch `band` X panels
// and ~74/band W panels instead of every X panel (M-fastest over all m-tiles
// re-streams X from DRAM once per W panel group when X exceeds the L2).
__device__ __forceinline__ void pf_tile(int t, int m_tiles, int n_tiles, int band, int& m, int& n) {
  const int per = band * n_tiles;
  const int b = t / per;
  const int gm = min(band, m_tiles - b * band);
  const int r = t - b * per;
  m = b * band + r % gm;
  n = r / gm;
}

}  // namespace

__global__ void __launch_bounds__(kPfThreads, 1)
    gemm_pf_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap wmap, PfArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kPfStages * kPfStageBytes);  // [S] (leader's used)
  uint64_t* empty = full + kPfStages;                                                // [S]
  uint64_t* tfull = empty + kPfStages;                                               // [2]
  uint64_t* tempty = tfull + 2;                                                      // [2] (leader's used)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = tc::cluster_ctarank();
  const int pair = blockIdx.x >> 1, pairs = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kPfStages; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&tfull[i], 1);
      tc::mbar_init(&tempty[i], 8);  // 4 epilogue warps x 2 CTAs
    }
    tc::fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&xmap);
    tc::prefetch_tmap(&wmap);
  }
  if (warp == 1) tc::tmem_alloc2<512>(tslot);
  tc::tc_fence_before();
  tc::cluster_arrive_wait();  // barrier inits + TMEM address visible pair-wide
  tc::tc_fence_after();
  const uint32_t tmem = *tslot;

  pdl_wait();  // X (and the live row count) come from the previous kernel
  int M = a.M;
  if (a.m_dev != nullptr) M = min(M, *a.m_dev);
  const int m_tiles = (M + 2 * kPfRows - 1) / (2 * kPfRows);
  const int n_tiles = a.N / kPfN;
  const int tiles = m_tiles * n_tiles;
  const int KB = a.K / kPfBk;

  if (warp == 0) {
    // ---------------------------------------------------------- TMA producer --
    const uint32_t full0 = tc::mapa(tc::smem_u32(&full[0]), 0);  // leader's barriers
    int it = 0;
    for (int t = pair; t < tiles; t += pairs) {
      int tm, tn;
      pf_tile(t, m_tiles, n_tiles, a.band, tm, tn);
      const int mrow = tm * 2 * kPfRows + static_cast<int>(rank) * kPfRows;
      const int nrow = tn * kPfN + static_cast<int>(rank) * (kPfN / 2);
      for (int kb = 0; kb < KB; ++kb, ++it) {
        const int st = it % kPfStages;
        tc::mbar_wait(&empty[st], ((it / kPfStages) & 1) ^ 1);
        if (tc::elect_one_sync()) {
          uint8_t* sa = smem + st * kPfStageBytes;
          if (rank == 0) tc::mbar_expect_tx(&full[st], 2 * kPfStageBytes);
          const uint32_t fb = full0 + st * 8;
          tc::tma_load_2d_pair(sa, &xmap, fb, kb * kPfBk, mrow);
          tc::tma_load_2d_pair(sa + kPfABytes, &wmap, fb, kb * kPfBk, nrow);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    // ----------------------------------------------------------- MMA issuer --
    if (rank == 0) {
      const uint32_t idesc = tc::idesc_bf16_f32(2 * kPfRows, kPfN, false, false);
      const uint32_t base = tc::smem_u32(smem);
      int it = 0, i = 0;
      for (int t = pair; t < tiles; t += pairs, ++i) {
        const int acc = i & 1;
        tc::mbar_wait(&tempty[acc], ((i >> 1) & 1) ^ 1);
        tc::tc_fence_after();
        const uint32_t d = tmem + acc * kPfN;
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int st = it % kPfStages;
          tc::mbar_wait(&full[st], (it / kPfStages) & 1);
          tc::tc_fence_after();
          if (tc::elect_one_sync()) {
            const uint32_t sa = base + st * kPfStageBytes, sb = sa + kPfABytes;
#pragma unroll
            for (int k = 0; k < kPfBk / 16; ++k)
              tc::umma2_bf16_ss(d, tc::sdesc_sw128(sa + k * 32, 16, 1024), tc::sdesc_sw128(sb + k * 32, 16, 1024),
                                idesc, (kb > 0 || k > 0) ? 1u : 0u);
            tc::umma2_commit_mc(&empty[st], 0x3);
            if (kb == KB - 1) tc::umma2_commit_mc(&tfull[acc], 0x3);
          }
          __syncwarp();
        }
      }
    }
  } else {
    // ------------------------------------------------------------- epilogue --
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    const uint32_t tempty0 = tc::mapa(tc::smem_u32(&tempty[0]), 0);
    int i = 0;
    for (int t = pair; t < tiles; t += pairs, ++i) {
      const int acc = i & 1;
      tc::mbar_wait(&tfull[acc], (i >> 1) & 1);
      tc::tc_fence_after();
      int tm, tn;
      pf_tile(t, m_tiles, n_tiles, a.band, tm, tn);
      const int row = tm * 2 * kPfRows + static_cast<int>(rank) * kPfRows + q * 32 + lane;
      const int n0 = tn * kPfN;
      const uint32_t tl = tmem + (static_cast<uint32_t>(q * 32) << 16) + acc * kPfN;
      if (a.swiglu) {
        // fused SwiGLU: TMEM columns [0, 128) = gate, [128, 256) = up of the
        // same 128 FFN features; rounded to bf16 first, as the unfused path
        // stores gate|up, then silu(g) * u -> act[row, tn * 128 + c]
#pragma unroll 1
        for (int c = 0; c < kPfN / 2; c += 32) {
          float g[32], u[32];
          tc::tmem_ld32(tl + c, g);
          tc::tmem_ld32(tl + kPfN / 2 + c, u);
          tc::tmem_wait_ld();
          tc::reg_fence<32>(g);
          tc::reg_fence<32>(u);
          if (row < M) {
            uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(a.y) +
                                                  static_cast<size_t>(row) * (a.N / 2) + tn * (kPfN / 2) + c);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              float o[8];
#pragma unroll
              for (int t = 0; t < 8; ++t) {
                const float gf = __bfloat162float(__float2bfloat16(g[8 * j + t]));
                const float uf = __bfloat162float(__float2bfloat16(u[8 * j + t]));
                o[t] = gf / (1.f + __expf(-gf)) * uf;
              }
              dst[j] = make_uint4(pack_bf16(o[0], o[1]), pack_bf16(o[2], o[3]), pack_bf16(o[4], o[5]),
                                  pack_bf16(o[6], o[7]));
            }
          }
        }
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive_cluster(tempty0 + acc * 8);
        continue;
      }
      if (a.ex.rope_tab != nullptr) {
        // qkv + RoPE + KV append: this 256-column tile = two heads of 128
        // (q heads rotated in place in y; k heads rotated and v heads copied
        // into the pool). Values are rounded to bf16 first, as the unfused
        // path stores qkv, then rotated exactly as rope_append does.
        const int D = 128, half = 64;
        int slot = 0, blk = 0, off = 0;
        if (row < M) {
          slot = a.ex.tok_slot[row];
          blk = slot >> 4;
          off = slot & 15;
        }
        const size_t layer_elems = static_cast<size_t>(2) * a.ex.hkv * 16 * D;
        __nv_bfloat16* kv_base = a.ex.pool + (static_cast<size_t>(blk) * a.ex.num_layers + a.ex.layer) * layer_elems;
#pragma unroll 1
        for (int hh = 0; hh < 2; ++hh) {
          const int h = (n0 + hh * D) / D;  // head index in the q | k | v layout
#pragma unroll 1
          for (int jc = 0; jc < half; jc += 32) {
            float va[32], vb[32];
            tc::tmem_ld32(tl + hh * D + jc, va);
            tc::tmem_ld32(tl + hh * D + half + jc, vb);
            tc::tmem_wait_ld();
            tc::reg_fence<32>(va);
            tc::reg_fence<32>(vb);
            if (row >= M) continue;
            __nv_bfloat16* dst;
            if (h < a.ex.hq) dst = static_cast<__nv_bfloat16*>(a.y) + static_cast<size_t>(row) * a.N + h * D;
            else if (h < a.ex.hq + a.ex.hkv) dst = kv_base + (static_cast<size_t>(h - a.ex.hq) * 16 + off) * D;
            else dst = kv_base + (static_cast<size_t>(a.ex.hkv + h - a.ex.hq - a.ex.hkv) * 16 + off) * D;
            const bool rot = h < a.ex.hq + a.ex.hkv;
            const float2* tab = a.ex.rope_tab + static_cast<size_t>(row) * half + jc;
#pragma unroll
            for (int j = 0; j < 32; j += 8) {
              uint32_t w1[4], w2[4];
#pragma unroll
              for (int k = 0; k < 8; k += 2) {
                float y1[2], y2[2];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                  const float x1 = __bfloat162float(__float2bfloat16(va[j + k + u]));
                  const float x2 = __bfloat162float(__float2bfloat16(vb[j + k + u]));
                  if (rot) {  // the same operations as rope_append_kernel
                    const float2 r = tab[j + k + u];
                    y1[u] = __fmaf_rn(x1, r.x, -__fmul_rn(x2, r.y));
                    y2[u] = __fmaf_rn(x2, r.x, __fmul_rn(x1, r.y));
                  } else {
                    y1[u] = x1;
                    y2[u] = x2;
                  }
                }
                w1[k / 2] = pack_bf16(y1[0], y1[1]);
                w2[k / 2] = pack_bf16(y2[0], y2[1]);
              }
              *reinterpret_cast<uint4*>(dst + jc + j) = make_uint4(w1[0], w1[1], w1[2], w1[3]);
              *reinterpret_cast<uint4*>(dst + half + jc + j) = make_uint4(w2[0], w2[1], w2[2], w2[3]);
            }
          }
        }
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive_cluster(tempty0 + acc * 8);
        continue;
      }
#pragma unroll 1
      for (int c = 0; c < kPfN; c += 32) {
        float v[32];
        tc::tmem_ld32(tl + c, v);
        tc::tmem_wait_ld();
        tc::reg_fence<32>(v);
        if (row < M && a.ex.resid != nullptr) {
          // residual add fused: x = x + bf16(acc), in place
          uint4* xr = reinterpret_cast<uint4*>(a.ex.resid + static_cast<size_t>(row) * a.N + n0 + c);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint4 xo = xr[j];
            const __nv_bfloat16* xe = reinterpret_cast<const __nv_bfloat16*>(&xo);
            float o[8];
#pragma unroll
            for (int t = 0; t < 8; ++t)
              o[t] = __bfloat162float(xe[t]) + __bfloat162float(__float2bfloat16(v[8 * j + t]));
            xr[j] = make_uint4(pack_bf16(o[0], o[1]), pack_bf16(o[2], o[3]), pack_bf16(o[4], o[5]),
                               pack_bf16(o[6], o[7]));
          }
        } else if (row < M) {
          if (a.f32_out) {
            float4* dst = reinterpret_cast<float4*>(static_cast<float*>(a.y) + static_cast<size_t>(row) * a.N + n0 + c);
#pragma unroll
            for (int j = 0; j < 8; ++j) dst[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          } else {
            uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(a.y) + static_cast<size_t>(row) * a.N + n0 + c);
#pragma unroll
            for (int j = 0; j < 4; ++j)
              dst[j] = make_uint4(pack_bf16(v[8 * j], v[8 * j + 1]), pack_bf16(v[8 * j + 2], v[8 * j + 3]),
                                  pack_bf16(v[8 * j + 4], v[8 * j + 5]), pack_bf16(v[8 * j + 6], v[8 * j + 7]));
          }
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive_cluster(tempty0 + acc * 8);
    }
  }

  // ------------------------------------------------------------- teardown --
  tc::tc_fence_before();
  tc::cluster_arrive_wait();
  tc::tc_fence_after();
  if (warp == 1) tc::tmem_dealloc2<512>(tmem);
}

bool gemm_pf_supported(int N, int K) { return N % kPfN == 0 && K % kPfBk == 0 && K >= kPfBk; }

int gemm_pf_rows_box() { return kPfRows; }

// Y[M, N] = X[M, K] . W[N, K]^T. xmap: X as [>= M rows][K], wmap: W as
// [N][K], both 64 x 128 boxes with 128-B swizzle. M is the host bound (grid
// size); m_dev, when set, the live row count read by the kernel.
void gemm_pf(const CUtensorMap* xmap, const CUtensorMap* wmap, void* y, int M, const int32_t* m_dev, int N, int K,
             bool f32_out, int sms, cudaStream_t s, bool swiglu, const PfExtra* ex) {
  smem_attr_once(reinterpret_cast<const void*>(gemm_pf_kernel), kPfSmem);
  PfArgs a{};
  if (ex) a.ex = *ex;
  a.y = y;
  a.m_dev = m_dev;
  a.M = M;
  a.N = N;
  a.K = K;
  a.f32_out = f32_out ? 1 : 0;
  a.swiglu = swiglu ? 1 : 0;
  static const int band_env = [] {
    const char* v = std::getenv("CS_PF_BAND");
    return v ? std::atoi(v) : 0;
  }();
  a.band = band_env > 0 ? band_env : 16;  // tools/gemm_pf_bench.cu sweep: 16 best at M 4096-8192
  const int tiles = ((M + 2 * kPfRows - 1) / (2 * kPfRows)) * (N / kPfN);
  const int pairs = std::max(1, std::min(sms / 2, tiles));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * pairs, 1, 1);
  cfg.blockDim = dim3(kPfThreads, 1, 1);
  cfg.dynamicSmemBytes = kPfSmem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  cudaLaunchKernelEx(&cfg, gemm_pf_kernel, *xmap, *wmap, a);
}

}  // namespace csk
