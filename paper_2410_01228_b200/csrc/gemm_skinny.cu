// Weight-streaming GEMM for few token rows (decode steps, SURVEY.md 8f rank 2
// "rest of the layer"): Y[M, N] = X[M, K] * W[N, K]^T with M <= 64, bf16 in,
// fp32 accumulate, bf16 or fp32 out. At M <= 64 every linear layer of the
// decode step is bound by reading W once from HBM; the library's kernels for
// these shapes reach 2-5.4 TB/s (profiles/r1), this one streams W at the HBM
// roofline:
//   * CTA = 64 output columns x a K range (split-K sized so ~4 CTAs/SM are
//     resident), 4 warps, each warp 16 columns x all M rows;
//   * 4-stage cp.async ring of [64 cols][64 k] W tiles (8 KB, 16-B coalesced
//     loads, XOR-swizzled) and the matching [M][64] X tiles;
//   * mma.sync m16n8k16 (the contraction is ~free next to the bytes);
//   * split-K partials in fp32 workspace, folded by the last-arriving CTA of
//     each column tile (self-resetting arrival counter).
#include <algorithm>

#include "common.cuh"

namespace csk {

namespace {

constexpr int kNT = 64;      // output columns per CTA
constexpr int kKC = 64;      // k per stage
constexpr int kStages = 4;
constexpr int kThreads = 128;

template <int MT>
struct SkLayout {
  static constexpr int w = 0;                                   // [stage][64 n][64 k]
  static constexpr int x = w + kStages * kNT * kKC * 2;         // [stage][MT*16 m][64 k]
  static constexpr int bytes = x + kStages * MT * 16 * kKC * 2;
};

__device__ __forceinline__ uint32_t swz64(int r, int c) {  // row of 64 bf16 = 8 chunks of 16 B
  return static_cast<uint32_t>(r * 128 + ((c ^ (r & 7)) << 4));
}

}  // namespace

template <int MT, bool OUT_F32>
__global__ void __launch_bounds__(kThreads) gemm_skinny_kernel(const __nv_bfloat16* __restrict__ X,
                                                               const __nv_bfloat16* __restrict__ W, void* Y, int N,
                                                               int K, int kchunks_per_split, float* ws,
                                                               int32_t* cnt) {
  using Lay = SkLayout<MT>;
  constexpr int M = MT * 16;
  extern __shared__ __align__(128) uint8_t smem[];
  const int nt = blockIdx.x, split = blockIdx.y, n_split = gridDim.y;
  const int n0 = nt * kNT;
  const int c0 = split * kchunks_per_split;
  const int n_ch = min(K / kKC - c0, kchunks_per_split);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  auto load_stage = [&](int ch, int st) {
    const int k0 = (c0 + ch) * kKC;
    uint8_t* sw = smem + Lay::w + st * kNT * kKC * 2;
    uint8_t* sx = smem + Lay::x + st * M * kKC * 2;
#pragma unroll
    for (int i = 0; i < (kNT * 8) / kThreads; ++i) {  // 64 rows x 8 chunks
      const int c = threadIdx.x + i * kThreads;
      const int r = c >> 3, u = c & 7;
      cp_async16(sw + swz64(r, u), W + static_cast<size_t>(n0 + r) * K + k0 + u * 8);
    }
#pragma unroll
    for (int i = 0; i < (M * 8 + kThreads - 1) / kThreads; ++i) {
      const int c = threadIdx.x + i * kThreads;
      if (c < M * 8) {
        const int r = c >> 3, u = c & 7;
        cp_async16(sx + swz64(r, u), X + static_cast<size_t>(r) * K + k0 + u * 8);
      }
    }
  };

  float acc[MT][2][4];
#pragma unroll
  for (int a = 0; a < MT; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = acc[a][b][2] = acc[a][b][3] = 0.f;

#pragma unroll
  for (int st = 0; st < kStages - 1; ++st) {
    if (st < n_ch) load_stage(st, st);
    cp_async_commit();
  }
  for (int ch = 0; ch < n_ch; ++ch) {
    const int nxt = ch + kStages - 1;
    if (nxt < n_ch) load_stage(nxt, nxt % kStages);
    cp_async_commit();
    cp_async_wait<kStages - 1>();
    __syncthreads();
    const uint8_t* sw = smem + Lay::w + (ch % kStages) * kNT * kKC * 2;
    const uint8_t* sx = smem + Lay::x + (ch % kStages) * M * kKC * 2;
#pragma unroll
    for (int ks = 0; ks < kKC / 16; ++ks) {
      // B: this warp's 16 columns (two n8 tiles) x k16, rows of W = columns
      uint32_t b0, b1, b2, b3;
      {
        const int mi = lane >> 3;
        const int row = warp * 16 + (mi >> 1) * 8 + (lane & 7);
        ldmatrix_x4(b0, b1, b2, b3, sw + swz64(row, ks * 2 + (mi & 1)));
      }
#pragma unroll
      for (int a = 0; a < MT; ++a) {
        uint32_t af[4];
        ldmatrix_x4(af[0], af[1], af[2], af[3], sx + swz64(a * 16 + (lane & 15), ks * 2 + (lane >> 4)));
        mma_bf16_16816(acc[a][0], af, b0, b1);
        mma_bf16_16816(acc[a][1], af, b2, b3);
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();

  // fragment (a, b, i): row a*16 + lane/4 (+8 for i >= 2), col warp*16 + b*8 + (lane%4)*2 + (i&1)
  const int gid = lane >> 2, tig = lane & 3;
  auto store = [&](int row, int col, float v0, float v1) {
    if (OUT_F32) {
      *reinterpret_cast<float2*>(static_cast<float*>(Y) + static_cast<size_t>(row) * N + col) = make_float2(v0, v1);
    } else {
      *reinterpret_cast<uint32_t*>(static_cast<__nv_bfloat16*>(Y) + static_cast<size_t>(row) * N + col) =
          pack_bf16(v0, v1);
    }
  };
  if (n_split == 1) {
#pragma unroll
    for (int a = 0; a < MT; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const int col = n0 + warp * 16 + b * 8 + tig * 2;
        store(a * 16 + gid, col, acc[a][b][0], acc[a][b][1]);
        store(a * 16 + gid + 8, col, acc[a][b][2], acc[a][b][3]);
      }
    return;
  }
  // split-K: partial tile -> workspace [split][M][64]; the last CTA folds
  float* part = ws + (static_cast<size_t>(nt) * n_split + split) * M * kNT;
#pragma unroll
  for (int a = 0; a < MT; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const int cl = warp * 16 + b * 8 + tig * 2;
      *reinterpret_cast<float2*>(part + (a * 16 + gid) * kNT + cl) = make_float2(acc[a][b][0], acc[a][b][1]);
      *reinterpret_cast<float2*>(part + (a * 16 + gid + 8) * kNT + cl) = make_float2(acc[a][b][2], acc[a][b][3]);
    }
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&cnt[nt], 1) == n_split - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const float* base = ws + static_cast<size_t>(nt) * n_split * M * kNT;
  for (int idx = threadIdx.x * 2; idx < M * kNT; idx += kThreads * 2) {
    float v0 = 0.f, v1 = 0.f;
    for (int sp = 0; sp < n_split; ++sp) {
      const float2 t = __ldcg(reinterpret_cast<const float2*>(base + static_cast<size_t>(sp) * M * kNT + idx));
      v0 += t.x;
      v1 += t.y;
    }
    store(idx / kNT, n0 + idx % kNT, v0, v1);
  }
  if (threadIdx.x == 0) cnt[nt] = 0;
}

// Launches Y = X W^T for M <= 64 rows (rows padded up to a multiple of 16
// are computed from whatever the X buffer holds and written to Y: both
// buffers must have 16-row slack). False if the shape is not supported.
bool gemm_skinny(const __nv_bfloat16* X, const __nv_bfloat16* W, void* Y, int M, int N, int K, bool out_f32,
                 float* ws, size_t ws_floats, int32_t* cnt, int cnt_len, int sms, cudaStream_t s) {
  if (M < 1 || M > 64 || N % kNT || K % kKC) return false;
  const int MT = (M + 15) / 16;
  const int tiles = N / kNT, chunks = K / kKC;
  int split = std::max(1, std::min(chunks / 4, (4 * sms + tiles - 1) / tiles));
  const int cps = (chunks + split - 1) / split;
  split = (chunks + cps - 1) / cps;
  if (split > 1 && (static_cast<size_t>(tiles) * split * MT * 16 * kNT > ws_floats || tiles > cnt_len)) return false;
#define CS_SK_CASE(MM)                                                                                        \
  if (MT == MM) {                                                                                             \
    const int smem = SkLayout<MM>::bytes;                                                                     \
    static bool attr = false;                                                                                 \
    if (!attr) {                                                                                              \
      cudaFuncSetAttribute(gemm_skinny_kernel<MM, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
      cudaFuncSetAttribute(gemm_skinny_kernel<MM, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);  \
      attr = true;                                                                                            \
    }                                                                                                         \
    if (out_f32)                                                                                              \
      gemm_skinny_kernel<MM, true><<<dim3(tiles, split), kThreads, smem, s>>>(X, W, Y, N, K, cps, ws, cnt);  \
    else                                                                                                      \
      gemm_skinny_kernel<MM, false><<<dim3(tiles, split), kThreads, smem, s>>>(X, W, Y, N, K, cps, ws, cnt); \
    return true;                                                                                              \
  }
  CS_SK_CASE(1)
  CS_SK_CASE(2)
  CS_SK_CASE(3)
  CS_SK_CASE(4)
#undef CS_SK_CASE
  return false;
}

}  // namespace csk
