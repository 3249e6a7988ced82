// Paged attention over the block-table-indexed KV pool.
//
// K1 attn_decode: single-query rows (decode entries and 1-token chunks) --
//   query position p attends keys [0, p]. One CTA per (entry, KV head,
//   split); the G query heads of the KV group are the MMA's M rows, so every
//   K/V byte is read from HBM once per group. Each warp streams whole 16-token
//   pages through a private 2-stage cp.async ring (16-byte coalesced loads,
//   XOR-swizzled smem) and keeps its own online softmax; warps and splits are
//   merged at the end. HBM-bound: the contractions run on mma.sync only to
//   keep the instruction count far below the byte rate.
// K2 (multi-query chunks: prefill / recompute) runs on tcgen05: attn_tc.cu.
#include <cuda.h>

#include "common.cuh"

namespace csk {

namespace {

constexpr int kPage = 16;

__device__ __forceinline__ const __nv_bfloat16* kv_page(const AttnParams& p, int32_t block, int kvh, int which,
                                                         int D) {
  const size_t layer_elems = static_cast<size_t>(2) * p.hkv * kPage * D;
  return p.pool + (static_cast<size_t>(block) * p.num_layers + p.layer) * layer_elems +
         (static_cast<size_t>(which) * p.hkv + kvh) * kPage * D;
}

template <int D>
__device__ __forceinline__ void load_page_async(uint8_t* sK, uint8_t* sV, const __nv_bfloat16* k,
                                                const __nv_bfloat16* v, int lane) {
  constexpr int CH = D / 8;  // 16-byte chunks per row
#pragma unroll
  for (int i = 0; i < (kPage * CH) / 32; ++i) {
    const int c = lane + 32 * i;
    const int r = c / CH, ch = c % CH;
    cp_async16(sK + swz<D>(r, ch), k + r * D + ch * 8);
    cp_async16(sV + swz<D>(r, ch), v + r * D + ch * 8);
  }
}

// (x[d], x[d + D/2]) -> rotated pair, rounded to bf16 (rope_append's operations)
__device__ __forceinline__ void rope_pair(uint32_t& lo, uint32_t& hi, float2 c0, float2 c1) {
  const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(&lo);
  const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&hi);
  const float2 af = __bfloat1622float2(a), bf = __bfloat1622float2(b);
  const __nv_bfloat162 y1 = __floats2bfloat162_rn(__fmaf_rn(af.x, c0.x, -__fmul_rn(bf.x, c0.y)),
                                                  __fmaf_rn(af.y, c1.x, -__fmul_rn(bf.y, c1.y)));
  const __nv_bfloat162 y2 = __floats2bfloat162_rn(__fmaf_rn(bf.x, c0.x, __fmul_rn(af.x, c0.y)),
                                                  __fmaf_rn(bf.y, c1.x, __fmul_rn(af.y, c1.y)));
  lo = *reinterpret_cast<const uint32_t*>(&y1);
  hi = *reinterpret_cast<const uint32_t*>(&y2);
}

// q fragments (mma.sync A layout: this thread holds dims ks*16 + tig*2 + {0,1}
// and +8 of rows gid, gid + 8) rotated in registers; dim d pairs with d + D/2,
// i.e. fragment ks with ks + KS/2 at the same register index.
template <int D>
__device__ __forceinline__ void rope_q_frags(uint32_t (*qa)[4], int tig, const float2* tab) {
  constexpr int KS = D / 16;
#pragma unroll
  for (int ks = 0; ks < KS / 2; ++ks) {
#pragma unroll
    for (int h8 = 0; h8 < 2; ++h8) {
      const int d = ks * 16 + tig * 2 + h8 * 8;
      const float2 c0 = tab[d], c1 = tab[d + 1];
      rope_pair(qa[ks][2 * h8], qa[ks + KS / 2][2 * h8], c0, c1);          // row gid
      rope_pair(qa[ks][2 * h8 + 1], qa[ks + KS / 2][2 * h8 + 1], c0, c1);  // row gid + 8
    }
  }
}

// The new token of a decode row: k (rotated) and v of KV head kvh from the
// qkv row into the pool at the token's (block, slot). Called by the whole CTA
// that will read the pair's last page, before any of that page is loaded.
template <int D>
__device__ __forceinline__ void append_new_kv(const AttnParams& p, int row, int kvh) {
  const float2* tab = p.rope_tab + static_cast<size_t>(row) * (D / 2);
  const int slot = p.tok_slot[row];
  const int blk = slot >> 4, off = slot & 15;
  __nv_bfloat16* pool = const_cast<__nv_bfloat16*>(p.pool);
  const size_t layer_elems = static_cast<size_t>(2) * p.hkv * kPage * D;
  __nv_bfloat16* kb = pool + (static_cast<size_t>(blk) * p.num_layers + p.layer) * layer_elems;
  const __nv_bfloat16* src = p.qkv + static_cast<size_t>(row) * p.qkv_stride;
  const __nv_bfloat16* k = src + static_cast<size_t>(p.hq + kvh) * D;
  const __nv_bfloat16* v = src + static_cast<size_t>(p.hq + p.hkv + kvh) * D;
  __nv_bfloat16* kd = kb + (static_cast<size_t>(kvh) * kPage + off) * D;
  __nv_bfloat16* vd = kb + (static_cast<size_t>(p.hkv + kvh) * kPage + off) * D;
  for (int j = threadIdx.x; j < D / 4; j += blockDim.x) {  // 2 frequencies per thread, bf16x2
    uint32_t lo = *reinterpret_cast<const uint32_t*>(k + 2 * j);
    uint32_t hi = *reinterpret_cast<const uint32_t*>(k + 2 * j + D / 2);
    rope_pair(lo, hi, tab[2 * j], tab[2 * j + 1]);
    *reinterpret_cast<uint32_t*>(kd + 2 * j) = lo;
    *reinterpret_cast<uint32_t*>(kd + 2 * j + D / 2) = hi;
  }
  for (int j = threadIdx.x; j < D / 8; j += blockDim.x)
    reinterpret_cast<uint4*>(vd)[j] = reinterpret_cast<const uint4*>(v)[j];
  // the page is then read back through L2 by cp.async.cg: the stores must
  // be performed at GPU scope first
  __threadfence();
}

}  // namespace

// ------------------------------------------------------------------- K1 ----
template <int D, int G>
__global__ void __launch_bounds__(128) attn_decode_kernel(AttnParams p) {
  pdl_trigger();
  constexpr int KS = D / 16;
  constexpr int NTD = D / 8;
  constexpr int PB = kPage * D * 2;  // bytes per K (or V) page
  extern __shared__ __align__(128) uint8_t smem[];
  const int split = blockIdx.x, kvh = blockIdx.y, di = blockIdx.z;
  // split count and size live in the device descriptor so a captured graph
  // (grid sized for the bucket) serves every plan of its bucket
  const int S = p.desc->dec_splits;
  if (di >= p.desc->n_dec_cur || split >= S) return;
  const int pps = p.desc->dec_pps;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int ent = p.dec_ent[di];
  const int row = p.ent_q0[ent];
  const int kv_len = p.ent_kvlen[ent];
  const int n_pages = (kv_len + kPage - 1) / kPage;
  const int pg0 = split * pps;
  const int pg1 = min(n_pages, pg0 + pps);
  const int32_t* bt = p.block_table + p.ent_bt[ent];

  uint32_t qa[KS][4];
  {
    const __nv_bfloat16* q = p.qkv + static_cast<size_t>(row) * p.qkv_stride + static_cast<size_t>(kvh) * G * D;
    const int r0 = gid, r1 = gid + 8;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int d0 = ks * 16 + tig * 2;
      qa[ks][0] = r0 < G ? *reinterpret_cast<const uint32_t*>(q + r0 * D + d0) : 0u;
      qa[ks][1] = r1 < G ? *reinterpret_cast<const uint32_t*>(q + r1 * D + d0) : 0u;
      qa[ks][2] = r0 < G ? *reinterpret_cast<const uint32_t*>(q + r0 * D + d0 + 8) : 0u;
      qa[ks][3] = r1 < G ? *reinterpret_cast<const uint32_t*>(q + r1 * D + d0 + 8) : 0u;
    }
  }
  if (p.k1_rope) {
    rope_q_frags<D>(qa, tig, p.rope_tab + static_cast<size_t>(row) * (D / 2));
    if (pg0 < pg1 && pg1 == n_pages) {  // this split reads the last page: the new token's K/V first
      append_new_kv<D>(p, row, kvh);
      __syncthreads();
    }
  }

  float o[NTD][4];
#pragma unroll
  for (int i = 0; i < NTD; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

  uint8_t* wbuf = smem + warp * 4 * PB;  // [stage][K|V]
  int pg = pg0 + warp;
  if (pg < pg1) {
    load_page_async<D>(wbuf, wbuf + PB, kv_page(p, bt[pg], kvh, 0, D), kv_page(p, bt[pg], kvh, 1, D), lane);
  }
  cp_async_commit();
  int stage = 0;
  for (; pg < pg1; pg += 4) {
    const int nxt = pg + 4;
    if (nxt < pg1) {
      uint8_t* nb = wbuf + (stage ^ 1) * 2 * PB;
      load_page_async<D>(nb, nb + PB, kv_page(p, bt[nxt], kvh, 0, D), kv_page(p, bt[nxt], kvh, 1, D), lane);
    }
    cp_async_commit();
    cp_async_wait<1>();
    __syncwarp();
    const uint8_t* sK = wbuf + stage * 2 * PB;
    const uint8_t* sV = sK + PB;

    float s[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int mi = lane >> 3;
      const int tok = (mi >> 1) * 8 + (lane & 7);
      uint32_t b0, b1, b2, b3;
      ldmatrix_x4(b0, b1, b2, b3, sK + swz<D>(tok, ks * 2 + (mi & 1)));
      mma_bf16_16816(s[0], qa[ks], b0, b1);
      mma_bf16_16816(s[1], qa[ks], b2, b3);
    }
    const int base = pg * kPage;
    float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const bool ok = base + nt * 8 + tig * 2 + j < kv_len;
        s[nt][j] = ok ? s[nt][j] * p.scale_log2 : -INFINITY;
        s[nt][2 + j] = ok ? s[nt][2 + j] * p.scale_log2 : -INFINITY;
        mx0 = fmaxf(mx0, s[nt][j]);
        mx1 = fmaxf(mx1, s[nt][2 + j]);
      }
    }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
    const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
    const float al0 = exp2f(m0 - mn0), al1 = exp2f(m1 - mn1);
    m0 = mn0;
    m1 = mn1;
    uint32_t pa[4];
    float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const float p0 = exp2f(s[nt][0] - mn0), p1 = exp2f(s[nt][1] - mn0);
      const float p2 = exp2f(s[nt][2] - mn1), p3 = exp2f(s[nt][3] - mn1);
      rs0 += p0 + p1;
      rs1 += p2 + p3;
      pa[nt * 2 + 0] = pack_bf16(p0, p1);
      pa[nt * 2 + 1] = pack_bf16(p2, p3);
    }
    l0 = l0 * al0 + rs0;
    l1 = l1 * al1 + rs1;
#pragma unroll
    for (int i = 0; i < NTD; ++i) {
      o[i][0] *= al0;
      o[i][1] *= al0;
      o[i][2] *= al1;
      o[i][3] *= al1;
    }
#pragma unroll
    for (int nd = 0; nd < D / 16; ++nd) {
      const int mi = lane >> 3;
      const int tok = (mi & 1) * 8 + (lane & 7);
      uint32_t v0, v1, v2, v3;
      ldmatrix_x4_trans(v0, v1, v2, v3, sV + swz<D>(tok, nd * 2 + (mi >> 1)));
      mma_bf16_16816(o[nd * 2], pa, v0, v1);
      mma_bf16_16816(o[nd * 2 + 1], pa, v2, v3);
    }
    __syncwarp();
    stage ^= 1;
  }
  cp_async_wait<0>();
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);

  // Merge the 4 warps: [warp][16 rows] m, l and [warp][16][D] partial O.
  __syncthreads();
  float* sm_m = reinterpret_cast<float*>(smem);
  float* sm_l = sm_m + 4 * 16;
  float* sm_o = sm_l + 4 * 16;
  if (tig == 0) {
    sm_m[warp * 16 + gid] = m0;
    sm_m[warp * 16 + gid + 8] = m1;
    sm_l[warp * 16 + gid] = l0;
    sm_l[warp * 16 + gid + 8] = l1;
  }
#pragma unroll
  for (int nt = 0; nt < NTD; ++nt) {
    const int d = nt * 8 + tig * 2;
    sm_o[(warp * 16 + gid) * D + d] = o[nt][0];
    sm_o[(warp * 16 + gid) * D + d + 1] = o[nt][1];
    sm_o[(warp * 16 + gid + 8) * D + d] = o[nt][2];
    sm_o[(warp * 16 + gid + 8) * D + d + 1] = o[nt][3];
  }
  __syncthreads();
  const int SG = gridDim.x;  // workspace stride (launch grid)
  const size_t item = (static_cast<size_t>(di) * p.hkv + kvh) * SG + split;
  for (int idx = threadIdx.x; idx < G * D; idx += blockDim.x) {
    const int r = idx / D, d = idx % D;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < 4; ++w) M = fmaxf(M, sm_m[w * 16 + r]);
    float L = 0.f, O = 0.f;
    if (M != -INFINITY) {
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const float f = exp2f(sm_m[w * 16 + r] - M);
        L += sm_l[w * 16 + r] * f;
        O += sm_o[(w * 16 + r) * D + d] * f;
      }
    }
    if (S == 1) {
      p.out[static_cast<size_t>(row) * p.hq * D + static_cast<size_t>(kvh * G + r) * D + d] =
          __float2bfloat16(L > 0.f ? O / L : 0.f);
    } else {
      float* wm = p.ws + item * G * 2;
      float* wo = p.ws + static_cast<size_t>(gridDim.z) * p.hkv * SG * G * 2 + item * G * D;
      if (d == 0) {
        wm[r * 2] = M;
        wm[r * 2 + 1] = L;
      }
      wo[r * D + d] = O;
    }
  }
  if (S == 1) return;
  // Split-K merge, fused: the last CTA of this (entry, KV head) to finish
  // folds all S partials (no separate combine launch) and re-arms the counter.
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  int32_t* cnt = p.dec_cnt + static_cast<size_t>(di) * p.hkv + kvh;
  if (threadIdx.x == 0) s_last = atomicAdd(cnt, 1) == S - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  float* wgt = sm_m;         // [S][G] merge weights (smem reused: >= 128*8 floats)
  float* inv_l = sm_m + S * G;
  const size_t base_item = (static_cast<size_t>(di) * p.hkv + kvh) * SG;
  const float* wm = p.ws + base_item * G * 2;
  const float* wo = p.ws + static_cast<size_t>(gridDim.z) * p.hkv * SG * G * 2 + base_item * G * D;
  for (int r = warp; r < G; r += 4) {
    float M = -INFINITY;
    for (int sp = lane; sp < S; sp += 32) M = fmaxf(M, __ldcg(wm + (sp * G + r) * 2));
#pragma unroll
    for (int o = 16; o; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    float L = 0.f;
    for (int sp = lane; sp < S; sp += 32) {
      const float ms = __ldcg(wm + (sp * G + r) * 2);
      const float f = (M == -INFINITY || ms == -INFINITY) ? 0.f : exp2f(ms - M);
      wgt[sp * G + r] = f;
      L += __ldcg(wm + (sp * G + r) * 2 + 1) * f;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
    if (lane == 0) inv_l[r] = L > 0.f ? 1.f / L : 0.f;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < G * D; idx += blockDim.x) {
    const int r = idx / D, d = idx % D;
    float O = 0.f;
#pragma unroll 8
    for (int sp = 0; sp < S; ++sp) O += __ldcg(wo + (sp * G + r) * D + d) * wgt[sp * G + r];
    p.out[static_cast<size_t>(row) * p.hq * D + static_cast<size_t>(kvh * G + r) * D + d] =
        __float2bfloat16(O * inv_l[r]);
  }
  if (threadIdx.x == 0) *cnt = 0;
}

// ---------------------------------------------------------- K1 stream-K ----
// The decode work is (entry, KV head) pairs x their pages. A fixed grid of
// `gridDim.x` CTAs (all resident: the occupancy limit x SMs) splits the
// flattened page sequence of ALL pairs into equal contiguous ranges of W
// pages, so every CTA streams the same number of K/V bytes whatever the mix
// of context lengths -- no wave tail, no idle SMs on a 39-sequence step. A
// CTA walks the pair segments of its range; a pair covered by one CTA is
// written directly, a pair cut by range boundaries leaves one fp32 partial
// (m, l, O) per covering CTA (slot 0 = the CTA's first segment, slot 1 = its
// last) and the last covering CTA to finish folds them (per-pair arrival
// counter, self-resetting). W and the pair layout come from the device
// descriptor (n_dec_cur) and the page prefix sums, so a captured graph serves
// every plan of its bucket and a safepoint drop re-balances the next layer.
template <int D, int G, int NS>
__global__ void __launch_bounds__(128, 3) attn_decode_sk_kernel(AttnParams p) {
  pdl_trigger();
  constexpr int KS = D / 16;
  constexpr int NTD = D / 8;
  constexpr int PB = kPage * D * 2;  // bytes per K (or V) page
  constexpr int kMinPages = 16;      // >= 4 pages per warp
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ int s_last;
  const int n_dec = p.desc->n_dec_cur;
  if (n_dec <= 0) return;
  const int hkv = p.hkv;
  const int total = hkv * p.dec_pfx[n_dec];
  const int W = max(kMinPages, (total + static_cast<int>(gridDim.x) - 1) / static_cast<int>(gridDim.x));
  const int c = blockIdx.x;
  const int g_begin = c * W;
  const int g_end = min(total, g_begin + W);
  if (g_begin >= g_end) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  constexpr int kPart = G * (D + 2);  // floats per partial: m[G], l[G], O[G][D]

  // first decode entry of the range: largest i with hkv * pfx[i] <= g_begin
  int i;
  {
    int lo = 0, hi = n_dec - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (hkv * p.dec_pfx[mid] <= g_begin) lo = mid; else hi = mid - 1;
    }
    i = lo;
  }
  int g = g_begin;
  while (g < g_end) {
    while (hkv * p.dec_pfx[i + 1] <= g) ++i;
    const int n_i = p.dec_pfx[i + 1] - p.dec_pfx[i];
    const int base_i = hkv * p.dec_pfx[i];
    const int kvh = (g - base_i) / n_i;
    const int P = base_i + kvh * n_i;  // this pair's first global page
    const int seg_end = min(g_end, P + n_i);
    const int pg0 = g - P, pg1 = seg_end - P;
    const bool first_seg = g == g_begin;
    g = seg_end;

    const int ent = p.dec_ent[i];
    const int row = p.ent_q0[ent];
    const int kv_len = p.ent_kvlen[ent];
    const int32_t* bt = p.block_table + p.ent_bt[ent];

    uint32_t qa[KS][4];
    {
      const __nv_bfloat16* q = p.qkv + static_cast<size_t>(row) * p.qkv_stride + static_cast<size_t>(kvh) * G * D;
      const int r0 = gid, r1 = gid + 8;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const int d0 = ks * 16 + tig * 2;
        qa[ks][0] = r0 < G ? *reinterpret_cast<const uint32_t*>(q + r0 * D + d0) : 0u;
        qa[ks][1] = r1 < G ? *reinterpret_cast<const uint32_t*>(q + r1 * D + d0) : 0u;
        qa[ks][2] = r0 < G ? *reinterpret_cast<const uint32_t*>(q + r0 * D + d0 + 8) : 0u;
        qa[ks][3] = r1 < G ? *reinterpret_cast<const uint32_t*>(q + r1 * D + d0 + 8) : 0u;
      }
    }
    if (p.k1_rope) {
      rope_q_frags<D>(qa, tig, p.rope_tab + static_cast<size_t>(row) * (D / 2));
      if (pg1 == n_i) {  // this segment reads the pair's last page: the new token's K/V first
        append_new_kv<D>(p, row, kvh);
        __syncthreads();
      }
    }
    float o[NTD][4];
#pragma unroll
    for (int k = 0; k < NTD; ++k) o[k][0] = o[k][1] = o[k][2] = o[k][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

    // per-warp ring of NS pages (K and V): NS - 1 pages in flight while one
    // is consumed
    uint8_t* wbuf = smem + warp * NS * 2 * PB;  // [stage][K|V]
    int pg = pg0 + warp;
#pragma unroll
    for (int s0 = 0; s0 < NS - 1; ++s0) {
      const int pp = pg + 4 * s0;
      if (pp < pg1) {
        uint8_t* nb = wbuf + s0 * 2 * PB;
        load_page_async<D>(nb, nb + PB, kv_page(p, bt[pp], kvh, 0, D), kv_page(p, bt[pp], kvh, 1, D), lane);
      }
      cp_async_commit();
    }
    int stage = 0;
    for (; pg < pg1; pg += 4) {
      const int nxt = pg + 4 * (NS - 1);
      if (nxt < pg1) {
        uint8_t* nb = wbuf + ((stage + NS - 1) % NS) * 2 * PB;
        load_page_async<D>(nb, nb + PB, kv_page(p, bt[nxt], kvh, 0, D), kv_page(p, bt[nxt], kvh, 1, D), lane);
      }
      cp_async_commit();
      cp_async_wait<NS - 1>();
      __syncwarp();
      const uint8_t* sK = wbuf + stage * 2 * PB;
      const uint8_t* sV = sK + PB;
      float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const int mi = lane >> 3;
        const int tok = (mi >> 1) * 8 + (lane & 7);
        uint32_t b0, b1, b2, b3;
        ldmatrix_x4(b0, b1, b2, b3, sK + swz<D>(tok, ks * 2 + (mi & 1)));
        mma_bf16_16816(sc[0], qa[ks], b0, b1);
        mma_bf16_16816(sc[1], qa[ks], b2, b3);
      }
      const int base = pg * kPage;
      float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const bool ok = base + nt * 8 + tig * 2 + j < kv_len;
          sc[nt][j] = ok ? sc[nt][j] * p.scale_log2 : -INFINITY;
          sc[nt][2 + j] = ok ? sc[nt][2 + j] * p.scale_log2 : -INFINITY;
          mx0 = fmaxf(mx0, sc[nt][j]);
          mx1 = fmaxf(mx1, sc[nt][2 + j]);
        }
      }
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
      const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
      const float al0 = exp2f(m0 - mn0), al1 = exp2f(m1 - mn1);
      m0 = mn0;
      m1 = mn1;
      uint32_t pa[4];
      float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const float p0 = exp2f(sc[nt][0] - mn0), p1 = exp2f(sc[nt][1] - mn0);
        const float p2 = exp2f(sc[nt][2] - mn1), p3 = exp2f(sc[nt][3] - mn1);
        rs0 += p0 + p1;
        rs1 += p2 + p3;
        pa[nt * 2 + 0] = pack_bf16(p0, p1);
        pa[nt * 2 + 1] = pack_bf16(p2, p3);
      }
      l0 = l0 * al0 + rs0;
      l1 = l1 * al1 + rs1;
#pragma unroll
      for (int k = 0; k < NTD; ++k) {
        o[k][0] *= al0;
        o[k][1] *= al0;
        o[k][2] *= al1;
        o[k][3] *= al1;
      }
#pragma unroll
      for (int nd = 0; nd < D / 16; ++nd) {
        const int mi = lane >> 3;
        const int tok = (mi & 1) * 8 + (lane & 7);
        uint32_t v0, v1, v2, v3;
        ldmatrix_x4_trans(v0, v1, v2, v3, sV + swz<D>(tok, nd * 2 + (mi >> 1)));
        mma_bf16_16816(o[nd * 2], pa, v0, v1);
        mma_bf16_16816(o[nd * 2 + 1], pa, v2, v3);
      }
      __syncwarp();
      stage = (stage + 1) % NS;
    }
    cp_async_wait<0>();
    l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
    l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 2);

    // merge the 4 warps in smem (aliases the K/V ring: all warps are done)
    __syncthreads();
    float* sm_m = reinterpret_cast<float*>(smem);
    float* sm_l = sm_m + 4 * 16;
    float* sm_o = sm_l + 4 * 16;
    if (tig == 0) {
      sm_m[warp * 16 + gid] = m0;
      sm_m[warp * 16 + gid + 8] = m1;
      sm_l[warp * 16 + gid] = l0;
      sm_l[warp * 16 + gid + 8] = l1;
    }
#pragma unroll
    for (int nt = 0; nt < NTD; ++nt) {
      const int d = nt * 8 + tig * 2;
      sm_o[(warp * 16 + gid) * D + d] = o[nt][0];
      sm_o[(warp * 16 + gid) * D + d + 1] = o[nt][1];
      sm_o[(warp * 16 + gid + 8) * D + d] = o[nt][2];
      sm_o[(warp * 16 + gid + 8) * D + d + 1] = o[nt][3];
    }
    __syncthreads();
    const bool full = pg0 == 0 && pg1 == n_i;
    float* part = p.ws_sk + (static_cast<size_t>(c) * 2 + (first_seg ? 0 : 1)) * kPart;
    for (int idx = threadIdx.x; idx < G * D; idx += blockDim.x) {
      const int r = idx / D, d = idx % D;
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < 4; ++w) M = fmaxf(M, sm_m[w * 16 + r]);
      float L = 0.f, O = 0.f;
      if (M != -INFINITY) {
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const float f = exp2f(sm_m[w * 16 + r] - M);
          L += sm_l[w * 16 + r] * f;
          O += sm_o[(w * 16 + r) * D + d] * f;
        }
      }
      if (full) {
        p.out[static_cast<size_t>(row) * p.hq * D + static_cast<size_t>(kvh * G + r) * D + d] =
            __float2bfloat16(L > 0.f ? O / L : 0.f);
      } else {
        if (d == 0) {
          part[r] = M;
          part[G + r] = L;
        }
        part[2 * G + r * D + d] = O;
      }
    }
    if (!full) {
      // the last of the pair's covering CTAs folds their partials
      const int c_first = P / W, c_last = (P + n_i - 1) / W;
      __threadfence();
      __syncthreads();
      int32_t* cnt = p.dec_cnt + static_cast<size_t>(i) * hkv + kvh;
      if (threadIdx.x == 0) s_last = atomicAdd(cnt, 1) == c_last - c_first;
      __syncthreads();
      if (s_last) {
        __threadfence();
        const int nseg = c_last - c_first + 1;
        for (int idx = threadIdx.x; idx < G * D; idx += blockDim.x) {
          const int r = idx / D, d = idx % D;
          float M = -INFINITY;
          for (int k = 0; k < nseg; ++k) {
            const int cc = c_first + k;
            const float* pp = p.ws_sk + (static_cast<size_t>(cc) * 2 + (cc * W >= P ? 0 : 1)) * kPart;
            M = fmaxf(M, __ldcg(pp + r));
          }
          float L = 0.f, O = 0.f;
          if (M != -INFINITY) {
            for (int k = 0; k < nseg; ++k) {
              const int cc = c_first + k;
              const float* pp = p.ws_sk + (static_cast<size_t>(cc) * 2 + (cc * W >= P ? 0 : 1)) * kPart;
              const float ms = __ldcg(pp + r);
              const float f = ms == -INFINITY ? 0.f : exp2f(ms - M);
              L += __ldcg(pp + G + r) * f;
              O += __ldcg(pp + 2 * G + r * D + d) * f;
            }
          }
          p.out[static_cast<size_t>(row) * p.hq * D + static_cast<size_t>(kvh * G + r) * D + d] =
              __float2bfloat16(L > 0.f ? O / L : 0.f);
        }
        if (threadIdx.x == 0) *cnt = 0;
      }
    }
    __syncthreads();  // smem (merge scratch = K/V ring) is free for the next segment
  }
}

// ------------------------------------------------------------- launchers ----
int decode_sk_smem_bytes(int D, int ns) {
  const int ring = 4 * ns * 2 * kPage * D * 2, merge = (4 * 16 * 2 + 4 * 16 * D) * 4;
  return ring > merge ? ring : merge;
}
int decode_smem_bytes(int D) { return 4 * 4 * kPage * D * 2 > (4 * 16 * 2 + 4 * 16 * D) * 4 ? 4 * 4 * kPage * D * 2 : (4 * 16 * 2 + 4 * 16 * D) * 4; }

bool launch_prefill_tc(const AttnParams& p, const CUtensorMap* kv_map, int head_dim, int group, int n_pt_grid,
                       cudaStream_t s);
bool launch_prefill_tc2(const AttnParams& p, const CUtensorMap* kv_map, int head_dim, int group, int n_pt_grid,
                        cudaStream_t s);

template <int D, int G>
static void launch_attention_t(const AttnParams& p, const CUtensorMap* kv_map, int n_dec_grid, int n_pt_grid,
                               cudaStream_t s) {
  if (n_dec_grid > 0) {
    const int smem = decode_smem_bytes(D);
    if (p.sk_ctas > 0) {
      if (p.sk_stages == 3) {
        const int sm3 = decode_sk_smem_bytes(D, 3);
        smem_attr_once(reinterpret_cast<const void*>(attn_decode_sk_kernel<D, G, 3>), sm3);
        attn_decode_sk_kernel<D, G, 3><<<p.sk_ctas, 128, sm3, s>>>(p);
      } else {
        smem_attr_once(reinterpret_cast<const void*>(attn_decode_sk_kernel<D, G, 2>), smem);
        attn_decode_sk_kernel<D, G, 2><<<p.sk_ctas, 128, smem, s>>>(p);
      }
    } else {
      smem_attr_once(reinterpret_cast<const void*>(attn_decode_kernel<D, G>), smem);
      dim3 grid(p.n_splits, p.hkv, n_dec_grid);
      attn_decode_kernel<D, G><<<grid, 128, smem, s>>>(p);
    }
  }
  if (n_pt_grid > 0) {
    if (!(p.k2_pair && launch_prefill_tc2(p, kv_map, D, G, n_pt_grid, s))) launch_prefill_tc(p, kv_map, D, G, n_pt_grid, s);
  }
}

// Resident CTAs of the stream-K decode kernel per SM (its grid = this x SMs).
int decode_sk_ctas_per_sm(int head_dim, int group, int ns) {
  int n = 0;
  const int smem = decode_sk_smem_bytes(head_dim, ns);
#define CS_SK_OCC(DD, GG)                                                                                 \
  if (head_dim == DD && group == GG) {                                                                    \
    if (ns == 3) {                                                                                        \
      smem_attr_once(reinterpret_cast<const void*>(attn_decode_sk_kernel<DD, GG, 3>), smem);              \
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, attn_decode_sk_kernel<DD, GG, 3>, 128, smem);     \
    } else {                                                                                              \
      smem_attr_once(reinterpret_cast<const void*>(attn_decode_sk_kernel<DD, GG, 2>), smem);              \
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, attn_decode_sk_kernel<DD, GG, 2>, 128, smem);     \
    }                                                                                                     \
  }
  CS_SK_OCC(64, 1)
  CS_SK_OCC(64, 2)
  CS_SK_OCC(64, 4)
  CS_SK_OCC(128, 1)
  CS_SK_OCC(128, 2)
  CS_SK_OCC(128, 4)
  CS_SK_OCC(128, 5)
  CS_SK_OCC(128, 8)
#undef CS_SK_OCC
  return n;
}

// Dispatch on (head_dim, group size); returns false for an unsupported shape.
bool launch_attention(const AttnParams& p, const CUtensorMap* kv_map, int head_dim, int group, int n_dec_grid,
                      int n_pt_grid, cudaStream_t s) {
#define CS_ATTN_CASE(DD, GG)                                    \
  if (head_dim == DD && group == GG) {                          \
    launch_attention_t<DD, GG>(p, kv_map, n_dec_grid, n_pt_grid, s); \
    return true;                                                \
  }
  CS_ATTN_CASE(64, 1)
  CS_ATTN_CASE(64, 2)
  CS_ATTN_CASE(64, 4)
  CS_ATTN_CASE(128, 1)
  CS_ATTN_CASE(128, 2)
  CS_ATTN_CASE(128, 4)
  CS_ATTN_CASE(128, 5)
  CS_ATTN_CASE(128, 8)
#undef CS_ATTN_CASE
  return false;
}

}  // namespace csk
