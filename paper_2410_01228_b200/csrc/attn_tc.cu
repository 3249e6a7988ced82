// K2 on the 5th-generation tensor cores: prefill-chunk paged attention
// (reference stand-in: the k2*P(P+C) term of
// oracle_latency, proj/src/perf_model.cpp:56-65).
//
// One CTA = 128 packed query rows (token, head-in-group) of one entry x one KV
// head; keys stream in tiles of 128 (8 pages of 16 tokens) through a 2-stage
// shared-memory ring fed by TMA straight from the block-table-indexed HBM
// pool (one 2D tensor map over the pool's [rows][D] view; a page of one
// (layer, K|V, head) is 16 contiguous rows). Warp roles:
//   warp 4      TMA producer (one lane): K and V pages of tile j -> stage j%2
//   warp 5      MMA issuer (one lane):   S_j = Q K_j^T   (tcgen05.mma, SS,
//               M=128 N=128 K=D) into a double-buffered TMEM S, then
//               O += P_j V_j (M=128 N=D K=128, V read MN-major) into TMEM O
//   warps 0-3   softmax/epilogue, one thread per row == one TMEM lane:
//               tcgen05.ld S row, causal mask on absolute positions
//               (recompute positions may be non-contiguous), online softmax
//               with lazy rescale (O in TMEM is corrected only when the row
//               max grows by > 2^8), P as bf16 into swizzled smem, final
//               O / l from TMEM to HBM.
// Synchronisation: mbarriers for TMA->MMA (k_full/v_full), MMA->TMA
// (kv_empty, via tcgen05.commit), MMA->softmax (s_full, o_done) and
// softmax->MMA (p_full, 128 arrivals).
#include "common.cuh"
#include "tc.cuh"

namespace csk {

namespace {

constexpr int kRows = 128;   // UMMA M: packed query rows per CTA
constexpr int kKeys = 128;   // keys per tile
constexpr int kPage = 16;
constexpr int kThreads = 192;
constexpr int kChunkBytes = kRows * 128;  // one [128 rows][64 bf16] SWIZZLE_128B chunk = 16 KB

template <int D>
struct TcLayout {
  static constexpr int kChunks = D / 64;
  static constexpr int q = 0;
  static constexpr int k = q + kChunks * kChunkBytes;              // 2 stages
  static constexpr int v = k + 2 * kChunks * kChunkBytes;          // 2 stages
  static constexpr int pm = v + 2 * kChunks * kChunkBytes;         // P: 2 chunks (128 keys)
  static constexpr int bar = pm + 2 * kChunkBytes;
  static constexpr int bytes = bar + 128 + 1024;                   // barriers + 1 KB alignment slack
  // D=64 fits two CTAs per SM by size; force one (each allocates 512 TMEM cols)
  static constexpr int launch_bytes = bytes < 120 * 1024 ? 120 * 1024 : bytes;
  static constexpr int tmem_s = 0;      // S double buffer: cols [0,128) and [128,256)
  static constexpr int tmem_o = 256;    // O: cols [256, 256 + D)
};

__device__ __forceinline__ int32_t pool_row(const AttnParams& p, int32_t block, int which, int kvh) {
  // row index of the first token of (block, layer, K|V, head) in the pool's
  // [rows][D] view: [blocks][L][2][Hkv][16][D]
  const int64_t r = ((static_cast<int64_t>(block) * p.num_layers + p.layer) * 2 + which) * p.hkv + kvh;
  return static_cast<int32_t>(r * kPage);
}

}  // namespace

template <int D, int G>
__global__ void __launch_bounds__(kThreads, 1)
    attn_prefill_tc_kernel(AttnParams p, const __grid_constant__ CUtensorMap kv_map) {
  using Lay = TcLayout<D>;
  constexpr int CH = Lay::kChunks;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int n_pt = p.desc->n_pt_cur;
  if (static_cast<int>(blockIdx.x) >= n_pt) return;
  const int tile_idx = n_pt - 1 - static_cast<int>(blockIdx.x);  // latest (heaviest) tiles first
  const int kvh = blockIdx.y;
  const PrefillTile t = p.tiles[tile_idx];
  const int ent = t.entry;
  const int q0 = p.ent_q0[ent];
  const int n_rows = p.ent_qlen[ent] * G;
  const int kv_len = p.ent_kvlen[ent];
  const int32_t* bt = p.block_table + p.ent_bt[ent];
  const int n_pages = (kv_len + kPage - 1) / kPage;
  const int last_row = min(t.row0 + kRows, n_rows) - 1;
  const int kv_hi = min(kv_len, p.tok_pos[q0 + last_row / G] + 1);
  const int n_kt = (kv_hi + kKeys - 1) / kKeys;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  uint8_t* sQ = smem + Lay::q;
  uint8_t* sK = smem + Lay::k;
  uint8_t* sV = smem + Lay::v;
  uint8_t* sP = smem + Lay::pm;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Lay::bar);
  uint64_t* k_full = bars + 0;     // [2]
  uint64_t* v_full = bars + 2;     // [2]
  uint64_t* kv_empty = bars + 4;   // [2]
  uint64_t* s_full = bars + 6;     // [2]
  uint64_t* p_full = bars + 8;
  uint64_t* o_done = bars + 9;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 10);

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&k_full[i], 1);
      tc::mbar_init(&v_full[i], 1);
      tc::mbar_init(&kv_empty[i], 1);
      tc::mbar_init(&s_full[i], 1);
    }
    tc::mbar_init(p_full, kRows);
    tc::mbar_init(o_done, 1);
    tc::fence_mbar_init();
  }
  if (warp == 4 && lane == 0) tc::prefetch_tmap(&kv_map);
  if (warp == 0) tc::tmem_alloc<512>(tmem_slot);

  // Q tile: softmax thread r loads packed row r (token q0 + gr/G, head
  // kvh*G + gr%G) into the SWIZZLE_128B K-major layout the UMMA reads.
  if (warp < 4) {
    const int r = threadIdx.x;
    const int gr = t.row0 + r;
    const bool valid = gr < n_rows;
    const __nv_bfloat16* src =
        p.qkv + static_cast<size_t>(q0 + (valid ? gr : 0) / G) * p.qkv_stride + static_cast<size_t>(kvh * G + (valid ? gr : 0) % G) * D;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint4 val = valid ? *reinterpret_cast<const uint4*>(src + c * 64 + u * 8) : make_uint4(0, 0, 0, 0);
        *reinterpret_cast<uint4*>(sQ + c * kChunkBytes + r * 128 + ((u ^ (r & 7)) << 4)) = val;
      }
    }
    tc::fence_async_smem();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 4) {
    // ------------------------------------------------------ TMA producer --
    if (lane == 0) {
      constexpr uint32_t kTileBytes = CH * kChunkBytes;  // 128 keys x D bf16
      for (int j = 0; j < n_kt; ++j) {
        const int st = j & 1;
        if (j >= 2) tc::mbar_wait(&kv_empty[st], ((j >> 1) - 1) & 1);
        for (int which = 0; which < 2; ++which) {
          uint64_t* bar = which == 0 ? &k_full[st] : &v_full[st];
          uint8_t* dst = (which == 0 ? sK : sV) + st * CH * kChunkBytes;
          tc::mbar_expect_tx(bar, kTileBytes);
#pragma unroll 1
          for (int pi = 0; pi < kKeys / kPage; ++pi) {
            // pages past the tile's last one load a valid page: their keys are
            // masked to p = 0, and finite V keeps 0 * V == 0
            const int pg = min(j * (kKeys / kPage) + pi, n_pages - 1);
            const int32_t row = pool_row(p, bt[pg], which, kvh);
#pragma unroll
            for (int c = 0; c < CH; ++c) tc::tma_load_2d(dst + c * kChunkBytes + pi * kPage * 128, &kv_map, bar, c * 64, row);
          }
        }
      }
    }
  } else if (warp == 5) {
    // -------------------------------------------------------- MMA issuer --
    if (lane == 0) {
      constexpr uint32_t idesc_s = tc::idesc_bf16_f32(kRows, kKeys, false, false);
      constexpr uint32_t idesc_o = tc::idesc_bf16_f32(kRows, D, false, true);
      const uint32_t q_addr = tc::smem_u32(sQ), k_addr = tc::smem_u32(sK), v_addr = tc::smem_u32(sV),
                     p_addr = tc::smem_u32(sP);
      auto issue_s = [&](int j) {
        const int st = j & 1;
        tc::mbar_wait(&k_full[st], (j >> 1) & 1);
        tc::tc_fence_after();
        const uint32_t kb = k_addr + st * CH * kChunkBytes;
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const uint32_t off = (ks >> 2) * kChunkBytes + (ks & 3) * 32;
          tc::umma_bf16_ss(tmem + Lay::tmem_s + st * kKeys, tc::sdesc_sw128(q_addr + off, 16, 1024),
                           tc::sdesc_sw128(kb + off, 16, 1024), idesc_s, ks > 0 ? 1u : 0u);
        }
        tc::umma_commit(&s_full[st]);
      };
      issue_s(0);
      for (int j = 0; j < n_kt; ++j) {
        const int st = j & 1;
        if (j + 1 < n_kt) issue_s(j + 1);
        tc::mbar_wait(p_full, j & 1);
        tc::mbar_wait(&v_full[st], (j >> 1) & 1);
        tc::tc_fence_after();
        const uint32_t vb = v_addr + st * CH * kChunkBytes;
#pragma unroll
        for (int ks = 0; ks < kKeys / 16; ++ks) {
          // A = P (K-major, 2 chunks of 64 keys); B = V tile read MN-major:
          // 16 keys = two 8-key atoms (SBO 1024 B), 64-dim chunks LBO apart
          const uint32_t a_off = (ks >> 2) * kChunkBytes + (ks & 3) * 32;
          tc::umma_bf16_ss(tmem + Lay::tmem_o, tc::sdesc_sw128(p_addr + a_off, 16, 1024),
                           tc::sdesc_sw128(vb + ks * 16 * 128, kChunkBytes, 1024), idesc_o,
                           (j > 0 || ks > 0) ? 1u : 0u);
        }
        tc::umma_commit(o_done);
        tc::umma_commit(&kv_empty[st]);
      }
    }
  } else {
    // ------------------------------------------- softmax + epilogue (rows) --
    const int r = threadIdx.x;
    const int gr = t.row0 + r;
    const bool valid = gr < n_rows;
    // invalid rows run the same math on the last row's position (discarded)
    const int pos = p.tok_pos[q0 + (valid ? gr : last_row) / G];
    const uint32_t lane_base = static_cast<uint32_t>(warp * 32) << 16;
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < n_kt; ++j) {
      const int st = j & 1;
      tc::mbar_wait(&s_full[st], (j >> 1) & 1);
      tc::tc_fence_after();
      float s[kKeys];
#pragma unroll
      for (int c = 0; c < kKeys / 32; ++c) tc::tmem_ld32(tmem + lane_base + Lay::tmem_s + st * kKeys + c * 32, s + c * 32);
      tc::tmem_wait_ld();
      tc::reg_fence<kKeys>(s);
      const int kbase = j * kKeys;
      float mx = -INFINITY;
#pragma unroll
      for (int i = 0; i < kKeys; ++i) {
        s[i] = (kbase + i <= pos) ? s[i] * p.scale_log2 : -INFINITY;
        mx = fmaxf(mx, s[i]);
      }
      const float m_new = fmaxf(m_used, mx);
      const bool rescale = m_new > m_used + 8.f;  // true on the first tile (m_used = -inf)
      const float alpha = rescale ? exp2f(m_used - m_new) : 1.f;
      if (rescale) m_used = m_new;
      uint32_t pk[kKeys / 2];
      float rs = 0.f;
#pragma unroll
      for (int i = 0; i < kKeys; i += 2) {
        const float p0 = exp2f(s[i] - m_used), p1 = exp2f(s[i + 1] - m_used);
        pk[i / 2] = pack_bf16(p0, p1);
        const float2 rp = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pk[i / 2]));
        rs += rp.x + rp.y;  // sum what the MMA multiplies (bf16-rounded P)
      }
      l = l * alpha + rs;
      if (j > 0) {
        tc::mbar_wait(o_done, (j - 1) & 1);  // PV_{j-1} done: P buffer and O are ours
        tc::tc_fence_after();
        if (rescale) {
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            float o[32];
            tc::tmem_ld32(tmem + lane_base + Lay::tmem_o + c * 32, o);
            tc::tmem_wait_ld();
            tc::reg_fence<32>(o);
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] *= alpha;
            tc::tmem_st32(tmem + lane_base + Lay::tmem_o + c * 32, o);
          }
          tc::tmem_wait_st();
        }
      }
      // P row -> smem, K-major SWIZZLE_128B: 2 chunks of 64 keys, 8 x 16 B each
#pragma unroll
      for (int c = 0; c < 2; ++c) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int b = c * 32 + u * 4;
          *reinterpret_cast<uint4*>(sP + c * kChunkBytes + r * 128 + ((u ^ (r & 7)) << 4)) =
              make_uint4(pk[b], pk[b + 1], pk[b + 2], pk[b + 3]);
        }
      }
      tc::fence_async_smem();
      tc::tc_fence_before();
      tc::mbar_arrive(p_full);
    }
    // epilogue: O / l -> HBM
    tc::mbar_wait(o_done, (n_kt - 1) & 1);
    tc::tc_fence_after();
    const float inv = l > 0.f ? 1.f / l : 0.f;
    __nv_bfloat16* dst = p.out + static_cast<size_t>(q0 + (valid ? gr : 0) / G) * p.hq * D +
                         static_cast<size_t>(kvh * G + (valid ? gr : 0) % G) * D;
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      float o[32];
      tc::tmem_ld32(tmem + lane_base + Lay::tmem_o + c * 32, o);
      tc::tmem_wait_ld();
      tc::reg_fence<32>(o);
      if (valid) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          *reinterpret_cast<uint4*>(dst + c * 32 + i) =
              make_uint4(pack_bf16(o[i] * inv, o[i + 1] * inv), pack_bf16(o[i + 2] * inv, o[i + 3] * inv),
                         pack_bf16(o[i + 4] * inv, o[i + 5] * inv), pack_bf16(o[i + 6] * inv, o[i + 7] * inv));
        }
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

template <int D, int G>
void launch_prefill_tc_t(const AttnParams& p, const CUtensorMap* kv_map, int n_pt_grid, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_prefill_tc_kernel<D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         TcLayout<D>::launch_bytes);
    attr = true;
  }
  attn_prefill_tc_kernel<D, G><<<dim3(n_pt_grid, p.hkv), kThreads, TcLayout<D>::launch_bytes, s>>>(p, *kv_map);
}

bool launch_prefill_tc(const AttnParams& p, const CUtensorMap* kv_map, int head_dim, int group, int n_pt_grid,
                       cudaStream_t s) {
#define CS_TC_CASE(DD, GG)                                   \
  if (head_dim == DD && group == GG) {                       \
    launch_prefill_tc_t<DD, GG>(p, kv_map, n_pt_grid, s);    \
    return true;                                             \
  }
  CS_TC_CASE(64, 1)
  CS_TC_CASE(64, 2)
  CS_TC_CASE(64, 4)
  CS_TC_CASE(128, 1)
  CS_TC_CASE(128, 2)
  CS_TC_CASE(128, 4)
  CS_TC_CASE(128, 5)
  CS_TC_CASE(128, 8)
#undef CS_TC_CASE
  return false;
}

}  // namespace csk
