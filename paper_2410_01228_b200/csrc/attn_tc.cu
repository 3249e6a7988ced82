// K2 on the 5th-generation tensor cores: prefill-chunk paged attention
// (reference stand-in: the k2*P(P+C) term of
// oracle_latency, proj/src/perf_model.cpp:56-65).
//
// One CTA = two 128-row query tiles (256 packed (token, head-in-group) rows of
// one entry) x one KV head. Keys stream in tiles of 128 (8 pages of 16
// tokens) through a 2-stage shared-memory ring fed by TMA straight from the
// block-table-indexed HBM pool (one 2D tensor map over the pool's [rows][D]
// view; a page of one (layer, K|V, head) is 16 contiguous rows), so every K/V
// byte loaded serves 256 query rows. Warp roles (320 threads):
//   warp 8      TMA producer (one lane): K and V pages of key tile j -> stage j%2
//   warp 9      MMA issuer (one lane), ping-pong over the two query tiles:
//               S_i = Q_i K_j^T (SS, M=128 N=128 K=D) into TMEM S_i, then
//               O_i += P_i V_j (TS: P_i read from TMEM, V_j from smem
//               MN-major; M=128 N=D K=128) into TMEM O_i
//   warps 0-3   softmax/epilogue of query tile 0, warps 4-7 of tile 1; one
//               thread per row == one TMEM lane: tcgen05.ld the S row, causal
//               mask on absolute positions (recompute positions may be
//               non-contiguous), online softmax with lazy rescale (O_i in TMEM
//               is corrected only when the row max grows by > 2^8), P_i as
//               packed bf16 written back over S_i's columns (tcgen05.st),
//               final O_i / l to HBM.
// While softmax i works on S_i(j), the tensor core runs the other tile's
// S/PV, so MUFU/ALU time overlaps the UMMA time.
// TMEM (512 cols): S_0 [0,128)  S_1 [128,256)  O_0 [256,256+D)  O_1 [384,384+D).
// mbarriers: k_full/v_full (TMA->MMA), kv_empty (MMA->TMA, tcgen05.commit),
// s_full_i / o_done_i (MMA->softmax i), p_full_i (softmax i -> MMA, 128 arrivals).
#include "common.cuh"
#include "tc.cuh"

namespace csk {

namespace {

constexpr int kRows = 128;   // UMMA M: rows per query tile
constexpr int kQT = 2;       // query tiles per CTA
constexpr int kKeys = 128;   // keys per tile
constexpr int kPage = 16;
constexpr int kThreads = 320;
constexpr int kChunkBytes = 128 * 128;  // one [128 rows][64 bf16] SWIZZLE_128B chunk = 16 KB

template <int D>
struct TcLayout {
  static constexpr int kChunks = D / 64;
  static constexpr int q = 0;                                        // [tile][chunk]
  static constexpr int k = q + kQT * kChunks * kChunkBytes;          // [stage][chunk]
  static constexpr int v = k + 2 * kChunks * kChunkBytes;
  static constexpr int bar = v + 2 * kChunks * kChunkBytes;
  static constexpr int bytes = bar + 128 + 1024;                     // barriers + 1 KB alignment slack
  // one CTA per SM (each allocates all 512 TMEM columns)
  static constexpr int launch_bytes = bytes < 120 * 1024 ? 120 * 1024 : bytes;
  static constexpr int tmem_s = 0;      // + i * 128
  static constexpr int tmem_o = 256;    // + i * 128
};

__device__ __forceinline__ int32_t pool_row(const AttnParams& p, int32_t block, int which, int kvh) {
  // row of the first token of (block, layer, K|V, head) in the pool's [rows][D]
  // view of [blocks][L][2][Hkv][16][D]
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
  const bool has2 = t.row0 + kRows < n_rows;  // second query tile present
  const int last_row = min(t.row0 + kQT * kRows, n_rows) - 1;
  const int kv_hi = min(kv_len, p.tok_pos[q0 + last_row / G] + 1);
  const int n_kt = (kv_hi + kKeys - 1) / kKeys;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  uint8_t* sQ = smem + Lay::q;
  uint8_t* sK = smem + Lay::k;
  uint8_t* sV = smem + Lay::v;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Lay::bar);
  uint64_t* k_full = bars + 0;     // [2 stages]
  uint64_t* v_full = bars + 2;     // [2]
  uint64_t* kv_empty = bars + 4;   // [2]
  uint64_t* s_full = bars + 6;     // [2 query tiles]
  uint64_t* p_full = bars + 8;     // [2]
  uint64_t* o_done = bars + 10;    // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&k_full[i], 1);
      tc::mbar_init(&v_full[i], 1);
      tc::mbar_init(&kv_empty[i], 1);
      tc::mbar_init(&s_full[i], 1);
      tc::mbar_init(&p_full[i], kRows);
      tc::mbar_init(&o_done[i], 1);
    }
    tc::fence_mbar_init();
  }
  if (warp == 8 && lane == 0) tc::prefetch_tmap(&kv_map);
  if (warp == 0) tc::tmem_alloc<512>(tmem_slot);

  // Q tiles: softmax thread (i, r) loads packed row row0 + 128 i + r (token
  // q0 + gr/G, head kvh*G + gr%G) into the SWIZZLE_128B K-major UMMA layout.
  if (warp < 8) {
    const int qi = warp >> 2, r = threadIdx.x & 127;
    const int gr = t.row0 + qi * kRows + r;
    const bool valid = gr < n_rows;
    const __nv_bfloat16* src = p.qkv + static_cast<size_t>(q0 + (valid ? gr : 0) / G) * p.qkv_stride +
                               static_cast<size_t>(kvh * G + (valid ? gr : 0) % G) * D;
    uint8_t* dq = sQ + qi * CH * kChunkBytes;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint4 val = valid ? *reinterpret_cast<const uint4*>(src + c * 64 + u * 8) : make_uint4(0, 0, 0, 0);
        *reinterpret_cast<uint4*>(dq + c * kChunkBytes + r * 128 + ((u ^ (r & 7)) << 4)) = val;
      }
    }
    tc::fence_async_smem();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 8) {
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
            // pages past the last one reload a valid page: their keys are
            // masked to p = 0, and finite V keeps 0 * V == 0
            const int pg = min(j * (kKeys / kPage) + pi, n_pages - 1);
            const int32_t row = pool_row(p, bt[pg], which, kvh);
#pragma unroll
            for (int c = 0; c < CH; ++c)
              tc::tma_load_2d(dst + c * kChunkBytes + pi * kPage * 128, &kv_map, bar, c * 64, row);
          }
        }
      }
    }
  } else if (warp == 9) {
    // -------------------------------------------------------- MMA issuer --
    if (lane == 0) {
      constexpr uint32_t idesc_s = tc::idesc_bf16_f32(kRows, kKeys, false, false);
      constexpr uint32_t idesc_o = tc::idesc_bf16_f32(kRows, D, false, true);
      const uint32_t q_addr = tc::smem_u32(sQ), k_addr = tc::smem_u32(sK), v_addr = tc::smem_u32(sV);
      const int nq = has2 ? 2 : 1;
      auto issue_s = [&](int qi, int j) {
        const uint32_t kb = k_addr + (j & 1) * CH * kChunkBytes;
        const uint32_t qb = q_addr + qi * CH * kChunkBytes;
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const uint32_t off = (ks >> 2) * kChunkBytes + (ks & 3) * 32;
          tc::umma_bf16_ss(tmem + Lay::tmem_s + qi * 128, tc::sdesc_sw128(qb + off, 16, 1024),
                           tc::sdesc_sw128(kb + off, 16, 1024), idesc_s, ks > 0 ? 1u : 0u);
        }
        tc::umma_commit(&s_full[qi]);
      };
      auto issue_pv = [&](int qi, int j) {
        const uint32_t vb = v_addr + (j & 1) * CH * kChunkBytes;
#pragma unroll
        for (int ks = 0; ks < kKeys / 16; ++ks) {
          // A = P_i in TMEM (16 keys = 8 packed columns); B = V read
          // MN-major: 16 keys = two 8-key atoms (SBO), 64-dim chunks LBO apart
          tc::umma_bf16_ts(tmem + Lay::tmem_o + qi * 128, tmem + Lay::tmem_s + qi * 128 + ks * 8,
                           tc::sdesc_sw128(vb + ks * 16 * 128, kChunkBytes, 1024), idesc_o,
                           (j > 0 || ks > 0) ? 1u : 0u);
        }
        tc::umma_commit(&o_done[qi]);
      };
      tc::mbar_wait(&k_full[0], 0);
      tc::tc_fence_after();
      for (int qi = 0; qi < nq; ++qi) issue_s(qi, 0);
      for (int j = 0; j < n_kt; ++j) {
        const int st = j & 1;
        tc::mbar_wait(&v_full[st], (j >> 1) & 1);
        const bool next = j + 1 < n_kt;
        for (int qi = 0; qi < nq; ++qi) {
          tc::mbar_wait(&p_full[qi], j & 1);
          tc::tc_fence_after();
          issue_pv(qi, j);
          if (qi == nq - 1) tc::umma_commit(&kv_empty[st]);  // K_j, V_j fully consumed
          if (next) {
            // S_i(j+1) overwrites the P_i(j) columns PV_i(j) reads: UMMAs from
            // one thread execute in issue order
            if (qi == 0) {
              tc::mbar_wait(&k_full[(j + 1) & 1], ((j + 1) >> 1) & 1);
              tc::tc_fence_after();
            }
            issue_s(qi, j + 1);
          }
        }
      }
    }
  } else {
    // ------------------------------------------- softmax + epilogue (rows) --
    const int qi = warp >> 2, r = threadIdx.x & 127;
    if (qi == 0 || has2) {
      const int gr = t.row0 + qi * kRows + r;
      const bool valid = gr < n_rows;
      // invalid rows run the same math on the last row's position (discarded)
      const int pos = p.tok_pos[q0 + (valid ? gr : last_row) / G];
      const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
      const uint32_t ts = tmem + lane_base + Lay::tmem_s + qi * 128;
      const uint32_t to = tmem + lane_base + Lay::tmem_o + qi * 128;
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j < n_kt; ++j) {
        tc::mbar_wait(&s_full[qi], j & 1);
        tc::tc_fence_after();
        float s[kKeys];
#pragma unroll
        for (int c = 0; c < kKeys / 32; ++c) tc::tmem_ld32(ts + c * 32, s + c * 32);
        tc::tmem_wait_ld();
        tc::reg_fence<kKeys>(s);
        const int kbase = j * kKeys;
        float mx = -INFINITY;
        if (kbase + kKeys - 1 <= pos) {  // whole tile visible (all but the diagonal tiles)
#pragma unroll
          for (int i = 0; i < kKeys; ++i) {
            s[i] *= p.scale_log2;
            mx = fmaxf(mx, s[i]);
          }
        } else {
#pragma unroll
          for (int i = 0; i < kKeys; ++i) {
            s[i] = (kbase + i <= pos) ? s[i] * p.scale_log2 : -INFINITY;
            mx = fmaxf(mx, s[i]);
          }
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
          rs += p0 + p1;
          pk[i / 2] = pack_bf16(p0, p1);
        }
        l = l * alpha + rs;
        // tcgen05.ld/st are warp-collective (.sync.aligned): the correction
        // runs for the whole warp if any of its rows needs it (alpha = 1 for
        // the others)
        if (__any_sync(0xffffffffu, rescale) && j > 0) {
          tc::mbar_wait(&o_done[qi], (j - 1) & 1);  // PV_i(j-1) landed in O_i
          tc::tc_fence_after();
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            float o[32];
            tc::tmem_ld32(to + c * 32, o);
            tc::tmem_wait_ld();
            tc::reg_fence<32>(o);
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] *= alpha;
            tc::tmem_st32(to + c * 32, o);
          }
        }
        // P_i(j) over S_i's first 64 columns (S_i(j) is in registers already;
        // PV_i(j-1), the last reader of P_i(j-1), ran before S_i(j))
        tc::tmem_st32u(ts, pk);
        tc::tmem_st32u(ts + 32, pk + 32);
        tc::tmem_wait_st();
        tc::tc_fence_before();
        tc::mbar_arrive(&p_full[qi]);
      }
      // epilogue: O_i / l -> HBM
      tc::mbar_wait(&o_done[qi], (n_kt - 1) & 1);
      tc::tc_fence_after();
      const float inv = l > 0.f ? 1.f / l : 0.f;
      __nv_bfloat16* dst = p.out + static_cast<size_t>(q0 + (valid ? gr : 0) / G) * p.hq * D +
                           static_cast<size_t>(kvh * G + (valid ? gr : 0) % G) * D;
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        float o[32];
        tc::tmem_ld32(to + c * 32, o);
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

// Rows per K2 work tile (engine.cu builds the tile list with this step).
int prefill_tile_rows() { return kQT * kRows; }

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
