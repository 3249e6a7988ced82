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
//   warp 8      TMA producer (elected lane): K and V pages of key tile j -> stage j%2
//   warp 9      MMA issuer (elected lane), ping-pong over the two query tiles:
//               S_i(j) = Q_i K_j^T (SS, M=128 N=128 K=D: full rate, smem at
//               128 B/clk) into TMEM S_i, and O_i += P_i(j) V_j (TS: P_i read
//               from TMEM, V_j from smem MN-major; M=128 N=D K=128) into TMEM O_i
//   warps 0-3   softmax/epilogue of query tile 0, warps 4-7 of tile 1; one
//               thread per row == one TMEM lane: tcgen05.ld the S row, causal
//               mask on absolute positions (recompute positions may be
//               non-contiguous), online softmax with lazy rescale (O_i in TMEM
//               is corrected only when the row max grows by > 2^8), P_i as
//               packed bf16 written back over S_i's columns (tcgen05.st),
//               final O_i / l to HBM.
// While softmax i makes P_i(j), the tensor core runs the other tile's PV and
// S, so MUFU/ALU time overlaps the UMMA time (tools/umma_bench.cu: SS N=64
// runs at 2/3 rate, smem-bound; SS N>=128 and TS at the full 4096 MAC/clk).
// TMEM (512 cols): S_0 [0,128)  S_1 [128,256)  O_0 [256,256+D)  O_1 [384,384+D).
// mbarriers (each waited at most one phase behind): k_full/v_full/kv_empty
// per stage, s_full/p_full/o_done per query tile, o_final after the last PV.
#include "common.cuh"
#include "tc.cuh"

#ifdef CS_K2_TIMERS  // experiment builds only: per-role cycle accounting printed by one CTA
#include <cstdio>
// bounded wait: reports (tag, j, parity, CTA) and traps instead of hanging
#define K2_WAIT(bar, par, tag, jj)                                                                          \
  do {                                                                                                      \
    uint32_t ok_ = 0;                                                                                       \
    for (long it_ = 0; it_ < 20000000 && !ok_; ++it_) {                                                     \
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"        \
                   "selp.b32 %0, 1, 0, p;\n\t}"                                                          \
                   : "=r"(ok_) : "r"(tc::smem_u32(bar)), "r"(par) : "memory");                              \
    }                                                                                                       \
    if (!ok_) {                                                                                             \
      printf("K2 HANG %s j=%d par=%d n_kt=%d cta=(%d,%d,%d) tid=%d\n", tag, (int)(jj), (int)(par), n_kt,  \
             blockIdx.x, blockIdx.y, blockIdx.z, threadIdx.x);                                             \
      asm volatile("trap;");                                                                                \
    }                                                                                                       \
  } while (0)
#define K2T_DECL(x) long long x = 0
#define K2T_NOW() clock64()
#define K2T_ADD(x, t0) x += clock64() - (t0)
#else
#define K2_WAIT(bar, par, tag, jj) tc::mbar_wait(bar, par)
#define K2T_DECL(x)
#define K2T_NOW() 0LL
#define K2T_ADD(x, t0)
#endif

namespace csk {

namespace {

constexpr int kRows = 128;   // UMMA M: rows per query tile
constexpr int kQT = 2;       // query tiles per CTA
constexpr int kKeys = 128;   // keys per tile (UMMA N of S, K of PV)
constexpr int kStages = 2;   // K/V ring depth
constexpr int kPage = 16;
constexpr int kThreads = 320;
#ifndef CS_K2_POLY
#define CS_K2_POLY 2  // tools/k2_sweep.py: 2 of 8 beats 0, 3 and 4 (profiles/r1/k2_poly_sweep.md)
#endif
constexpr int kPoly8 = CS_K2_POLY;  // score pairs (of every 8) exponentiated by ex2_poly2
constexpr int kChunkBytes = 128 * 128;        // [128 rows][64 bf16] SWIZZLE_128B chunk (Q) = 16 KB
constexpr int kKvChunkBytes = kKeys * 128;    // [128 keys][64 bf16] chunk (K, V) = 16 KB

template <int D>
struct TcLayout {
  static constexpr int kChunks = D / 64;
  static constexpr int q = 0;                                        // [tile][chunk]
  static constexpr int k = q + kQT * kChunks * kChunkBytes;          // [stage][chunk]
  static constexpr int v = k + kStages * kChunks * kKvChunkBytes;
  static constexpr int bar = v + kStages * kChunks * kKvChunkBytes;
  static constexpr int bytes = bar + 256 + 1024;                     // barriers + 1 KB alignment slack
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
  const long long t_kernel = K2T_NOW();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // blockIdx.x = (rank of the tile in the heaviest-first order) x hkv + KV
  // head: the block scheduler hands out the longest tiles first
  const int n_pt = p.desc->n_pt_cur;
  const int tile_idx = p.tile_order[blockIdx.x / p.hkv];
  const int kvh = blockIdx.x % p.hkv;
  if (tile_idx >= n_pt) return;  // an offline tile dropped at a safepoint
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
  // split-K over key tiles (small grids over long contexts): this CTA runs
  // key tiles [jb, jb + n_kt) of [0, ceil(kv_hi / 64))
  const int split = blockIdx.z;
  const int jb = split * p.k2_tiles_per_split;
  const int n_kt = min((kv_hi + kKeys - 1) / kKeys - jb, p.k2_tiles_per_split);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (n_kt <= 0) {  // causal: no keys of this split reach these rows
    if (p.k2_splits > 1) {
      float* ws = p.ws2 + ((static_cast<size_t>(tile_idx) * p.hkv + kvh) * p.k2_splits + split) * (D + 2) * 256;
      for (int r = threadIdx.x; r < 256; r += blockDim.x) ws[D * 256 + r] = -INFINITY;
    }
    return;
  }
  uint8_t* sQ = smem + Lay::q;
  uint8_t* sK = smem + Lay::k;
  uint8_t* sV = smem + Lay::v;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Lay::bar);
  uint64_t* k_full = bars + 0;                   // [kStages]
  uint64_t* v_full = k_full + kStages;           // [kStages]
  uint64_t* kv_empty = v_full + kStages;         // [kStages]
  uint64_t* s_full = kv_empty + kStages;         // [query tile]
  uint64_t* p_full = s_full + 2;                 // [query tile]
  uint64_t* o_done = p_full + 2;                 // [query tile] once per PV
  uint64_t* o_final = o_done + 2;                // [query tile] after the last PV
  uint64_t* q_ready = o_final + 2;               // [query tile] Q tile staged in smem
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_ready + 2);

  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      tc::mbar_init(&k_full[i], 1);
      tc::mbar_init(&v_full[i], 1);
      tc::mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&s_full[i], 1);
      tc::mbar_init(&p_full[i], kRows);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&o_done[i], 1);
      tc::mbar_init(&o_final[i], 1);
      tc::mbar_init(&q_ready[i], kRows);
    }
    tc::fence_mbar_init();
  }
  if (warp == 8 && lane == 0) tc::prefetch_tmap(&kv_map);
  if (warp == 0) tc::tmem_alloc<512>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

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
    tc::mbar_arrive(&q_ready[qi]);  // the TMA warp is already streaming K/V meanwhile
  }

  if (warp == 8) {
    // ------------------------------------------------------ TMA producer --
    // warp-wide loop, one elected lane issues
    {
      constexpr uint32_t kTileBytes = CH * kKvChunkBytes;  // 128 keys x D bf16
      for (int j = 0; j < n_kt; ++j) {
        const int st = j % kStages;
        if (j >= kStages) K2_WAIT(&kv_empty[st], ((j / kStages) - 1) & 1, "kv_empty", j);
        // lane pi < 8 resolves page pi of the tile (pages past the last one
        // reload a valid page: masked to p = 0, finite V keeps 0 * V == 0)
        const int pg = min((jb + j) * (kKeys / kPage) + (lane & 7), n_pages - 1);
        const int32_t blk = bt[pg];
        int32_t pblk[kKeys / kPage];
#pragma unroll
        for (int pi = 0; pi < kKeys / kPage; ++pi) pblk[pi] = __shfl_sync(0xffffffffu, blk, pi);
        if (tc::elect_one_sync()) {
          for (int which = 0; which < 2; ++which) {
            uint64_t* bar = which == 0 ? &k_full[st] : &v_full[st];
            uint8_t* dst = (which == 0 ? sK : sV) + st * CH * kKvChunkBytes;
            tc::mbar_expect_tx(bar, kTileBytes);
#pragma unroll
            for (int pi = 0; pi < kKeys / kPage; ++pi) {
              const int32_t row = pool_row(p, pblk[pi], which, kvh);
#pragma unroll
              for (int c = 0; c < CH; ++c)
                tc::tma_load_2d(dst + c * kKvChunkBytes + pi * kPage * 128, &kv_map, bar, c * 64, row);
            }
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == 9) {
    // -------------------------------------------------------- MMA issuer --
    // warp-wide loop (descriptors in the uniform datapath), one elected lane
    // issues each group of UMMAs and its commit
    {
      constexpr uint32_t idesc_s = tc::idesc_bf16_f32(kRows, kKeys, false, false);
      constexpr uint32_t idesc_o = tc::idesc_bf16_f32(kRows, D, false, true);
      const uint32_t q_addr = tc::smem_u32(sQ), k_addr = tc::smem_u32(sK), v_addr = tc::smem_u32(sV);
      const int nq = has2 ? 2 : 1;
      // S_i(j) -> TMEM S_i; needs K_j landed
      auto issue_s = [&](int qi, int j) {
        const uint32_t kb = k_addr + (j % kStages) * CH * kKvChunkBytes;
        const uint32_t qb = q_addr + qi * CH * kChunkBytes;
        const uint32_t d_tmem = tmem + Lay::tmem_s + qi * 128;
        if (tc::elect_one_sync()) {
#pragma unroll
          for (int ks = 0; ks < D / 16; ++ks) {
            const uint32_t qoff = (ks >> 2) * kChunkBytes + (ks & 3) * 32;
            const uint32_t koff = (ks >> 2) * kKvChunkBytes + (ks & 3) * 32;
            tc::umma_bf16_ss(d_tmem, tc::sdesc_sw128(qb + qoff, 16, 1024), tc::sdesc_sw128(kb + koff, 16, 1024),
                             idesc_s, ks > 0 ? 1u : 0u);
          }
          tc::umma_commit(&s_full[qi]);
        }
        __syncwarp();
      };
      // O_i += P_i(j) V_j; P_i(j) is packed bf16 over S_i's first 64 columns
      auto issue_pv = [&](int qi, int j, bool release_stage) {
        const uint32_t vb = v_addr + (j % kStages) * CH * kKvChunkBytes;
        const uint32_t pa = tmem + Lay::tmem_s + qi * 128;
        const uint32_t d_tmem = tmem + Lay::tmem_o + qi * 128;
        if (tc::elect_one_sync()) {
#pragma unroll
          for (int ks = 0; ks < kKeys / 16; ++ks) {
            // B = V read MN-major: 16 keys = two 8-key atoms (SBO), 64-dim
            // chunks LBO apart
            tc::umma_bf16_ts(d_tmem, pa + ks * 8, tc::sdesc_sw128(vb + ks * 16 * 128, kKvChunkBytes, 1024), idesc_o,
                             (j > 0 || ks > 0) ? 1u : 0u);
          }
          tc::umma_commit(&o_done[qi]);
          if (j == n_kt - 1) tc::umma_commit(&o_final[qi]);
          if (release_stage) tc::umma_commit(&kv_empty[j % kStages]);  // K_j, V_j fully consumed
        }
        __syncwarp();
      };
      K2T_DECL(t_wk);
      K2T_DECL(t_wv);
      K2T_DECL(t_wp);
      const long long t_begin = K2T_NOW();
      auto wait_k = [&](int j) {
        const long long t0 = K2T_NOW();
        K2_WAIT(&k_full[j % kStages], (j / kStages) & 1, "k_full", j);
        K2T_ADD(t_wk, t0);
        tc::tc_fence_after();
      };
      // prologue: S(0) for both query tiles
      wait_k(0);
      for (int qi = 0; qi < nq; ++qi) {
        tc::mbar_wait(&q_ready[qi], 0);
        issue_s(qi, 0);
      }
      // ping-pong: while softmax i makes P_i(j), the tensor core runs the
      // other tile's PV / S
      for (int j = 0; j < n_kt; ++j) {
        const int st = j % kStages;
        long long t0 = K2T_NOW();
        K2_WAIT(&v_full[st], (j / kStages) & 1, "v_full", j);
        K2T_ADD(t_wv, t0);
        const bool next = j + 1 < n_kt;
        if (next) wait_k(j + 1);
        for (int qi = 0; qi < nq; ++qi) {
          t0 = K2T_NOW();
          K2_WAIT(&p_full[qi], j & 1, "p_full", j);
          K2T_ADD(t_wp, t0);
          tc::tc_fence_after();
          issue_pv(qi, j, qi == nq - 1);
          // S_i(j+1) overwrites the P_i(j) columns PV_i(j) reads: UMMAs from
          // one thread execute in issue order
          if (next) issue_s(qi, j + 1);
        }
      }
#ifdef CS_K2_TIMERS
      if (lane == 0 && kvh == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - p.hkv) && blockIdx.z == 0)
        printf("K2T mma  cta=%d n_kt=%d total=%lld wait_k=%lld wait_v=%lld wait_p=%lld\n", blockIdx.x, n_kt,
               clock64() - t_begin, t_wk, t_wv, t_wp);
#endif
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
      const uint32_t ts0 = tmem + lane_base + Lay::tmem_s + qi * 128;
      const uint32_t to = tmem + lane_base + Lay::tmem_o + qi * 128;
      const float scale = p.scale_log2;
      float m_used = -INFINITY, l = 0.f;  // m_used in scaled (log2) units
      K2T_DECL(t_ws);
      K2T_DECL(t_wo);
      const long long t_sbegin = K2T_NOW();
      for (int j = 0; j < n_kt; ++j) {
        const uint32_t ts = ts0;
        const long long t0 = K2T_NOW();
        K2_WAIT(&s_full[qi], j & 1, "s_full", j);
        K2T_ADD(t_ws, t0);
        tc::tc_fence_after();
        float s[kKeys];
#pragma unroll
        for (int c = 0; c < kKeys / 32; ++c) tc::tmem_ld32(ts + c * 32, s + c * 32);
        tc::tmem_wait_ld();
        tc::reg_fence<kKeys>(s);
        const int kbase = (jb + j) * kKeys;
        if (kbase + kKeys - 1 > pos) {  // diagonal tile: causal mask
#pragma unroll
          for (int i = 0; i < kKeys; ++i) s[i] = (kbase + i <= pos) ? s[i] : -INFINITY;
        }
        // raw (unscaled) max, 8 independent chains; scale > 0 commutes with max
        float mxa[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) mxa[a] = s[a];
#pragma unroll
        for (int i = 8; i < kKeys; ++i) mxa[i & 7] = fmaxf(mxa[i & 7], s[i]);
        const float mx = fmaxf(fmaxf(fmaxf(mxa[0], mxa[1]), fmaxf(mxa[2], mxa[3])),
                               fmaxf(fmaxf(mxa[4], mxa[5]), fmaxf(mxa[6], mxa[7])));
        const float m_new = fmaxf(m_used, mx * scale);
        const bool rescale = m_new > m_used + 8.f;  // true on the first tile (m_used = -inf)
        const float alpha = rescale ? tc::ex2_approx(m_used - m_new) : 1.f;
        if (rescale) m_used = m_new;
        // a split's rows may see no valid key yet (m_used = -inf): p = 0
        const float msub = m_used == -INFINITY ? 0.f : m_used;
        uint32_t pk[kKeys / 2];
        // packed fp32x2 FMA / add (FFMA2, FADD2): half the ALU issue slots
        const float2 sc2 = make_float2(scale, scale), ms2 = make_float2(-msub, -msub);
        float2 rsa[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
        for (int i = 0; i < kKeys; i += 2) {
          const float2 x = __ffma2_rn(make_float2(s[i], s[i + 1]), sc2, ms2);
          // kPoly8 of every 8 pairs on the FMA pipe: the MUFU (16 ex2/clk/SM)
          // is otherwise as busy as the tensor core
          const float2 pp = ((i >> 1) & 7) < kPoly8 ? tc::ex2_poly2(x)
                                                    : make_float2(tc::ex2_approx(x.x), tc::ex2_approx(x.y));
          rsa[(i >> 1) & 1] = __fadd2_rn(rsa[(i >> 1) & 1], pp);
          pk[i / 2] = pack_bf16(pp.x, pp.y);
        }
        const float rs = (rsa[0].x + rsa[1].x) + (rsa[0].y + rsa[1].y);
        l = l * alpha + rs;
        // tcgen05.ld/st are warp-collective (.sync.aligned): the correction
        // runs for the whole warp if any of its rows needs it (alpha = 1 for
        // the others)
        if (__any_sync(0xffffffffu, rescale) && j > 0) {
          const long long t1 = K2T_NOW();
          K2_WAIT(&o_done[qi], (j - 1) & 1, "o_done_rescale", j);  // PV_i(j-1) landed in O_i
          K2T_ADD(t_wo, t1);
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
        // P_i(j) over S_i's first 64 columns (S_i(j) is in registers; PV_i(j-1),
        // the previous reader, ran before S_i(j))
        tc::tmem_st32u(ts, pk);
        tc::tmem_st32u(ts + 32, pk + 32);
        tc::tmem_wait_st();
        tc::tc_fence_before();
        tc::mbar_arrive(&p_full[qi]);
      }
#ifdef CS_K2_TIMERS
      if (r == 0 && kvh == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - p.hkv) && blockIdx.z == 0)
        printf("K2T smax cta=%d qi=%d loop=%lld wait_s=%lld wait_o=%lld\n", blockIdx.x, qi, clock64() - t_sbegin,
               t_ws, t_wo);
#endif
      // epilogue: O_i / l -> HBM (or this split's partial -> workspace).
      // o_done may be 0..2 phases ahead here (parity-ambiguous): the last PV
      // signals its own barrier
      K2_WAIT(&o_final[qi], 0, "o_final", n_kt);
      tc::tc_fence_after();
      if (p.k2_splits > 1) {
        float* ws = p.ws2 + ((static_cast<size_t>(tile_idx) * p.hkv + kvh) * p.k2_splits + split) * (D + 2) * 256;
        const int rr = qi * kRows + r;
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          float o[32];
          tc::tmem_ld32(to + c * 32, o);
          tc::tmem_wait_ld();
          tc::reg_fence<32>(o);
#pragma unroll
          for (int i = 0; i < 32; ++i) ws[(c * 32 + i) * 256 + rr] = o[i];
        }
        ws[D * 256 + rr] = l > 0.f ? m_used : -INFINITY;
        ws[(D + 1) * 256 + rr] = l;
      } else {
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
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
#ifdef CS_K2_TIMERS
  if (threadIdx.x == 0 && kvh == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - p.hkv) && blockIdx.z == 0)
    printf("K2T cta  cta=%d n_kt=%d kernel=%lld\n", blockIdx.x, n_kt, clock64() - t_kernel);
#endif
  (void)t_kernel;
}

// Split-K merge for K2: one CTA per (tile, KV head, 32 head dims), one thread
// per packed row; partials are [d][row] so every load is coalesced across the
// rows, and the split weights are recomputed per split (no local arrays).
template <int D, int G>
__global__ void __launch_bounds__(256) attn_prefill_combine_kernel(AttnParams p) {
  const int tile = blockIdx.x, kvh = blockIdx.y, d0 = blockIdx.z * 32;
  if (tile >= p.desc->n_pt_cur) return;
  const PrefillTile t = p.tiles[tile];
  const int ent = t.entry;
  const int gr = t.row0 + threadIdx.x;
  if (gr >= p.ent_qlen[ent] * G) return;
  const int S = p.k2_splits;
  const float* ws = p.ws2 + (static_cast<size_t>(tile) * p.hkv + kvh) * S * (D + 2) * 256;
  const int r = threadIdx.x;
  float M = -INFINITY;
  for (int sp = 0; sp < S; ++sp) M = fmaxf(M, ws[(sp * (D + 2) + D) * 256 + r]);
  float o[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) o[i] = 0.f;
  float L = 0.f;
  for (int sp = 0; sp < S; ++sp) {
    const float* w_sp = ws + sp * (D + 2) * 256;
    const float m = w_sp[D * 256 + r];
    if (m == -INFINITY) continue;  // skipped splits may hold stale partials
    const float w = exp2f(m - M);
    L += w * w_sp[(D + 1) * 256 + r];
#pragma unroll
    for (int i = 0; i < 32; ++i) o[i] = fmaf(w, w_sp[(d0 + i) * 256 + r], o[i]);
  }
  const float inv = L > 0.f ? 1.f / L : 0.f;
  __nv_bfloat16* dst = p.out + static_cast<size_t>(p.ent_q0[ent] + gr / G) * p.hq * D +
                       static_cast<size_t>(kvh * G + gr % G) * D + d0;
#pragma unroll
  for (int i = 0; i < 32; i += 8)
    *reinterpret_cast<uint4*>(dst + i) =
        make_uint4(pack_bf16(o[i] * inv, o[i + 1] * inv), pack_bf16(o[i + 2] * inv, o[i + 3] * inv),
                   pack_bf16(o[i + 4] * inv, o[i + 5] * inv), pack_bf16(o[i + 6] * inv, o[i + 7] * inv));
}

template <int D, int G>
void launch_prefill_tc_t(const AttnParams& p, const CUtensorMap* kv_map, int n_pt_grid, cudaStream_t s) {
  smem_attr_once(reinterpret_cast<const void*>(attn_prefill_tc_kernel<D, G>), TcLayout<D>::launch_bytes);
  attn_prefill_tc_kernel<D, G><<<dim3(n_pt_grid * p.hkv, 1, p.k2_splits), kThreads, TcLayout<D>::launch_bytes, s>>>(
      p, *kv_map);
  if (p.k2_splits > 1) attn_prefill_combine_kernel<D, G><<<dim3(n_pt_grid, p.hkv, D / 32), 256, 0, s>>>(p);
}

// Rows per K2 work tile (engine.cu builds the tile list with this step).
int prefill_tile_rows() { return kQT * kRows; }
// Keys per K2 key tile (the unit of its split-K).
int prefill_tile_keys() { return kKeys; }

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
