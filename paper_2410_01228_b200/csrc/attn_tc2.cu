// K2 on CTA pairs (tcgen05 cta_group::2): prefill-chunk paged attention for
// head_dim 128 (reference stand-in: the k2*P(P+C) term of
// oracle_latency, proj/src/perf_model.cpp:56-65).
//
// Why pairs: the single-CTA kernel (attn_tc.cu) issues S = Q K^T with both
// operands in shared memory (SS, M=128 N=128) -- 128 B/clk of smem reads,
// exactly the smem port rate -- while TMA refills the K/V ring and the PV
// MMA reads V from smem too: ~125 B/clk of demand, so the MMAs and the K/V
// loads stall each other (role timers: the MMA warp blocked issuing ~2,400
// of ~3,400 cycles per key tile, waiting on K ~19%). With cta_group::2 the
// leader CTA issues M=256 MMAs over both CTAs' smem: A (the Q rows) is split
// by rows, B by columns -- each CTA stages HALF of every K tile (64 keys) and
// HALF of every V tile (64 head dims) -- so per SM the smem operand traffic
// and the K/V TMA bytes both halve (~78 B/clk of demand per key tile).
//
// Unit of work = one CTA pair x one KV head x 512 packed (token,
// head-in-group) rows of one entry, as four 128-row sub-tiles T0..T3:
// CTA r holds T_r (query tile 0) and T_{r+2} (query tile 1). The pair's MMA
// for query tile qi is M=256 = {T_qi of CTA 0, T_qi+... of CTA 1}: every
// CTA's TMEM receives its own 128 rows, so the softmax stays CTA-local
// exactly as in attn_tc.cu (one thread = one row = one TMEM lane, P written
// back over S as packed bf16, lazy O rescale, FFMA2 + polynomial exp2).
//
// Warp roles per CTA (320 threads): warps 0-3 softmax of query tile 0,
// 4-7 of query tile 1, warp 8 TMA producer (this CTA's K and V halves,
// completion counted on the LEADER's barriers), warp 9 MMA issuer (leader
// only). Barriers: k_full / v_full / p_full / q_ready live in the leader
// (expect-tx of both halves; remote arrivals from the peer), kv_empty /
// s_full / o_done / o_final in both CTAs (multicast commits).
// TMEM (512 cols per CTA): S_0 [0,128) S_1 [128,256) O_0 [256,384) O_1 [384,512).
#include "common.cuh"
#include "tc.cuh"

namespace csk {

namespace {

constexpr int kR = 128;      // rows per CTA per query tile (TMEM lanes)
constexpr int kKeys = 128;   // keys per key tile (pair-wide)
constexpr int kS = 3;        // K/V ring depth
constexpr int kPg = 16;
constexpr int kThr = 320;
constexpr int kD = 128;
constexpr int kQBytes = kR * 128;          // [128 rows][64 bf16] SWIZZLE_128B chunk = 16 KB
constexpr int kKHalf = (kKeys / 2) * 128;  // [64 keys][64 dims] chunk = 8 KB (x2 chunks per stage)
constexpr int kVHalf = kKeys * 128;        // [128 keys][64 dims] = 16 KB per stage
#ifndef CS_K2_POLY
#define CS_K2_POLY 2
#endif
constexpr int kPoly = CS_K2_POLY;

struct L2 {
  static constexpr int q = 0;                      // [tile 2][chunk 2] 16 KB
  static constexpr int k = q + 2 * 2 * kQBytes;    // [stage][chunk 2] 8 KB
  static constexpr int v = k + kS * 2 * kKHalf;    // [stage] 16 KB
  static constexpr int bar = v + kS * kVHalf;
  static constexpr int bytes = bar + 256 + 1024;
};

__device__ __forceinline__ int32_t pool_row2(const AttnParams& p, int32_t block, int which, int kvh) {
  const int64_t r = ((static_cast<int64_t>(block) * p.num_layers + p.layer) * 2 + which) * p.hkv + kvh;
  return static_cast<int32_t>(r * kPg);
}

// O (+)= P[tmem, M split over the pair] * V[smem, N split over the pair]
__device__ __forceinline__ void umma2_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

}  // namespace

template <int G>
__global__ void __launch_bounds__(kThr, 1)
    attn_prefill_tc2_kernel(AttnParams p, const __grid_constant__ CUtensorMap kv_map) {
  constexpr int CH = kD / 64;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t rank = tc::cluster_ctarank();
  const int unit = blockIdx.x >> 1;
  const int n_pt = p.desc->n_pt_cur;
  const int tile_idx = p.tile_order[unit / p.hkv];
  const int kvh = unit % p.hkv;
  if (tile_idx >= n_pt) return;  // pair-uniform: an offline tile dropped at a safepoint
  const PrefillTile t = p.tiles[tile_idx];
  const int ent = t.entry;
  const int q0 = p.ent_q0[ent];
  const int n_rows = p.ent_qlen[ent] * G;
  const int kv_len = p.ent_kvlen[ent];
  const int32_t* bt = p.block_table + p.ent_bt[ent];
  const int n_pages = (kv_len + kPg - 1) / kPg;
  const bool has2 = t.row0 + 2 * kR < n_rows;  // the pair's second M=256 tile
  const int last_row = min(t.row0 + 4 * kR, n_rows) - 1;
  const int kv_hi = min(kv_len, p.tok_pos[q0 + last_row / G] + 1);
  const int split = blockIdx.z;
  const int jb = split * p.k2_tiles_per_split;
  const int n_kt = min((kv_hi + kKeys - 1) / kKeys - jb, p.k2_tiles_per_split);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kWsRows = 4 * kR;

  if (n_kt <= 0) {  // pair-uniform: no keys of this split reach these rows
    if (p.k2_splits > 1) {
      float* ws = p.ws2 + ((static_cast<size_t>(tile_idx) * p.hkv + kvh) * p.k2_splits + split) * (kD + 2) * kWsRows;
      for (int r = threadIdx.x; r < 2 * kR; r += blockDim.x) {
        const int lr = (r >> 7) * 2 * kR + static_cast<int>(rank) * kR + (r & 127);
        ws[kD * kWsRows + lr] = -INFINITY;
      }
    }
    return;
  }
  uint8_t* sQ = smem + L2::q;
  uint8_t* sK = smem + L2::k;
  uint8_t* sV = smem + L2::v;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L2::bar);
  uint64_t* k_full = bars + 0;           // [kS]   leader
  uint64_t* v_full = k_full + kS;        // [kS]   leader
  uint64_t* kv_empty = v_full + kS;      // [kS]   both (multicast)
  uint64_t* s_full = kv_empty + kS;      // [2]    both (multicast)
  uint64_t* p_full = s_full + 2;         // [2]    leader (8 warp arrivals)
  uint64_t* o_done = p_full + 2;         // [2]    both (multicast)
  uint64_t* o_final = o_done + 2;        // [2]    both (multicast)
  uint64_t* q_ready = o_final + 2;       // [2]    leader (8 warp arrivals)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_ready + 2);

  if (threadIdx.x == 0) {
    for (int i = 0; i < kS; ++i) {
      tc::mbar_init(&k_full[i], 1);
      tc::mbar_init(&v_full[i], 1);
      tc::mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&s_full[i], 1);
      tc::mbar_init(&p_full[i], 8);
      tc::mbar_init(&o_done[i], 1);
      tc::mbar_init(&o_final[i], 1);
      tc::mbar_init(&q_ready[i], 8);
    }
    tc::fence_mbar_init();
  }
  if (warp == 8 && lane == 0) tc::prefetch_tmap(&kv_map);
  if (warp == 0) tc::tmem_alloc2<512>(tmem_slot);
  tc::tc_fence_before();
  tc::cluster_arrive_wait();  // barrier inits + TMEM address visible pair-wide
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // the leader's barriers, by their shared::cluster addresses
  const uint32_t k_full0 = tc::mapa(tc::smem_u32(k_full), 0);
  const uint32_t v_full0 = tc::mapa(tc::smem_u32(v_full), 0);
  const uint32_t p_full0 = tc::mapa(tc::smem_u32(p_full), 0);
  const uint32_t q_ready0 = tc::mapa(tc::smem_u32(q_ready), 0);

  // Q: softmax thread (qi, r) stages packed row row0 + 256 qi + 128 rank + r
  // (token q0 + gr / G, head kvh * G + gr % G) in the SWIZZLE_128B K-major
  // UMMA layout, then its warp arrives on the leader's q_ready[qi].
  if (warp < 8) {
    const int qi = warp >> 2, r = threadIdx.x & 127;
    if (qi == 0 || has2) {
      const int gr = t.row0 + qi * 2 * kR + static_cast<int>(rank) * kR + r;
      const bool valid = gr < n_rows;
      const __nv_bfloat16* src = p.qkv + static_cast<size_t>(q0 + (valid ? gr : 0) / G) * p.qkv_stride +
                                 static_cast<size_t>(kvh * G + (valid ? gr : 0) % G) * kD;
      uint8_t* dq = sQ + qi * CH * kQBytes;
#pragma unroll
      for (int c = 0; c < CH; ++c) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint4 val = valid ? *reinterpret_cast<const uint4*>(src + c * 64 + u * 8) : make_uint4(0, 0, 0, 0);
          *reinterpret_cast<uint4*>(dq + c * kQBytes + r * 128 + ((u ^ (r & 7)) << 4)) = val;
        }
      }
      tc::fence_async_smem();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive_cluster(q_ready0 + qi * 8);
    }
  }

  if (warp == 8) {
    // ------------------------------------------------------ TMA producer --
    // this CTA's halves: keys [64 rank, 64 rank + 64) of the tile (4 pages,
    // both 64-dim chunks) and head dims [64 rank, 64 rank + 64) of all 128
    // keys (8 pages); completion on the leader's barriers, whose expect-tx
    // (set by the leader's producer) covers both CTAs' bytes
    for (int j = 0; j < n_kt; ++j) {
      const int st = j % kS;
      if (j >= kS) tc::mbar_wait(&kv_empty[st], ((j / kS) - 1) & 1);
      const int pg = min((jb + j) * (kKeys / kPg) + (lane & 7), n_pages - 1);
      const int32_t blk = bt[pg];
      int32_t pblk[kKeys / kPg], kblk[4];
#pragma unroll
      for (int pi = 0; pi < kKeys / kPg; ++pi) pblk[pi] = __shfl_sync(0xffffffffu, blk, pi);
#pragma unroll
      for (int pi = 0; pi < 4; ++pi) kblk[pi] = __shfl_sync(0xffffffffu, blk, 4 * static_cast<int>(rank) + pi);
      if (tc::elect_one_sync()) {
        if (rank == 0) {
          tc::mbar_expect_tx(&k_full[st], 2 * CH * kKHalf);
          tc::mbar_expect_tx(&v_full[st], 2 * kVHalf);
        }
        uint8_t* dk = sK + st * CH * kKHalf;
#pragma unroll
        for (int pi = 0; pi < 4; ++pi) {
          const int32_t row = pool_row2(p, kblk[pi], 0, kvh);
#pragma unroll
          for (int c = 0; c < CH; ++c)
            tc::tma_load_2d_pair(dk + c * kKHalf + pi * kPg * 128, &kv_map, k_full0 + st * 8, c * 64, row);
        }
        uint8_t* dv = sV + st * kVHalf;
#pragma unroll
        for (int pi = 0; pi < kKeys / kPg; ++pi) {
          const int32_t row = pool_row2(p, pblk[pi], 1, kvh);
          tc::tma_load_2d_pair(dv + pi * kPg * 128, &kv_map, v_full0 + st * 8, static_cast<int>(rank) * 64, row);
        }
      }
      __syncwarp();
    }
  } else if (warp == 9) {
    // -------------------------------------------------------- MMA issuer --
    if (rank == 0) {
      constexpr uint32_t idesc_s = tc::idesc_bf16_f32(2 * kR, kKeys, false, false);
      constexpr uint32_t idesc_o = tc::idesc_bf16_f32(2 * kR, kD, false, true);
      const uint32_t q_addr = tc::smem_u32(sQ), k_addr = tc::smem_u32(sK), v_addr = tc::smem_u32(sV);
      const int nq = has2 ? 2 : 1;
      auto issue_s = [&](int qi, int j) {
        const uint32_t kb = k_addr + (j % kS) * CH * kKHalf;
        const uint32_t qb = q_addr + qi * CH * kQBytes;
        const uint32_t d_tmem = tmem + qi * 128;
        if (tc::elect_one_sync()) {
#pragma unroll
          for (int ks = 0; ks < kD / 16; ++ks) {
            const uint32_t qoff = (ks >> 2) * kQBytes + (ks & 3) * 32;
            const uint32_t koff = (ks >> 2) * kKHalf + (ks & 3) * 32;
            tc::umma2_bf16_ss(d_tmem, tc::sdesc_sw128(qb + qoff, 16, 1024), tc::sdesc_sw128(kb + koff, 16, 1024),
                              idesc_s, ks > 0 ? 1u : 0u);
          }
          tc::umma2_commit_mc(&s_full[qi], 0x3);
        }
        __syncwarp();
      };
      auto issue_pv = [&](int qi, int j, bool release_stage) {
        const uint32_t vb = v_addr + (j % kS) * kVHalf;
        const uint32_t pa = tmem + qi * 128;
        const uint32_t d_tmem = tmem + 256 + qi * 128;
        if (tc::elect_one_sync()) {
#pragma unroll
          for (int ks = 0; ks < kKeys / 16; ++ks)
            umma2_bf16_ts(d_tmem, pa + ks * 8, tc::sdesc_sw128(vb + ks * 16 * 128, kVHalf, 1024), idesc_o,
                          (j > 0 || ks > 0) ? 1u : 0u);
          tc::umma2_commit_mc(&o_done[qi], 0x3);
          if (j == n_kt - 1) tc::umma2_commit_mc(&o_final[qi], 0x3);
          if (release_stage) tc::umma2_commit_mc(&kv_empty[j % kS], 0x3);
        }
        __syncwarp();
      };
      auto wait_k = [&](int j) {
        tc::mbar_wait(&k_full[j % kS], (j / kS) & 1);
        tc::tc_fence_after();
      };
      wait_k(0);
      for (int qi = 0; qi < nq; ++qi) {
        tc::mbar_wait(&q_ready[qi], 0);
        issue_s(qi, 0);
      }
      for (int j = 0; j < n_kt; ++j) {
        tc::mbar_wait(&v_full[j % kS], (j / kS) & 1);
        const bool next = j + 1 < n_kt;
        if (next) wait_k(j + 1);
        for (int qi = 0; qi < nq; ++qi) {
          tc::mbar_wait(&p_full[qi], j & 1);
          tc::tc_fence_after();
          issue_pv(qi, j, qi == nq - 1);
          if (next) issue_s(qi, j + 1);
        }
      }
    }
  } else {
    // ------------------------------------------- softmax + epilogue (rows) --
    const int qi = warp >> 2, r = threadIdx.x & 127;
    if (qi == 0 || has2) {
      const int lr = qi * 2 * kR + static_cast<int>(rank) * kR + r;  // row within the 512-row unit
      const int gr = t.row0 + lr;
      const bool valid = gr < n_rows;
      const int pos = p.tok_pos[q0 + (valid ? gr : last_row) / G];
      const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
      const uint32_t ts = tmem + lane_base + qi * 128;
      const uint32_t to = tmem + lane_base + 256 + qi * 128;
      const float scale = p.scale_log2;
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j < n_kt; ++j) {
        tc::mbar_wait(&s_full[qi], j & 1);
        tc::tc_fence_after();
        float s[kKeys];
#pragma unroll
        for (int c = 0; c < kKeys / 32; ++c) tc::tmem_ld32(ts + c * 32, s + c * 32);
        tc::tmem_wait_ld();
        tc::reg_fence<kKeys>(s);
        const int kbase = (jb + j) * kKeys;
        if (kbase + kKeys - 1 > pos) {
#pragma unroll
          for (int i = 0; i < kKeys; ++i) s[i] = (kbase + i <= pos) ? s[i] : -INFINITY;
        }
        float mxa[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) mxa[a] = s[a];
#pragma unroll
        for (int i = 8; i < kKeys; ++i) mxa[i & 7] = fmaxf(mxa[i & 7], s[i]);
        const float mx = fmaxf(fmaxf(fmaxf(mxa[0], mxa[1]), fmaxf(mxa[2], mxa[3])),
                               fmaxf(fmaxf(mxa[4], mxa[5]), fmaxf(mxa[6], mxa[7])));
        const float m_new = fmaxf(m_used, mx * scale);
        const bool rescale = m_new > m_used + 8.f;
        const float alpha = rescale ? tc::ex2_approx(m_used - m_new) : 1.f;
        if (rescale) m_used = m_new;
        const float msub = m_used == -INFINITY ? 0.f : m_used;
        uint32_t pk[kKeys / 2];
        const float2 sc2 = make_float2(scale, scale), ms2 = make_float2(-msub, -msub);
        float2 rsa[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
        for (int i = 0; i < kKeys; i += 2) {
          const float2 x = __ffma2_rn(make_float2(s[i], s[i + 1]), sc2, ms2);
          const float2 pp = ((i >> 1) & 7) < kPoly ? tc::ex2_poly2(x)
                                                   : make_float2(tc::ex2_approx(x.x), tc::ex2_approx(x.y));
          rsa[(i >> 1) & 1] = __fadd2_rn(rsa[(i >> 1) & 1], pp);
          pk[i / 2] = pack_bf16(pp.x, pp.y);
        }
        const float rs = (rsa[0].x + rsa[1].x) + (rsa[0].y + rsa[1].y);
        l = l * alpha + rs;
        if (__any_sync(0xffffffffu, rescale) && j > 0) {
          tc::mbar_wait(&o_done[qi], (j - 1) & 1);  // PV(j-1) landed in O
          tc::tc_fence_after();
#pragma unroll
          for (int c = 0; c < kD / 32; ++c) {
            float o[32];
            tc::tmem_ld32(to + c * 32, o);
            tc::tmem_wait_ld();
            tc::reg_fence<32>(o);
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] *= alpha;
            tc::tmem_st32(to + c * 32, o);
          }
        }
        tc::tmem_st32u(ts, pk);
        tc::tmem_st32u(ts + 32, pk + 32);
        tc::tmem_wait_st();
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive_cluster(p_full0 + qi * 8);
      }
      tc::mbar_wait(&o_final[qi], 0);
      tc::tc_fence_after();
      if (p.k2_splits > 1) {
        float* ws =
            p.ws2 + ((static_cast<size_t>(tile_idx) * p.hkv + kvh) * p.k2_splits + split) * (kD + 2) * kWsRows;
#pragma unroll
        for (int c = 0; c < kD / 32; ++c) {
          float o[32];
          tc::tmem_ld32(to + c * 32, o);
          tc::tmem_wait_ld();
          tc::reg_fence<32>(o);
#pragma unroll
          for (int i = 0; i < 32; ++i) ws[(c * 32 + i) * kWsRows + lr] = o[i];
        }
        ws[kD * kWsRows + lr] = l > 0.f ? m_used : -INFINITY;
        ws[(kD + 1) * kWsRows + lr] = l;
      } else {
        const float inv = l > 0.f ? 1.f / l : 0.f;
        __nv_bfloat16* dst = p.out + static_cast<size_t>(q0 + (valid ? gr : 0) / G) * p.hq * kD +
                             static_cast<size_t>(kvh * G + (valid ? gr : 0) % G) * kD;
#pragma unroll
        for (int c = 0; c < kD / 32; ++c) {
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
  tc::cluster_arrive_wait();  // the leader's MMAs read this CTA's smem / write its TMEM until o_final
  tc::tc_fence_after();
  if (warp == 0) tc::tmem_dealloc2<512>(tmem);
}

// Split-K merge for the pair kernel: one CTA per (tile, KV head, 32 head
// dims), one thread per packed row of the 512-row unit.
template <int G>
__global__ void __launch_bounds__(512) attn_prefill_combine2_kernel(AttnParams p) {
  constexpr int kWsRows = 4 * kR;
  const int tile = blockIdx.x, kvh = blockIdx.y, d0 = blockIdx.z * 32;
  if (tile >= p.desc->n_pt_cur) return;
  const PrefillTile t = p.tiles[tile];
  const int ent = t.entry;
  const int gr = t.row0 + threadIdx.x;
  if (gr >= p.ent_qlen[ent] * G) return;
  const int S = p.k2_splits;
  const float* ws = p.ws2 + (static_cast<size_t>(tile) * p.hkv + kvh) * S * (kD + 2) * kWsRows;
  const int r = threadIdx.x;
  float M = -INFINITY;
  for (int sp = 0; sp < S; ++sp) M = fmaxf(M, ws[(sp * (kD + 2) + kD) * kWsRows + r]);
  float o[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) o[i] = 0.f;
  float L = 0.f;
  for (int sp = 0; sp < S; ++sp) {
    const float* w_sp = ws + sp * (kD + 2) * kWsRows;
    const float m = w_sp[kD * kWsRows + r];
    if (m == -INFINITY) continue;
    const float w = exp2f(m - M);
    L += w * w_sp[(kD + 1) * kWsRows + r];
#pragma unroll
    for (int i = 0; i < 32; ++i) o[i] = fmaf(w, w_sp[(d0 + i) * kWsRows + r], o[i]);
  }
  const float inv = L > 0.f ? 1.f / L : 0.f;
  __nv_bfloat16* dst = p.out + static_cast<size_t>(p.ent_q0[ent] + gr / G) * p.hq * kD +
                       static_cast<size_t>(kvh * G + gr % G) * kD + d0;
#pragma unroll
  for (int i = 0; i < 32; i += 8)
    *reinterpret_cast<uint4*>(dst + i) =
        make_uint4(pack_bf16(o[i] * inv, o[i + 1] * inv), pack_bf16(o[i + 2] * inv, o[i + 3] * inv),
                   pack_bf16(o[i + 4] * inv, o[i + 5] * inv), pack_bf16(o[i + 6] * inv, o[i + 7] * inv));
}

template <int G>
static void launch_tc2_t(const AttnParams& p, const CUtensorMap* kv_map, int n_pt_grid, cudaStream_t s) {
  smem_attr_once(reinterpret_cast<const void*>(attn_prefill_tc2_kernel<G>), L2::bytes);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(n_pt_grid * p.hkv * 2, 1, p.k2_splits);
  cfg.blockDim = dim3(kThr, 1, 1);
  cfg.dynamicSmemBytes = L2::bytes;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, attn_prefill_tc2_kernel<G>, p, *kv_map);
  if (p.k2_splits > 1)
    attn_prefill_combine2_kernel<G><<<dim3(n_pt_grid, p.hkv, kD / 32), 4 * kR, 0, s>>>(p);
}

// Rows per pair work tile (engine.cu builds the tile list with this step).
int prefill_tc2_tile_rows() { return 4 * kR; }

// The pair kernel covers head_dim 128; false for other shapes (the single-CTA
// kernel in attn_tc.cu serves them).
bool launch_prefill_tc2(const AttnParams& p, const CUtensorMap* kv_map, int head_dim, int group, int n_pt_grid,
                        cudaStream_t s) {
  if (head_dim != kD) return false;
  switch (group) {
    case 1: launch_tc2_t<1>(p, kv_map, n_pt_grid, s); return true;
    case 2: launch_tc2_t<2>(p, kv_map, n_pt_grid, s); return true;
    case 4: launch_tc2_t<4>(p, kv_map, n_pt_grid, s); return true;
    case 5: launch_tc2_t<5>(p, kv_map, n_pt_grid, s); return true;
    case 8: launch_tc2_t<8>(p, kv_map, n_pt_grid, s); return true;
    default: return false;
  }
}

}  // namespace csk
