// Shared device helpers and the per-iteration descriptor layout.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <mutex>
#include <utility>

namespace csk {

// Opt a kernel into `bytes` of dynamic shared memory on the current device.
// The attribute is per device, so it is remembered per (kernel, device): one
// process may drive several GPUs (or several engines share one).
inline void smem_attr_once(const void* fn, int bytes) {
  static std::mutex m;
  static std::map<std::pair<const void*, int>, int> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(m);
  int& have = done[std::make_pair(fn, dev)];
  if (have >= bytes) return;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  have = bytes;
}

// Programmatic dependent launch: lets a kernel launched with the
// programmatic-serialization attribute (K7) start before this one finishes;
// its griddepcontrol.wait still blocks until this grid completed and its
// writes are visible. A no-op when no such dependent is queued.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Per-iteration counts. Written by the host (H2D) before the forward; the
// safepoint kernel truncates the *_cur fields in place to the online prefix
// when the preemption flag carries this iteration's epoch.
// Every kernel reads the *_cur counts, so a drop takes effect at the next
// launch on the stream without host involvement.
struct IterDesc {
  int32_t n_tok_cur, n_tok_all, n_tok_on;      // token rows (GEMM M)
  int32_t n_ent_cur, n_ent_all, n_ent_on;      // plan entries
  int32_t n_dec_cur, n_dec_all, n_dec_on;      // single-query attention rows
  int32_t n_pt_cur, n_pt_all, n_pt_on;         // prefill attention tiles
  int32_t dropped_at;                          // layer of the drop, -1 if none
  int32_t dec_splits;                          // K1 split-K: active splits (<= launch grid.x)
  int32_t dec_pps;                             // K1 split-K: pages per split
  int32_t pad0;
  uint64_t epoch;
  uint64_t drop_ns;                            // %globaltimer at the drop
  uint64_t start_ns;                           // %globaltimer at layer 0's head (instrumented plans)
};

// Mapped (zero-copy) host<->device record for the preemption handshake.
struct PreemptMailbox {
  volatile uint64_t flag_epoch;      // host writes the epoch to preempt
  volatile uint64_t flag_host_ns;    // host CLOCK_MONOTONIC at the store
  volatile int32_t seen_layer;       // device: layer of the observed drop
  volatile int32_t pad;
  volatile uint64_t seen_epoch;      // device: epoch it dropped
  volatile uint64_t seen_gpu_ns;     // device %globaltimer at the drop
  volatile uint64_t progress;        // device: epoch * 1024 + layer the forward has entered
};

// Layer-boundary preemption check fused into the layer's first kernel
// (add_rmsnorm): CTA 0 reads the mailbox and truncates the descriptor; the
// kernel boundary publishes the truncation to every later launch.
struct SafepointArg {
  PreemptMailbox* mb;          // mapped mailbox (null: no check, no progress)
  const __nv_bfloat16* tail;   // TP: the all-reduced vote (mode 2)
  int32_t layer;
  int32_t mode;                // 0 progress only, 1 host flag (g = 1), 2 agreed vote (g > 1)
};

// Prefill tile: TILE_ROWS query rows (token, head-in-group) of one entry.
struct PrefillTile {
  int32_t entry;
  int32_t row0;      // first packed row (token_local * G + h) within the entry
};

// Up to 3 (local_start, global_start) row segments: maps a rank's rows of a
// sharded weight onto the global tensor (q|k|v or gate|up blocks).
struct RowMap {
  int32_t n;
  int32_t local_start[3];
  int64_t global_start[3];
};

struct AttnParams {
  const __nv_bfloat16* qkv;     // [T, (Hq + 2 Hkv) * D] rank-local heads
  __nv_bfloat16* out;           // [T, Hq * D]
  const __nv_bfloat16* pool;    // KV pool [blocks][L][2][Hkv][16][D]
  const IterDesc* desc;
  const int32_t* tok_pos;       // [T]
  const int32_t* ent_q0;        // [E] first token row of the entry
  const int32_t* ent_qlen;      // [E]
  const int32_t* ent_kvlen;     // [E]
  const int32_t* ent_bt;        // [E] offset into block_table
  const int32_t* block_table;   // flat
  const int32_t* dec_ent;       // [n_dec] entry index of single-query entries
  const PrefillTile* tiles;     // [n_pt]
  const int32_t* tile_order;    // [n_pt] K2 launch order: tile indices, most keys first
  float* ws;                    // K1 split-K partials
  int32_t* dec_cnt;             // K1 split-K arrival counters [entry][kv head], self-resetting
  float* ws2;                   // K2 split-K partials [tile][kvh][split] x {O [D][256], m [256], l [256]}
  int32_t layer, num_layers, hq, hkv, qkv_stride;
  int32_t n_splits, pages_per_split;   // K1: splits over pages
  const int32_t* dec_pfx;       // [n_dec + 1] K1 stream-K: prefix sums of the decode entries' page counts
  float* ws_sk;                 // K1 stream-K partials [cta][2] x {m[G], l[G], O[G][D]}
  int32_t sk_ctas;              // K1 stream-K grid (0: the split-K kernel)
  int32_t sk_stages;            // K1 stream-K per-warp ring depth (2 or 3)
  // decode-only (CUDA-graph) iterations: K1 applies RoPE to q in registers
  // and the CTA reading a pair's last page appends the new token's k / v
  // (rope_append does not run); qkv then holds un-rotated q / k
  int32_t k1_rope;
  float rope_theta;
  const float2* rope_tab;       // [T][D/2] (cos, sin) of the iteration (rope_table_kernel)
  const int32_t* tok_slot;      // [T] block * 16 + slot of each token row
  int32_t k2_splits, k2_tiles_per_split;  // K2: splits over 128-key tiles
  int32_t k2_pair;                        // K2 on CTA pairs (attn_tc2.cu, head_dim 128)
  float scale_log2;             // softmax_scale * log2(e)
};

// K8 epilogue fusions (gemm_pf.cu), tp = 1 prefill layers:
//  * resid: y = x + acc -- the residual add of the next RMSNorm, written in
//    place over x (bit-identical to storing acc as bf16 and adding after);
//  * rope: the qkv projection's q / k heads rotated (RoPE, (cos, sin) from a
//    per-iteration [token][D/2] table) and k / v scattered into the KV pool
//    at each token's (block, slot) -- bit-identical to rope_append.
struct PfExtra {
  __nv_bfloat16* resid = nullptr;     // x [M, N] bf16, updated in place (y unused)
  const float2* rope_tab = nullptr;   // [token][D/2] (cos, sin); null: no rope
  const int32_t* tok_slot = nullptr;  // [token] block * 16 + slot
  __nv_bfloat16* pool = nullptr;
  int32_t hq = 0, hkv = 0, D = 0, num_layers = 0, layer = 0;
};

// Peer-memory all-reduce arguments (kernels.cu p2p_allreduce): for each of
// the g ranks, the partial buffer of this step and its exchange-region words.
struct P2PArgs {
  const __nv_bfloat16* part[8];
  uint64_t* flag[8];   // published step of each rank
  uint64_t* step[8];   // step counter of each rank (only step[rank] is used)
  uint64_t* flag2[8];  // two-shot: reduce-scatter phase published by each rank
  int* arrive;         // this rank's block-arrival counter
  int* arrive2;        // two-shot: this rank's reduce-scatter arrival counter
  int32_t rank, g;
};

__host__ __device__ inline uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

// Teacher-forced synthetic token id: id(req,pos).
__host__ __device__ inline int32_t token_id(uint64_t seed, int64_t req, int64_t pos, int32_t vocab) {
  uint64_t h = mix64(seed ^ mix64(static_cast<uint64_t>(req) * 0x100000001b3ULL + static_cast<uint64_t>(pos)));
  return static_cast<int32_t>(h % static_cast<uint64_t>(vocab));
}

// Uniform in [-1, 1) from (seed, tensor, index); used for random-init weights.
__host__ __device__ inline float hash_uniform(uint64_t seed, uint64_t tensor, uint64_t idx) {
  uint64_t h = mix64(seed ^ mix64(tensor * 0x9E3779B97F4A7C15ULL ^ mix64(idx)));
  return static_cast<float>(static_cast<int64_t>(h >> 40) - (1LL << 23)) * (1.0f / 8388608.0f);
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ void ldmatrix_x4(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, const void* p) {
  uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(p));
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(s));
}
__device__ __forceinline__ void ldmatrix_x4_trans(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3,
                                                  const void* p) {
  uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(p));
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(s));
}

// D = A(16x16 bf16, row) * B(16x8 bf16, col) + D (fp32)
__device__ __forceinline__ void mma_bf16_16816(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Byte offset of 16-byte chunk c of row r in a [rows][D] bf16 tile stored
// with an XOR swizzle over 8-chunk groups (conflict-free ldmatrix).
template <int D>
__device__ __forceinline__ uint32_t swz(int r, int c) {
  return static_cast<uint32_t>(r * (D * 2) + ((c ^ (r & 7)) << 4));
}

}  // namespace csk
