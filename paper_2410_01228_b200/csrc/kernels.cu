// Element-wise / row kernels of the layer forward, the KV
// append (K3), the preemption safepoint (K6) and the checkpoint gather /
// restore scatter over the host link (K4 / K5).
#include <algorithm>
#include <cstdio>

#include <cstdlib>

#include "common.cuh"

namespace csk {

// ------------------------------------------------------------- weights ----
// Deterministic random init by GLOBAL element index so a KV-head-sharded
// rank holds exactly its slice of the unsharded tensor. Rows map through up
// to 3 (local_start, global_start) segments (q|k|v or gate|up blocks).

__global__ void init_matrix_kernel(__nv_bfloat16* w, int64_t rows, int64_t cols, int64_t global_cols,
                                   int64_t col_off, RowMap map, uint64_t seed, uint64_t tensor, float scale,
                                   float offset) {
  const int64_t total = rows * cols;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / cols, c = i % cols;
    int seg = 0;
    for (int s = 1; s < map.n; ++s)
      if (r >= map.local_start[s]) seg = s;
    const int64_t gr = map.global_start[seg] + (r - map.local_start[seg]);
    const uint64_t gidx = static_cast<uint64_t>(gr * global_cols + col_off + c);
    const float u = hash_uniform(seed, tensor, gidx);
    w[i] = __float2bfloat16_rn(__fadd_rn(offset, __fmul_rn(scale, u)));
  }
}

void init_matrix(__nv_bfloat16* w, int64_t rows, int64_t cols, int64_t global_cols, int64_t col_off,
                 const RowMap& map, uint64_t seed, uint64_t tensor, float scale, float offset, cudaStream_t s) {
  init_matrix_kernel<<<1184, 256, 0, s>>>(w, rows, cols, global_cols, col_off, map, seed, tensor, scale, offset);
}

// ------------------------------------------------------------ embedding ----
__global__ void embed_kernel(__nv_bfloat16* x, const __nv_bfloat16* emb, const int32_t* tok_ids, int hidden,
                             const IterDesc* desc) {
  const int t = blockIdx.x;
  if (t >= desc->n_tok_cur) return;
  const uint4* src = reinterpret_cast<const uint4*>(emb + static_cast<size_t>(tok_ids[t]) * hidden);
  uint4* dst = reinterpret_cast<uint4*>(x + static_cast<size_t>(t) * hidden);
  for (int i = threadIdx.x; i < hidden / 8; i += blockDim.x) dst[i] = src[i];
}

void embed(__nv_bfloat16* x, const __nv_bfloat16* emb, const int32_t* tok_ids, int hidden, const IterDesc* desc,
           int grid, cudaStream_t s) {
  if (grid > 0) embed_kernel<<<grid, 128, 0, s>>>(x, emb, tok_ids, hidden, desc);
}

// --------------------------------------------------------- add + RMSNorm ----
// x[r] += add[r] (if add), xn[r'] = x[r] * rsqrt(mean(x^2) + eps) * w.
// rows: the row set is all token rows (< n_tok_cur) or, with row_idx, the
// gathered rows row_idx[i] for i < n_ent_cur (final norm of sampled rows).
// One CTA per row, CH 16-byte chunks per thread kept in registers: one read
// of x (and add), one write of x and xn.
// Truncates every *_cur count to the online prefix (online entries form a
// prefix of the plan, scheduler.cpp:183-317) and records the layer + device
// time in the mapped mailbox.
__device__ __forceinline__ void apply_drop(IterDesc* desc, PreemptMailbox* mb, int layer) {
  desc->n_tok_cur = desc->n_tok_on;
  desc->n_ent_cur = desc->n_ent_on;
  desc->n_dec_cur = desc->n_dec_on;
  desc->n_pt_cur = desc->n_pt_on;
  desc->dropped_at = layer;
  const uint64_t now = globaltimer_ns();
  desc->drop_ns = now;
  mb->seen_layer = layer;
  mb->seen_gpu_ns = now;
  __threadfence_system();
  mb->seen_epoch = desc->epoch;
}

// K6 at the head of layer `sp.layer` (one thread): publish progress, then if
// the host flag carries this iteration's epoch (g = 1) or the all-reduced
// vote is set (g > 1) and offline work remains, drop it.
__device__ __forceinline__ void safepoint_check(IterDesc* desc, const SafepointArg& sp) {
  if (sp.mb == nullptr) return;
  if (sp.layer == 0) desc->start_ns = globaltimer_ns();
  // the flag is read BEFORE this layer's progress is published: a host that
  // stores the flag on seeing layer l (the reference's Alg. 1 firing inside
  // layer l) must land the drop at layer l + 1, never at l itself (the read
  // would otherwise race the host's reaction to the progress write)
  const uint64_t flag = sp.mb->flag_epoch;
  __threadfence_system();
  sp.mb->progress = desc->epoch * 1024ull + static_cast<uint64_t>(sp.layer);
  if (sp.mode == 0 || desc->dropped_at >= 0) return;
  if (sp.mode == 1) {
    if (flag != desc->epoch) return;
    if (desc->n_ent_on >= desc->n_ent_cur) return;  // nothing offline to drop
  } else if (__bfloat162float(sp.tail[0]) <= 0.f) {
    return;
  }
  apply_drop(desc, sp.mb, sp.layer);
}

template <int CH>
__global__ void add_rmsnorm_kernel(__nv_bfloat16* x, const __nv_bfloat16* add, const __nv_bfloat16* w,
                                   __nv_bfloat16* xn, int hidden, float eps, const IterDesc* desc,
                                   const int32_t* row_idx, SafepointArg sp, unsigned long long* zero_keys) {
  pdl_trigger();  // the next projection (K7) may start streaming its weights
  const int i = blockIdx.x;
  if (sp.mb != nullptr && i == static_cast<int>(gridDim.x) - 1) {
    // one extra CTA runs K6 (the mapped-mailbox read is a PCIe round trip)
    // while the row CTAs normalise: rows may see the counts before or after
    // the drop; a dropped row's norm is never read again, the next launch
    // sees the cut
    if (threadIdx.x == 0) safepoint_check(const_cast<IterDesc*>(desc), sp);
    return;
  }
  // final norm: re-arm the argmax key of this entry row (argmax_kernel
  // atomicMax-es into it after the lm_head), instead of a memset node
  if (zero_keys != nullptr && threadIdx.x == 0) zero_keys[i] = 0ull;
  int r;
  if (row_idx != nullptr) {
    if (i >= desc->n_ent_cur) return;
    r = row_idx[i];
  } else {
    if (i >= desc->n_tok_cur) return;
    r = i;
  }
  __nv_bfloat16* xr = x + static_cast<size_t>(r) * hidden;
  const __nv_bfloat16* ar = add ? add + static_cast<size_t>(r) * hidden : nullptr;
  // the norm weights are loaded with x (not after the reduction): one memory
  // round trip less on this latency-bound kernel
  uint4 wv[CH];
#pragma unroll
  for (int k = 0; k < CH; ++k) {
    const int c = (k * blockDim.x + threadIdx.x) * 8;
    if (c < hidden) wv[k] = *reinterpret_cast<const uint4*>(w + c);
  }
  float v[CH][8];
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < CH; ++k) {
    const int c = (k * blockDim.x + threadIdx.x) * 8;
    if (c >= hidden) {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[k][j] = 0.f;
      continue;
    }
    const uint4 xv = *reinterpret_cast<const uint4*>(xr + c);
    const __nv_bfloat16* xe = reinterpret_cast<const __nv_bfloat16*>(&xv);
#pragma unroll
    for (int j = 0; j < 8; ++j) v[k][j] = __bfloat162float(xe[j]);
    if (ar) {
      const uint4 av = *reinterpret_cast<const uint4*>(ar + c);
      const __nv_bfloat16* ae = reinterpret_cast<const __nv_bfloat16*>(&av);
      __nv_bfloat16 outv[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        outv[j] = __float2bfloat16(v[k][j] + __bfloat162float(ae[j]));
        v[k][j] = __bfloat162float(outv[j]);
      }
      *reinterpret_cast<uint4*>(xr + c) = *reinterpret_cast<const uint4*>(outv);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) ss += v[k][j] * v[k][j];
  }
  __shared__ float part[32];
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < (blockDim.x >> 5) ? part[threadIdx.x] : 0.f;
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) part[0] = t;
  }
  __syncthreads();
  const float inv = rsqrtf(part[0] / hidden + eps);
  __nv_bfloat16* yr = xn + static_cast<size_t>(row_idx ? i : r) * hidden;
#pragma unroll
  for (int k = 0; k < CH; ++k) {
    const int c = (k * blockDim.x + threadIdx.x) * 8;
    if (c >= hidden) continue;
    const __nv_bfloat16* we = reinterpret_cast<const __nv_bfloat16*>(&wv[k]);
    __nv_bfloat16 outv[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) outv[j] = __float2bfloat16(v[k][j] * inv * __bfloat162float(we[j]));
    *reinterpret_cast<uint4*>(yr + c) = *reinterpret_cast<const uint4*>(outv);
  }
}

void add_rmsnorm(__nv_bfloat16* x, const __nv_bfloat16* add, const __nv_bfloat16* w, __nv_bfloat16* xn, int hidden,
                 float eps, const IterDesc* desc, const int32_t* row_idx, int grid, cudaStream_t s,
                 const SafepointArg& sp, unsigned long long* zero_keys) {
  if (grid <= 0) return;
  if (sp.mb != nullptr) ++grid;  // + the K6 CTA
  const int vec = hidden / 8;
  // <= 512 threads: CH = ceil(vec / 512) chunks each (hidden <= 16384)
  const int threads = std::min(512, ((vec + 31) / 32) * 32);
  const int ch = (vec + threads - 1) / threads;
  if (ch == 1)
    add_rmsnorm_kernel<1><<<grid, threads, 0, s>>>(x, add, w, xn, hidden, eps, desc, row_idx, sp, zero_keys);
  else if (ch == 2)
    add_rmsnorm_kernel<2><<<grid, threads, 0, s>>>(x, add, w, xn, hidden, eps, desc, row_idx, sp, zero_keys);
  else
    add_rmsnorm_kernel<4><<<grid, threads, 0, s>>>(x, add, w, xn, hidden, eps, desc, row_idx, sp, zero_keys);
}

// ----------------------------------------------------------------- SwiGLU ----
// act[t, c] = silu(gate[t, c]) * up[t, c]. gu row layout: gate | up
// (interleave = 0) or gate|up interleaved in 128-column blocks (the weight
// layout K8 fuses this into its epilogue with; interleave = 1).
__global__ void silu_mul_kernel(const __nv_bfloat16* gu, __nv_bfloat16* act, int ffn, const IterDesc* desc,
                                int interleave) {
  pdl_trigger();
  const int t = blockIdx.y;
  if (t >= desc->n_tok_cur) return;
  const __nv_bfloat16* row = gu + static_cast<size_t>(t) * 2 * ffn;
  __nv_bfloat16* a = act + static_cast<size_t>(t) * ffn;
  for (int c = (blockIdx.x * blockDim.x + threadIdx.x) * 8; c < ffn; c += gridDim.x * blockDim.x * 8) {
    const int gc = interleave ? (c >> 7) * 256 + (c & 127) : c;
    const int uc = interleave ? gc + 128 : c + ffn;
    uint4 gv = *reinterpret_cast<const uint4*>(row + gc);
    uint4 uv = *reinterpret_cast<const uint4*>(row + uc);
    const __nv_bfloat16* ge = reinterpret_cast<const __nv_bfloat16*>(&gv);
    const __nv_bfloat16* ue = reinterpret_cast<const __nv_bfloat16*>(&uv);
    __nv_bfloat16 o[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float gf = __bfloat162float(ge[j]);
      o[j] = __float2bfloat16(gf / (1.f + __expf(-gf)) * __bfloat162float(ue[j]));
    }
    *reinterpret_cast<uint4*>(a + c) = *reinterpret_cast<uint4*>(o);
  }
}

void silu_mul(const __nv_bfloat16* gu, __nv_bfloat16* act, int ffn, const IterDesc* desc, int grid_rows,
              cudaStream_t s, bool interleave) {
  if (grid_rows <= 0) return;
  const int bx = (ffn / 8 + 255) / 256;
  silu_mul_kernel<<<dim3(bx < 1 ? 1 : (bx > 16 ? 16 : bx), grid_rows), 256, 0, s>>>(gu, act, ffn, desc,
                                                                                  interleave ? 1 : 0);
}

// ------------------------------------------------- RoPE + KV append (K3) ----
// Rotates q and k of every token row in place (rotate-half convention) and
// scatters k, v into the token's (block, slot) of this layer of the pool.
// One CTA per token: the D/2 (cos, sin) pairs of the token's position are
// computed once (accurate sincosf: positions reach 64K) and shared by all
// Hq + Hkv heads; rotations and the v copy move 16-B vectors (D % 16 == 0).
__global__ void __launch_bounds__(128) rope_append_kernel(__nv_bfloat16* qkv, const int32_t* tok_pos,
                                                          const int32_t* tok_slot, __nv_bfloat16* pool, int hq,
                                                          int hkv, int D, int num_layers, int layer, float theta,
                                                          const IterDesc* desc) {
  const int t = blockIdx.x;
  if (t >= desc->n_tok_cur) return;
  __shared__ float2 rot[128];  // (cos, sin) per frequency, D <= 256
  const int stride = (hq + 2 * hkv) * D;
  __nv_bfloat16* row = qkv + static_cast<size_t>(t) * stride;
  const float pos = static_cast<float>(tok_pos[t]);
  const int half = D / 2;
  for (int j = threadIdx.x; j < half; j += blockDim.x) {
    const float inv_freq = powf(theta, -2.f * static_cast<float>(j) / static_cast<float>(D));
    float sn, cs;
    sincosf(pos * inv_freq, &sn, &cs);
    rot[j] = make_float2(cs, sn);
  }
  __syncthreads();
  const int slot = tok_slot[t];
  const int blk = slot >> 4, off = slot & 15;
  const size_t layer_elems = static_cast<size_t>(2) * hkv * 16 * D;
  __nv_bfloat16* kv_base = pool + (static_cast<size_t>(blk) * num_layers + layer) * layer_elems;
  // 8 consecutive (j .. j+7) rotation pairs per thread: 16-B loads of both halves
  const int chunks = half / 8;
  for (int i = threadIdx.x; i < (hq + hkv) * chunks; i += blockDim.x) {
    const int h = i / chunks, j = (i % chunks) * 8;
    __nv_bfloat16* hp = row + h * D;
    const uint4 ua = *reinterpret_cast<const uint4*>(hp + j);
    const uint4 ub = *reinterpret_cast<const uint4*>(hp + j + half);
    const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&ua);
    const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&ub);
    uint4 uy1, uy2;
    __nv_bfloat162* y1 = reinterpret_cast<__nv_bfloat162*>(&uy1);
    __nv_bfloat162* y2 = reinterpret_cast<__nv_bfloat162*>(&uy2);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 a = __bfloat1622float2(a2[k]);
      const float2 b = __bfloat1622float2(b2[k]);
      const float2 r0 = rot[j + 2 * k], r1 = rot[j + 2 * k + 1];
      // explicit fma / mul (no contraction choice left to the compiler): the
      // K8 qkv epilogue (gemm_pf.cu) rotates with the same operations
      y1[k] = __floats2bfloat162_rn(__fmaf_rn(a.x, r0.x, -__fmul_rn(b.x, r0.y)),
                                    __fmaf_rn(a.y, r1.x, -__fmul_rn(b.y, r1.y)));
      y2[k] = __floats2bfloat162_rn(__fmaf_rn(b.x, r0.x, __fmul_rn(a.x, r0.y)),
                                    __fmaf_rn(b.y, r1.x, __fmul_rn(a.y, r1.y)));
    }
    __nv_bfloat16* dst = h < hq ? hp : kv_base + (static_cast<size_t>(h - hq) * 16 + off) * D;
    *reinterpret_cast<uint4*>(dst + j) = uy1;
    *reinterpret_cast<uint4*>(dst + j + half) = uy2;
  }
  // v rows: straight copy, 16 bytes per thread
  const __nv_bfloat16* v = row + (hq + hkv) * D;
  for (int i = threadIdx.x; i < hkv * D / 8; i += blockDim.x) {
    const int h = (i * 8) / D, d = (i * 8) % D;
    __nv_bfloat16* dst = kv_base + (static_cast<size_t>(hkv + h) * 16 + off) * D + d;
    *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(v + h * D + d);
  }
}

// Small per-iteration copies done by SMs through UVA-mapped pinned memory
// instead of the copy engines: the plan metadata H2D before a forward and
// the iteration descriptor + sampled-token keys D2H after it. On a copy
// engine they would queue behind the checkpoint / restore DMA chunks of the
// same direction (up to 256 MiB, ~5 ms) and stall the forward.
__global__ void sm_copy_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src, int64_t n16) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n16;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}

void sm_copy(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  const int64_t n16 = static_cast<int64_t>((bytes + 15) / 16);  // both buffers are 16-B padded
  if (n16 <= 0) return;
  const int blocks = static_cast<int>(std::min<int64_t>(64, (n16 + 255) / 256));
  sm_copy_kernel<<<blocks, 256, 0, s>>>(static_cast<uint4*>(dst), static_cast<const uint4*>(src), n16);
}

// desc (from the metadata) + E sampled-token keys -> the pinned host outputs
__global__ void out_copy_kernel(uint8_t* __restrict__ h_out, const IterDesc* __restrict__ desc,
                                const unsigned long long* __restrict__ keys, int E) {
  const int t = threadIdx.x;
  constexpr int kDescWords = static_cast<int>(sizeof(IterDesc) / 4);
  for (int i = t; i < kDescWords; i += blockDim.x)
    reinterpret_cast<uint32_t*>(h_out)[i] = reinterpret_cast<const uint32_t*>(desc)[i];
  unsigned long long* hk = reinterpret_cast<unsigned long long*>(h_out + sizeof(IterDesc));
  for (int i = t; i < E; i += blockDim.x) hk[i] = keys[i];
}

void out_copy(void* h_out, const IterDesc* desc, const void* keys, int E, cudaStream_t s) {
  out_copy_kernel<<<1, 256, 0, s>>>(static_cast<uint8_t*>(h_out), desc,
                                     static_cast<const unsigned long long*>(keys), E);
}

// (cos, sin) of every (token, frequency) of the iteration, [token][D/2]:
// positions are the same in every layer, so the K8 qkv epilogue reads this
// table instead of evaluating sincos per head. Same expressions as
// rope_append_kernel (bit-identical angles).
__global__ void rope_table_kernel(float2* tab, const int32_t* tok_pos, int D, float theta, const IterDesc* desc) {
  const int t = blockIdx.x;
  if (t >= desc->n_tok_all) return;
  const float pos = static_cast<float>(tok_pos[t]);
  for (int j = threadIdx.x; j < D / 2; j += blockDim.x) {
    const float inv_freq = powf(theta, -2.f * static_cast<float>(j) / static_cast<float>(D));
    float sn, cs;
    sincosf(pos * inv_freq, &sn, &cs);
    tab[static_cast<size_t>(t) * (D / 2) + j] = make_float2(cs, sn);
  }
}

void rope_table(float2* tab, const int32_t* tok_pos, int D, float theta, const IterDesc* desc, int grid,
                cudaStream_t s) {
  if (grid > 0) rope_table_kernel<<<grid, 64, 0, s>>>(tab, tok_pos, D, theta, desc);
}

void rope_append(__nv_bfloat16* qkv, const int32_t* tok_pos, const int32_t* tok_slot, __nv_bfloat16* pool, int hq,
                 int hkv, int D, int num_layers, int layer, float theta, const IterDesc* desc, int grid,
                 cudaStream_t s) {
  if (grid > 0)
    rope_append_kernel<<<grid, 128, 0, s>>>(qkv, tok_pos, tok_slot, pool, hq, hkv, D, num_layers, layer, theta, desc);
}

// ---------------------------------------------------------------- argmax ----
// Greedy sample: argmax over the vocab per sampled row, ties -> lowest id.
// 16 CTAs per row; each reduces its slice and folds (ordered value, ~id) into
// one 64-bit key per row with atomicMax. keys must be zeroed first; a row
// that stays 0 decodes to id -1 (rows >= n_ent_cur).
__device__ __forceinline__ unsigned long long argmax_key(float v, int i) {
  const uint32_t u = __float_as_uint(v);
  const uint32_t o = (u & 0x80000000u) ? ~u : (u | 0x80000000u);  // order-preserving
  return (static_cast<unsigned long long>(o) << 32) | (0xFFFFFFFFu - static_cast<uint32_t>(i));
}

__global__ void __launch_bounds__(256) argmax_kernel(const float* logits, int vocab, unsigned long long* keys,
                                                     const IterDesc* desc) {
  const int r = blockIdx.y;
  if (r >= desc->n_ent_cur) return;
  const float* row = logits + static_cast<size_t>(r) * vocab;
  const int chunk = (vocab + gridDim.x - 1) / gridDim.x;
  const int i0 = blockIdx.x * chunk, i1 = min(vocab, i0 + chunk);
  unsigned long long best = 0;
  if ((vocab & 3) == 0 && (chunk & 3) == 0) {
    // 16-byte loads, two in flight per thread (the logits are L2-resident:
    // the scan is load-latency bound, not bandwidth bound)
    const float4* row4 = reinterpret_cast<const float4*>(row);
    const int j0 = i0 >> 2, j1 = i1 >> 2;
    int j = j0 + threadIdx.x;
    for (; j + static_cast<int>(blockDim.x) < j1; j += 2 * blockDim.x) {
      const float4 a = row4[j], b = row4[j + blockDim.x];
      const float va[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int idx = (e < 4 ? j : j + static_cast<int>(blockDim.x)) * 4 + (e & 3);
        const unsigned long long k = argmax_key(va[e], idx);
        best = k > best ? k : best;
      }
    }
    for (; j < j1; j += blockDim.x) {
      const float4 a = row4[j];
      const float va[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const unsigned long long k = argmax_key(va[e], j * 4 + e);
        best = k > best ? k : best;
      }
    }
  } else {
    for (int i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
      const unsigned long long k = argmax_key(row[i], i);
      best = k > best ? k : best;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long k = __shfl_xor_sync(0xffffffffu, best, o);
    best = k > best ? k : best;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(&keys[r], best);
}

// keys[0, grid) must be zero (the final add_rmsnorm re-arms them) unless
// `zero` asks for a memset here
void argmax_rows(const float* logits, int vocab, unsigned long long* keys, const IterDesc* desc, int grid,
                 cudaStream_t s, bool zero) {
  if (grid <= 0) return;
  if (zero) cudaMemsetAsync(keys, 0, sizeof(unsigned long long) * grid, s);
  argmax_kernel<<<dim3(16, grid), 256, 0, s>>>(logits, vocab, keys, desc);
}

// ------------------------------------------------------- safepoint (K6) ----
// The check itself is fused into add_rmsnorm (safepoint_check above).

// TP: every rank votes 1.0 into an extra element of the next all-reduce when
// it sees the flag; after the sum every rank applies the same decision at the
// same layer, so row counts never diverge across ranks.
__global__ void safepoint_vote_kernel(__nv_bfloat16* tail, const IterDesc* desc, const PreemptMailbox* mb) {
  if (threadIdx.x >= 8) return;
  float v = 0.f;
  if (threadIdx.x == 0 && desc->dropped_at < 0 && mb->flag_epoch == desc->epoch &&
      desc->n_ent_on < desc->n_ent_cur)
    v = 1.f;
  tail[threadIdx.x] = __float2bfloat16(v);
}
void safepoint_vote(__nv_bfloat16* tail, const IterDesc* desc, const PreemptMailbox* mb, cudaStream_t s) {
  safepoint_vote_kernel<<<1, 32, 0, s>>>(tail, desc, mb);
}

// Clock calibration: spin until the host stores its CLOCK_MONOTONIC into the
// mailbox word, then record %globaltimer next to it.
__global__ void calib_clock_kernel(volatile uint64_t* mb) {
  // mb points at PreemptMailbox: [1] = flag_host_ns, [4] = seen_gpu_ns.
  // Bounded spin: under a profiler that serialises launches the host store
  // can only come after the kernel exits -- give up after 20 ms (writes 1).
  const uint64_t t0 = globaltimer_ns();
  while (mb[1] == 0) {
    if (globaltimer_ns() - t0 > 20000000ull) {
      mb[4] = 1;
      __threadfence_system();
      return;
    }
  }
  mb[4] = globaltimer_ns();
  __threadfence_system();
}
void calib_clock(volatile uint64_t* mb, cudaStream_t s) { calib_clock_kernel<<<1, 1, 0, s>>>(mb); }

__global__ void read_globaltimer_kernel(volatile uint64_t* out) {
  out[0] = globaltimer_ns();
  __threadfence_system();
}
void read_globaltimer(uint64_t* mapped_out, cudaStream_t s) {
  read_globaltimer_kernel<<<1, 1, 0, s>>>(mapped_out);
}

// -------------------------------------------- checkpoint / restore (K4/K5) --
// One work item = one (segment, layer, k|v, head) run of (t1 - t0) tokens x D
// elements, contiguous in both the device block and the host slot (same
// [L][2][Hkv][16][D] layout). Device<->host bytes move by plain 16-byte loads
// and stores through the mapped pinned host pool, so one launch does both the
// gather and the host-link transfer (measured: 92% of cudaMemcpyAsync peak at
// 256-byte runs, tools/hostlink_bench.cu).
struct SegDesc {
  int32_t block, slot, t0, t1;
};

// Host slot layout (pinned pool): TOKEN-major, [16 tokens][runs][D] with
// runs = L * 2 * H_kv(rank) -- a page's token range [t0, t1) is ONE
// contiguous run of (t1 - t0) * runs * D elements, so a delta of a page is a
// single copy-engine transfer. Device blocks stay run-major
// [runs][16 tokens][D] (16 consecutive rows per (layer, K|V, head) for TMA).

// Zero-copy variant (CS_KV_ZEROCOPY=1, A/B only): SM warps move 16-B vectors
// straight between the block and the mapped pinned slot.
template <bool kToHost>
__global__ void __launch_bounds__(256) kv_move_kernel(__nv_bfloat16* pool, __nv_bfloat16* host,
                                                      const SegDesc* segs, int n_segs, int runs_per_seg, int D) {
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const size_t block_elems = static_cast<size_t>(runs_per_seg) * 16 * D;
  const int vpt = D / 8;  // 16-B vectors per token row
  for (int64_t item = w; item < static_cast<int64_t>(n_segs) * runs_per_seg; item += warps) {
    const int s = static_cast<int>(item / runs_per_seg);
    const int run = static_cast<int>(item % runs_per_seg);
    const SegDesc sd = segs[s];
    uint4* dev = reinterpret_cast<uint4*>(pool + static_cast<size_t>(sd.block) * block_elems +
                                          static_cast<size_t>(run) * 16 * D + static_cast<size_t>(sd.t0) * D);
    uint4* hst = reinterpret_cast<uint4*>(host + static_cast<size_t>(sd.slot) * block_elems +
                                          (static_cast<size_t>(sd.t0) * runs_per_seg + run) * D);
    const int n = (sd.t1 - sd.t0) * vpt;
    for (int i = lane; i < n; i += 32) {
      const size_t h = static_cast<size_t>(i / vpt) * runs_per_seg * vpt + (i % vpt);
      if (kToHost) {
        hst[h] = __ldcs(dev + i);
      } else {
        dev[i] = hst[h];
      }
    }
  }
}

void kv_move(bool to_host, __nv_bfloat16* pool, __nv_bfloat16* host_mapped, const void* segs_mapped, int n_segs,
             int runs_per_seg, int D, int sms, cudaStream_t s) {
  if (n_segs <= 0) return;
  const int64_t items = static_cast<int64_t>(n_segs) * runs_per_seg;
  // host-link bound (~57 GB/s): a few CTAs per SM keep enough stores in
  // flight, more only take thread slots from the concurrent forward
  int64_t grid = (items + 7) / 8;
  if (grid > static_cast<int64_t>(sms) * 2) grid = static_cast<int64_t>(sms) * 2;
  if (grid < 1) grid = 1;
  const SegDesc* sd = static_cast<const SegDesc*>(segs_mapped);
  if (to_host) {
    kv_move_kernel<true><<<static_cast<int>(grid), 256, 0, s>>>(pool, host_mapped, sd, n_segs, runs_per_seg, D);
  } else {
    kv_move_kernel<false><<<static_cast<int>(grid), 256, 0, s>>>(pool, host_mapped, sd, n_segs, runs_per_seg, D);
  }
}

// K4 / K5 (default): HBM <-> HBM pack / unpack between the blocks and a
// device staging buffer laid out like the host slots (token-major), so the
// host-link leg is plain copy-engine DMA (one cudaMemcpyAsync per merged
// host run) and no SM
// sits on PCIe latency for the length of the transfer. Segment s occupies
// staging elements [stage[s], stage[s] + (t1 - t0) * runs * D).
// One warp per (segment, run): 16-B vectors, the block side contiguous, the
// staging side in 2*D-byte rows.
template <bool kToStage>
__global__ void __launch_bounds__(256) kv_pack_kernel(__nv_bfloat16* pool, __nv_bfloat16* stage,
                                                      const SegDesc* segs, const int64_t* stage_off, int n_segs,
                                                      int runs_per_seg, int D) {
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const size_t block_elems = static_cast<size_t>(runs_per_seg) * 16 * D;
  const int vpt = D / 8;
  for (int64_t item = w; item < static_cast<int64_t>(n_segs) * runs_per_seg; item += warps) {
    const int s = static_cast<int>(item / runs_per_seg);
    const int run = static_cast<int>(item % runs_per_seg);
    const SegDesc sd = segs[s];
    uint4* dev = reinterpret_cast<uint4*>(pool + static_cast<size_t>(sd.block) * block_elems +
                                          static_cast<size_t>(run) * 16 * D + static_cast<size_t>(sd.t0) * D);
    uint4* stg = reinterpret_cast<uint4*>(stage + stage_off[s] + static_cast<size_t>(run) * D);
    const int n = (sd.t1 - sd.t0) * vpt;
    for (int i = lane; i < n; i += 32) {
      const size_t h = static_cast<size_t>(i / vpt) * runs_per_seg * vpt + (i % vpt);
      if (kToStage) {
        stg[h] = __ldcs(dev + i);
      } else {
        dev[i] = __ldcs(stg + h);
      }
    }
  }
}

void kv_pack(bool to_stage, __nv_bfloat16* pool, __nv_bfloat16* stage, const void* segs, const int64_t* stage_off,
             int n_segs, int runs_per_seg, int D, int sms, cudaStream_t s) {
  if (n_segs <= 0) return;
  const int64_t items = static_cast<int64_t>(n_segs) * runs_per_seg;
  // HBM-bound and short (2 x bytes at ~6.5 TB/s): 8 warps per CTA, up to 4
  // CTAs per SM, each warp a (segment, run) of <= 16 rows
  int64_t grid = (items + 7) / 8;
  if (grid > static_cast<int64_t>(sms) * 4) grid = static_cast<int64_t>(sms) * 4;
  if (grid < 1) grid = 1;
  const SegDesc* sd = static_cast<const SegDesc*>(segs);
  if (to_stage) {
    kv_pack_kernel<true><<<static_cast<int>(grid), 256, 0, s>>>(pool, stage, sd, stage_off, n_segs, runs_per_seg, D);
  } else {
    kv_pack_kernel<false><<<static_cast<int>(grid), 256, 0, s>>>(pool, stage, sd, stage_off, n_segs, runs_per_seg, D);
  }
}

// --------------------------------------------------------------- debug ----
__global__ void fill_pool_kernel(__nv_bfloat16* pool, size_t n, uint64_t seed) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    pool[i] = __float2bfloat16(hash_uniform(seed, 7, i));
  }
}
void fill_pool(__nv_bfloat16* pool, size_t n, uint64_t seed, cudaStream_t s) {
  fill_pool_kernel<<<2048, 256, 0, s>>>(pool, n, seed);
}

}  // namespace csk

namespace csk {

// ------------------------------------------ peer-memory all-reduce (C-1) ----
// KV-head-group sharding: the o_proj / down-proj partial sums
// of the g ranks are added by one kernel that reads every rank's partial
// buffer directly (NVLink peer memory across GPUs; the same device in the
// loopback test) -- no NCCL launch, no staging copy. Ordering is device-side
// so a captured CUDA graph replays correctly:
//   * each rank keeps a step counter in its exchange region; every block
//     reads seq = step + 1;
//   * block 0 publishes flag[rank] = seq (release, system scope) -- the GEMM
//     that wrote this rank's partial precedes this kernel on the stream;
//   * every block waits (acquire, system scope) until all peers' flags reach
//     seq, sums its chunk of the g partials in fp32 and writes bf16;
//   * the last block to finish stores step = seq.
// Partials alternate between two buffers per rank (host-chosen, the same
// sequence on every rank), so a partial is never overwritten while a peer can
// still be reading it. A bounded spin (2 s) traps instead of hanging.
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void __launch_bounds__(256) p2p_allreduce_kernel(P2PArgs a, __nv_bfloat16* out, int64_t count) {
  __shared__ uint64_t s_seq;
  __shared__ int s_last;
  if (threadIdx.x == 0) s_seq = *reinterpret_cast<volatile uint64_t*>(a.step[a.rank]) + 1;
  __syncthreads();
  const uint64_t seq = s_seq;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    __threadfence_system();
    st_release_sys(a.flag[a.rank], seq);
  }
  if (threadIdx.x < a.g) {
    const uint64_t t0 = globaltimer_ns();
    while (ld_acquire_sys(a.flag[threadIdx.x]) < seq) {
      if (globaltimer_ns() - t0 > 2000000000ull) {
        printf("p2p_allreduce: rank %d timed out waiting for rank %d (seq %llu, its flag %llu, its step %llu)\n",
               a.rank, threadIdx.x, static_cast<unsigned long long>(seq),
               static_cast<unsigned long long>(ld_acquire_sys(a.flag[threadIdx.x])),
               static_cast<unsigned long long>(ld_acquire_sys(a.step[threadIdx.x])));
        __trap();
      }
    }
  }
  __syncthreads();
  const int64_t nv = count / 8;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nv;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int p = 0; p < a.g; ++p) {
      const uint4 v = __ldcv(reinterpret_cast<const uint4*>(a.part[p]) + i);
      const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&v);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += __bfloat162float(e[j]);
    }
    uint4 o;
    __nv_bfloat16* oe = reinterpret_cast<__nv_bfloat16*>(&o);
#pragma unroll
    for (int j = 0; j < 8; ++j) oe[j] = __float2bfloat16(acc[j]);
    reinterpret_cast<uint4*>(out)[i] = o;
  }
  if (blockIdx.x == 0) {  // tail (count % 8)
    for (int64_t i = nv * 8 + threadIdx.x; i < count; i += blockDim.x) {
      float acc = 0.f;
      for (int p = 0; p < a.g; ++p) acc += __bfloat162float(a.part[p][i]);
      out[i] = __float2bfloat16(acc);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(a.arrive, 1) == static_cast<int>(gridDim.x) - 1;
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    *a.arrive = 0;
    *reinterpret_cast<volatile uint64_t*>(a.step[a.rank]) = seq;
  }
}

// Two-shot variant for large payloads (reduce-scatter + all-gather over peer
// memory). Rank r owns vector chunk r of the buffer: after the same flag
// handshake it sums chunk r of the g partials in fp32 and writes the bf16 sum
// back IN PLACE into its own partial (peers read only their own chunks of it
// in this phase); the blocks then meet at a second, grid-wide barrier that
// publishes flag2[rank]; once every rank's flag2 reaches seq, every block
// copies chunk p of rank p's (now reduced) partial into out. Remote bytes per
// rank: 2 (g-1)/g x payload instead of (g-1) x payload for the one-shot
// kernel; the fp32 summation order (rank 0..g-1) is the same, so both kernels
// produce bit-identical sums. Requires all blocks co-resident (grid <= SMs x
// resident blocks), as the one-shot flag wait already does.
__device__ __forceinline__ void p2p_wait_all(const P2PArgs& a, uint64_t* const* flags, uint64_t seq,
                                             const char* what) {
  if (threadIdx.x < a.g) {
    const uint64_t t0 = globaltimer_ns();
    while (ld_acquire_sys(flags[threadIdx.x]) < seq) {
      if (globaltimer_ns() - t0 > 2000000000ull) {
        printf("p2p_allreduce2: rank %d timed out in %s waiting for rank %d (seq %llu)\n", a.rank, what,
               threadIdx.x, static_cast<unsigned long long>(seq));
        __trap();
      }
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256) p2p_allreduce2_kernel(P2PArgs a, __nv_bfloat16* out, int64_t count) {
  __shared__ uint64_t s_seq;
  __shared__ int s_last;
  if (threadIdx.x == 0) s_seq = *reinterpret_cast<volatile uint64_t*>(a.step[a.rank]) + 1;
  __syncthreads();
  const uint64_t seq = s_seq;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    __threadfence_system();
    st_release_sys(a.flag[a.rank], seq);
  }
  p2p_wait_all(a, a.flag, seq, "phase 0");
  const int64_t nv = count / 8;
  const int64_t per = (nv + a.g - 1) / a.g;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  // phase 1: reduce-scatter, own chunk in place
  {
    uint4* mine = reinterpret_cast<uint4*>(const_cast<__nv_bfloat16*>(a.part[a.rank]));
    const int64_t v1 = min(nv, (a.rank + 1) * per);
    for (int64_t i = a.rank * per + tid; i < v1; i += stride) {
      float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      for (int p = 0; p < a.g; ++p) {
        const uint4 v = __ldcv(reinterpret_cast<const uint4*>(a.part[p]) + i);
        const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&v);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] += __bfloat162float(e[j]);
      }
      uint4 o;
      __nv_bfloat16* oe = reinterpret_cast<__nv_bfloat16*>(&o);
#pragma unroll
      for (int j = 0; j < 8; ++j) oe[j] = __float2bfloat16(acc[j]);
      __stcg(mine + i, o);
    }
    if (a.rank == a.g - 1 && blockIdx.x == 0) {  // tail (count % 8) belongs to the last rank
      __nv_bfloat16* m = const_cast<__nv_bfloat16*>(a.part[a.rank]);
      for (int64_t i = nv * 8 + threadIdx.x; i < count; i += blockDim.x) {
        float acc = 0.f;
        for (int p = 0; p < a.g; ++p) acc += __bfloat162float(a.part[p][i]);
        m[i] = __float2bfloat16(acc);
      }
    }
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(a.arrive2, 1) == static_cast<int>(gridDim.x) - 1;
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    *a.arrive2 = 0;
    __threadfence_system();
    st_release_sys(a.flag2[a.rank], seq);
  }
  p2p_wait_all(a, a.flag2, seq, "phase 1");
  // phase 2: all-gather of the reduced chunks
  for (int64_t i = tid; i < nv; i += stride) {
    const int owner = static_cast<int>(i / per);
    reinterpret_cast<uint4*>(out)[i] = __ldcv(reinterpret_cast<const uint4*>(a.part[owner]) + i);
  }
  if (blockIdx.x == 0) {
    for (int64_t i = nv * 8 + threadIdx.x; i < count; i += blockDim.x) out[i] = a.part[a.g - 1][i];
  }
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(a.arrive, 1) == static_cast<int>(gridDim.x) - 1;
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    *a.arrive = 0;
    *reinterpret_cast<volatile uint64_t*>(a.step[a.rank]) = seq;
  }
}

void p2p_allreduce2(const P2PArgs& a, __nv_bfloat16* out, int64_t count, int blocks, cudaStream_t s) {
  p2p_allreduce2_kernel<<<blocks, 256, 0, s>>>(a, out, count);
}

void p2p_allreduce(const P2PArgs& a, __nv_bfloat16* out, int64_t count, int blocks, cudaStream_t s) {
  if (count <= 0) return;
  p2p_allreduce_kernel<<<blocks, 256, 0, s>>>(a, out, count);
}

}  // namespace csk
