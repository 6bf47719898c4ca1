// Decode-time pieces of the GPT caller (transformer.py:413-440
// restated for one new token per sequence against a key/value cache):
//   kv_append        : scatter the k / v columns of the fused QKV GEMM output
//                      into the per-sequence f32 cache at the device-side
//                      positions (graph-capturable: positions live on device)
//   decode_attention : softmax((q . K^T) * 1/sqrt(dh)) . V over the first
//                      lens[b] cached tokens, one CTA per (sequence, head)
// The reference recomputes the whole context every step (evaluate.py:96-98);
// with causal attention and token-wise activation scales the cached k / v rows
// are exactly the rows that recomputation would produce, so caching changes no
// value — only float attention (tolerance parity) runs here.
#include <cuda.h>
#include <cuda_fp16.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include "zq_gemm.cuh"

namespace zq {

// cache[b, pos[b] + t, c] = qkv[b*rows_per_seq + t, col0 + c] for the k and v blocks
__global__ void kv_append_kernel(const float* __restrict__ qkv, int64_t ld_qkv, int rows_per_seq,
                                 int dl, const int32_t* __restrict__ pos, float* __restrict__ kc,
                                 float* __restrict__ vc, int64_t max_ctx, int64_t total4) {
  const int d4 = dl >> 2;
  pdl_trigger();
  pdl_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c4 = (int)(i % d4);
    const int64_t r = i / d4;  // token row of qkv
    const int b = (int)(r / rows_per_seq), t = (int)(r % rows_per_seq);
    const int64_t slot = ((int64_t)b * max_ctx + pos[b] + t) * dl + 4 * c4;
    const float* src = qkv + r * ld_qkv + 4 * c4;
    *reinterpret_cast<float4*>(kc + slot) = __ldg(reinterpret_cast<const float4*>(src + dl));
    *reinterpret_cast<float4*>(vc + slot) = __ldg(reinterpret_cast<const float4*>(src + 2 * dl));
  }
}

// Flash-decoding: a cluster of C CTAs per (sequence, head); CTA c takes the
// keys [c*chunk, (c+1)*chunk) below lens[b].  Inside a CTA every warp runs its
// own online softmax over keys c*chunk + warp, + 4, ... (four keys per step: the
// K and V rows of all four are loaded before any is used, so each warp keeps
// 8-16 KB of the cache in flight and K and V stream together), q stays in
// registers, scores are dot products reduced across the warp.  The four warp
// partials (m, l, o) are merged in shared memory, then each CTA combines dims
// [c*dh/C, (c+1)*dh/C) of the C partials through distributed shared memory:
//   o = sum_c o_c 2^(m_c - M) / sum_c l_c 2^(m_c - M)   (scores in log2 units).

__device__ __forceinline__ uint32_t dsm_map(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ float dsm_ld_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t cta_rank_in_cluster() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ float ex2f(float v) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}

// THREADS per CTA; LPK lanes per key, NF float4 chunks of the head per lane
// (LPK < 32: a warp runs 32 / LPK independent "virtual warps", so no lane idles:
// head_dim 64 -> 16 x 1, 96 -> 8 x 3, 128 -> 32 x 1, 256 -> 32 x 2); U keys per
// virtual-warp step have their K / V rows in flight together
template <int THREADS, int LPK, int NF, int U>
__global__ void __launch_bounds__(THREADS) decode_attention_kernel(
    const float* __restrict__ q, int64_t ld_q, const float* __restrict__ kc,
    const float* __restrict__ vc, int64_t max_ctx, int heads, int dh,
    const int32_t* __restrict__ lens, float scale, float* __restrict__ ctx, int64_t ld_ctx,
    int C, int chunk) {
  constexpr int NVW = (THREADS / 32) * (32 / LPK);  // virtual warps
  __shared__ __align__(16) float po[NVW][256];      // partial outputs; row 0 = o_c
  __shared__ float wst[NVW][2];
  __shared__ float stat[2];  // m_c, l_c (log2 units)
  pdl_trigger();
  pdl_wait();
  const int c = (int)cta_rank_in_cluster();
  const int bh = blockIdx.x / C;
  const int b = bh / heads, h = bh % heads;
  const int tid = threadIdx.x, lane = tid & 31;
  const int vw = tid / LPK, sl = tid % LPK;
  const int dl = heads * dh, d4 = dh >> 2;
  const int len = lens[b];
  const int j0 = c * chunk, j1 = min(len, j0 + chunk);
  const float* kb = kc + (int64_t)b * max_ctx * dl + h * dh;
  const float* vb = vc + (int64_t)b * max_ctx * dl + h * dh;
  const float sl2 = __fmul_rn(scale, 1.4426950408889634f);
  const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
  const float4* qr = reinterpret_cast<const float4*>(q + (int64_t)b * ld_q + h * dh);
  float4 qv[NF], o[NF];
  bool fo[NF];
#pragma unroll
  for (int i = 0; i < NF; ++i) {
    fo[i] = sl + LPK * i < d4;
    qv[i] = fo[i] ? __ldg(qr + sl + LPK * i) : z4;
    o[i] = z4;
  }
  float m = -INFINITY, l = 0.0f;
  // every virtual warp of a hardware warp runs the same trip count (shuffles)
  const int wbase = j0 + (vw - (lane / LPK));
  for (int jw = wbase; jw < j1; jw += U * NVW) {
    const int jj = jw + lane / LPK;
    float4 kk[U][NF], vv[U][NF];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = jj + u * NVW;
      const bool ok = j < j1;
      const float4* kr = reinterpret_cast<const float4*>(kb + (int64_t)j * dl);
      const float4* vr = reinterpret_cast<const float4*>(vb + (int64_t)j * dl);
#pragma unroll
      for (int i = 0; i < NF; ++i) {
        kk[u][i] = ok && fo[i] ? __ldg(kr + sl + LPK * i) : z4;
        vv[u][i] = ok && fo[i] ? __ldg(vr + sl + LPK * i) : z4;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float d = 0.0f;
#pragma unroll
      for (int i = 0; i < NF; ++i) {
        d = __fmaf_rn(qv[i].x, kk[u][i].x, d);
        d = __fmaf_rn(qv[i].y, kk[u][i].y, d);
        d = __fmaf_rn(qv[i].z, kk[u][i].z, d);
        d = __fmaf_rn(qv[i].w, kk[u][i].w, d);
      }
#pragma unroll
      for (int off = LPK / 2; off > 0; off >>= 1) d = __fadd_rn(d, __shfl_xor_sync(0xffffffffu, d, off));
      if (jj + u * NVW < j1) {
        const float sv = __fmul_rn(d, sl2);
        const float mn = fmaxf(m, sv);
        const float corr = ex2f(__fsub_rn(m, mn));  // m = -inf -> 0
        const float pj = ex2f(__fsub_rn(sv, mn));
        l = __fmaf_rn(l, corr, pj);
#pragma unroll
        for (int i = 0; i < NF; ++i) {
          o[i].x = __fmaf_rn(pj, vv[u][i].x, __fmul_rn(o[i].x, corr));
          o[i].y = __fmaf_rn(pj, vv[u][i].y, __fmul_rn(o[i].y, corr));
          o[i].z = __fmaf_rn(pj, vv[u][i].z, __fmul_rn(o[i].z, corr));
          o[i].w = __fmaf_rn(pj, vv[u][i].w, __fmul_rn(o[i].w, corr));
        }
        m = mn;
      }
    }
  }
#pragma unroll
  for (int i = 0; i < NF; ++i)
    if (fo[i]) *reinterpret_cast<float4*>(&po[vw][4 * (sl + LPK * i)]) = o[i];
  if (sl == 0) wst[vw][0] = m, wst[vw][1] = l;
  __syncthreads();
  // merge the virtual-warp partials: M = max m_w, L = sum l_w 2^(m_w - M), o_c = sum o_w 2^(m_w - M)
  float M = -INFINITY;
#pragma unroll
  for (int w = 0; w < NVW; ++w) M = fmaxf(M, wst[w][0]);
  float fw[NVW];
  float L = 0.0f;
#pragma unroll
  for (int w = 0; w < NVW; ++w) {
    fw[w] = wst[w][0] == -INFINITY ? 0.0f : ex2f(__fsub_rn(wst[w][0], M));
    L = __fmaf_rn(wst[w][1], fw[w], L);
  }
  __syncthreads();
  for (int i = tid; i < dh; i += THREADS) {
    float t = 0.0f;
#pragma unroll
    for (int w = 0; w < NVW; ++w) t = __fmaf_rn(po[w][i], fw[w], t);
    po[0][i] = t;
  }
  if (tid == 0) stat[0] = M, stat[1] = L;  // M = -inf for an empty chunk
  cluster_barrier();
  // combine dims [c*dh/C, (c+1)*dh/C) across the cluster
  const int da = (c * dh) / C, db = ((c + 1) * dh) / C;
  const uint32_t stat_a = smem_u32(stat), po_a = smem_u32(&po[0][0]);
  float MM = -INFINITY;
  for (int r = 0; r < C; ++r) MM = fmaxf(MM, dsm_ld_f32(dsm_map(stat_a, r)));
  float LL = 0.0f;
  for (int r = 0; r < C; ++r) {
    const float mr = dsm_ld_f32(dsm_map(stat_a, r));
    if (mr != -INFINITY) LL += dsm_ld_f32(dsm_map(stat_a + 4, r)) * ex2f(mr - MM);
  }
  for (int i = da + tid; i < db; i += THREADS) {
    float t = 0.0f;
    for (int r = 0; r < C; ++r) {
      const float mr = dsm_ld_f32(dsm_map(stat_a, r));
      if (mr != -INFINITY) t += dsm_ld_f32(dsm_map(po_a + 4 * i, r)) * ex2f(mr - MM);
    }
    ctx[(int64_t)b * ld_ctx + h * dh + i] = t / LL;
  }
  cluster_barrier();  // keep this CTA's partial alive until every peer has read it
}

// TMA-pipelined variant (the default for head_dim 64 / 96 / 128 / 256): the same
// cluster-of-C flash-decoding split and merge, but the K and V rows of each
// CTA's key range stream into a 4-stage shared-memory ring through TMA (one
// [KT keys x dh] box of each per stage, ~16 KB), so every SM keeps ~200 KB of
// the cache in flight instead of the ~30 KB of register loads above, which left
// long contexts (GPT-3 350M: 1030 keys, 67.5 MB per layer) at ~40% of HBM.
// Warp 4 is the producer; warps 0-3 run the per-virtual-warp online softmax out
// of shared memory (a key's row is read by LPK consecutive lanes, conflict-free).
// The key range of a CTA is split from the runtime length lens[b] (not max_ctx),
// so short contexts keep every CTA busy.
template <int DH, int KT, int LPK, int NF, int STG_ = 4>
struct DecTmaCfg {
  static constexpr int STG = STG_;
  static constexpr int TILE = KT * DH * 4;            // one K (or V) box
  static constexpr int SMEM = STG * 2 * TILE + 2 * STG * 8;
  static constexpr int NVW = 4 * (32 / LPK);          // virtual warps (4 compute warps)
  static constexpr int KPV = KT / NVW;                // keys per virtual warp per tile
  static_assert(KT % NVW == 0, "tile must split evenly over the virtual warps");
};

template <int DH, int KT, int LPK, int NF, int STG_>
__global__ void __launch_bounds__(160) decode_attention_tma_kernel(
    const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
    const float* __restrict__ q, int64_t ld_q, int64_t max_ctx, int heads,
    const int32_t* __restrict__ lens, float scale, float* __restrict__ ctx, int64_t ld_ctx, int C) {
  using Cfg = DecTmaCfg<DH, KT, LPK, NF, STG_>;
  constexpr int NVW = Cfg::NVW, STG = Cfg::STG;
  extern __shared__ __align__(128) uint8_t dsm[];
  float* sK = reinterpret_cast<float*>(dsm);
  float* sV = sK + STG * KT * DH;
  uint64_t* full = reinterpret_cast<uint64_t*>(dsm + STG * 2 * Cfg::TILE);
  uint64_t* empty = full + STG;
  __shared__ __align__(16) float po[NVW][DH];
  __shared__ float wst[NVW][2];
  __shared__ float stat[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    prefetch_tmap(&tmK);
    prefetch_tmap(&tmV);
    for (int s = 0; s < STG; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);
    }
    fence_barrier_init();
  }
  __syncthreads();
  pdl_trigger();
  const int c = (int)cta_rank_in_cluster();
  const int bh = blockIdx.x / C;
  const int b = bh / heads, h = bh % heads;
  // lens is written at the start of the step by a non-PDL kernel, so it is
  // complete before any kernel of the step starts; the cache rows below len - 1
  // were appended by earlier steps.  Only row len - 1 (this step's k / v, written
  // by the QKV GEMM that precedes this kernel) and q need the grid dependency:
  // the producer streams the first tiles that end before that row while the
  // QKV GEMM drains, then waits.
  const int len = lens[b];
  const int per = (((len + C - 1) / C) + KT - 1) / KT * KT;  // keys per CTA, whole tiles
  const int j0 = c * per, j1 = min(len, j0 + per);
  const int ntiles = j1 > j0 ? (j1 - j0 + KT - 1) / KT : 0;
  float m = -INFINITY, l = 0.0f;
  const int vw = tid / LPK, sl = tid % LPK;
  float4 o[NF];
  if (warp == 4) {
    if (lane == 0) {
      const int row0 = (int)((int64_t)b * max_ctx) + j0;
      int t = 0;
      for (; t < ntiles && t < STG && j0 + (t + 1) * KT <= len - 1; ++t) {
        mbar_arrive_expect_tx(&full[t], 2 * Cfg::TILE);
        tma_load_2d(sK + t * KT * DH, &tmK, &full[t], h * DH, row0 + t * KT);
        tma_load_2d(sV + t * KT * DH, &tmV, &full[t], h * DH, row0 + t * KT);
      }
      pdl_wait();
      for (; t < ntiles; ++t) {
        const int s = t % STG;
        if (t >= STG) mbar_wait(&empty[s], ((t / STG) - 1) & 1);
        mbar_arrive_expect_tx(&full[s], 2 * Cfg::TILE);
        tma_load_2d(sK + s * KT * DH, &tmK, &full[s], h * DH, row0 + t * KT);
        tma_load_2d(sV + s * KT * DH, &tmV, &full[s], h * DH, row0 + t * KT);
      }
    }
    pdl_wait();
  } else {
    pdl_wait();
    const float sl2 = __fmul_rn(scale, 1.4426950408889634f);
    const float4* qr = reinterpret_cast<const float4*>(q + (int64_t)b * ld_q + h * DH);
    float4 qv[NF];
#pragma unroll
    for (int i = 0; i < NF; ++i) {
      qv[i] = __ldg(qr + sl + LPK * i);
      o[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (int t = 0; t < ntiles; ++t) {
      const int s = t % STG;
      mbar_wait(&full[s], (t / STG) & 1);
      const float* kt = sK + s * KT * DH;
      const float* vt = sV + s * KT * DH;
      float4 kk[Cfg::KPV][NF], vv[Cfg::KPV][NF];
#pragma unroll
      for (int u = 0; u < Cfg::KPV; ++u) {
        const int r = vw + u * NVW;
#pragma unroll
        for (int i = 0; i < NF; ++i) {
          kk[u][i] = *reinterpret_cast<const float4*>(kt + r * DH + 4 * (sl + LPK * i));
          vv[u][i] = *reinterpret_cast<const float4*>(vt + r * DH + 4 * (sl + LPK * i));
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);  // the tile is in registers: the slot may refill
#pragma unroll
      for (int u = 0; u < Cfg::KPV; ++u) {
        float d = 0.0f;
#pragma unroll
        for (int i = 0; i < NF; ++i) {
          d = __fmaf_rn(qv[i].x, kk[u][i].x, d);
          d = __fmaf_rn(qv[i].y, kk[u][i].y, d);
          d = __fmaf_rn(qv[i].z, kk[u][i].z, d);
          d = __fmaf_rn(qv[i].w, kk[u][i].w, d);
        }
#pragma unroll
        for (int off = LPK / 2; off > 0; off >>= 1) d = __fadd_rn(d, __shfl_xor_sync(0xffffffffu, d, off));
        if (j0 + t * KT + vw + u * NVW < j1) {  // keys past len are never touched (the cache there is garbage)
          const float sv = __fmul_rn(d, sl2);
          const float mn = fmaxf(m, sv);
          const float corr = ex2f(__fsub_rn(m, mn));
          const float pj = ex2f(__fsub_rn(sv, mn));
          l = __fmaf_rn(l, corr, pj);
#pragma unroll
          for (int i = 0; i < NF; ++i) {
            o[i].x = __fmaf_rn(pj, vv[u][i].x, __fmul_rn(o[i].x, corr));
            o[i].y = __fmaf_rn(pj, vv[u][i].y, __fmul_rn(o[i].y, corr));
            o[i].z = __fmaf_rn(pj, vv[u][i].z, __fmul_rn(o[i].z, corr));
            o[i].w = __fmaf_rn(pj, vv[u][i].w, __fmul_rn(o[i].w, corr));
          }
          m = mn;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < NF; ++i) *reinterpret_cast<float4*>(&po[vw][4 * (sl + LPK * i)]) = o[i];
    if (sl == 0) wst[vw][0] = m, wst[vw][1] = l;
  }
  __syncthreads();
  float M = -INFINITY;
#pragma unroll
  for (int w = 0; w < NVW; ++w) M = fmaxf(M, wst[w][0]);
  float fw[NVW];
  float L = 0.0f;
#pragma unroll
  for (int w = 0; w < NVW; ++w) {
    fw[w] = wst[w][0] == -INFINITY ? 0.0f : ex2f(__fsub_rn(wst[w][0], M));
    L = __fmaf_rn(wst[w][1], fw[w], L);
  }
  __syncthreads();
  for (int i = tid; i < DH; i += 160) {
    float t = 0.0f;
#pragma unroll
    for (int w = 0; w < NVW; ++w) t = __fmaf_rn(po[w][i], fw[w], t);
    po[0][i] = t;
  }
  if (tid == 0) stat[0] = M, stat[1] = L;
  cluster_barrier();
  const int da = (c * DH) / C, db = ((c + 1) * DH) / C;
  const uint32_t stat_a = smem_u32(stat), po_a = smem_u32(&po[0][0]);
  float MM = -INFINITY;
  for (int r = 0; r < C; ++r) MM = fmaxf(MM, dsm_ld_f32(dsm_map(stat_a, r)));
  float LL = 0.0f;
  for (int r = 0; r < C; ++r) {
    const float mr = dsm_ld_f32(dsm_map(stat_a, r));
    if (mr != -INFINITY) LL += dsm_ld_f32(dsm_map(stat_a + 4, r)) * ex2f(mr - MM);
  }
  for (int i = da + tid; i < db; i += 160) {
    float t = 0.0f;
    for (int r = 0; r < C; ++r) {
      const float mr = dsm_ld_f32(dsm_map(stat_a, r));
      if (mr != -INFINITY) t += dsm_ld_f32(dsm_map(po_a + 4 * i, r)) * ex2f(mr - MM);
    }
    ctx[(int64_t)b * ld_ctx + h * DH + i] = t / LL;
  }
  cluster_barrier();
}

// ---------------------------------------------------------------------------
// Tied LM head + greedy argmax for a decode step (evaluate.py's logits =
// LN(x_last) @ E^T, argmax per sequence; float, tolerance parity):
//   prep   : per token, x -> power-of-two scale (max in [2^14, 2^15)) and f16
//            hi / lo rows (two-term split, 22 significant bits); keys zeroed
//   main   : persistent CTAs walk 128-row vocabulary tiles; a TMA warp streams
//            the f32 embedding tile by 64-column k-blocks, 4 converter warps
//            scale (one global power of two) and split it into f16 hi / lo
//            SWIZZLE_128B tiles, one warp issues tcgen05 kind::f16 MMAs
//            (E_hi x_hi + E_hi x_lo + E_lo x_hi; M = 128 vocab rows, N = 16
//            tokens) into a double-buffered TMEM accumulator; the converter
//            warps then read the 128 x 16 logits and fold them into a per-token
//            64-bit atomic max of (ordered logit bits, ~index): largest logit,
//            lowest index on ties — numpy's argmax rule
//   final  : keys -> int64 token ids
// The embedding streams from HBM once per step at up to the copy rate; the split
// costs ~4 FP32 ops per weight element on otherwise idle CUDA cores.
// ---------------------------------------------------------------------------
constexpr int kLmRows = 128, kLmK = 64, kLmS = 6, kLmTok = 16;
constexpr int kLmE = kLmRows * kLmK * 4;          // 32 KB: two [128 x 32] f32 boxes, converted in place
constexpr int kLmX = kLmTok * kLmK * 2;           // 2 KB f16 token tile
constexpr int kLmStage = kLmE + 2 * kLmX;         // 36 KB
constexpr int kLmSmem = kLmS * kLmStage + 256;

__device__ __forceinline__ float lm_pow2_scale(uint32_t max_bits) {  // max * f in [2^14, 2^15)
  const int E = (int)((max_bits >> 23) & 0xFF);
  int F = 268 - E;
  F = F < 1 ? 1 : (F > 254 ? 254 : F);
  return __uint_as_float((uint32_t)F << 23);
}
__device__ __forceinline__ void lm_split(float a, float b, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(a, b);
  const float2 hf = __half22float2(h);
  const __half2 l = __floats2half2_rn(__fsub_rn(a, hf.x), __fsub_rn(b, hf.y));
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}

__global__ void __launch_bounds__(256) lm_prep_kernel(const float* __restrict__ x, int64_t ld_x, int ntok, int dim,
                                                      __half* __restrict__ xh, __half* __restrict__ xl,
                                                      float* __restrict__ xinv,
                                                      unsigned long long* __restrict__ keys) {
  __shared__ uint32_t red[32];
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.x;
  const bool act = t < ntok;
  const float* xr = x + (int64_t)t * ld_x;
  uint32_t mb = 0;
  if (act)
    for (int i = threadIdx.x; i < dim; i += 256) mb = max(mb, __float_as_uint(xr[i]) & 0x7fffffffu);
  const float f = lm_pow2_scale(__float_as_uint(block_max_nonneg(__uint_as_float(mb), red)));
  for (int i = 2 * threadIdx.x; i < dim; i += 512) {
    uint32_t hi = 0, lo = 0;
    if (act) lm_split(__fmul_rn(xr[i], f), __fmul_rn(xr[i + 1], f), hi, lo);
    *reinterpret_cast<uint32_t*>(xh + (int64_t)t * dim + i) = hi;
    *reinterpret_cast<uint32_t*>(xl + (int64_t)t * dim + i) = lo;
  }
  if (threadIdx.x == 0) {
    xinv[t] = __uint_as_float((uint32_t)(254 - (int)(__float_as_uint(f) >> 23)) << 23);
    keys[t] = 0ull;
  }
}

__device__ __forceinline__ void mma_f16_ss(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

__global__ void __launch_bounds__(192, 1)
    lm_head_kernel(const __grid_constant__ CUtensorMap tmE, const __half* __restrict__ xh,
                   const __half* __restrict__ xl, const float* __restrict__ xinv, int ntok, int64_t vocab,
                   int dim, float fe, float inv_fe, unsigned long long* __restrict__ keys) {
  // Each stage: the two f32 boxes of a [128 x 64] embedding k-block, which the
  // converter thread of row r rewrites in place (row r only): box 0 row r <- the
  // 64 f16 hi values, box 1 row r <- the 64 f16 lo values, i.e. two K-major
  // SWIZZLE_128B f16 tiles; plus the tokens' f16 hi / lo k-block.
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kLmS * kLmStage);
  uint64_t* e_full = bars;             // [S] TMA bytes landed
  uint64_t* c_full = bars + kLmS;      // [S] converted (4 warps)
  uint64_t* s_empty = bars + 2 * kLmS; // [S] MMAs done with the stage
  uint64_t* t_full = bars + 3 * kLmS;  // [2]
  uint64_t* t_empty = t_full + 2;      // [2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(t_empty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = (int)((vocab + kLmRows - 1) / kLmRows);
  const int nkb = dim / kLmK;
  if (threadIdx.x == 0) {
    if (smem_u32(smem) & 1023) __trap();
    prefetch_tmap(&tmE);
    for (int i = 0; i < kLmS; ++i) mbar_init(&e_full[i], 1), mbar_init(&c_full[i], 4), mbar_init(&s_empty[i], 1);
    for (int i = 0; i < 2; ++i) mbar_init(&t_full[i], 1), mbar_init(&t_empty[i], 4);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tslot, 32);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  pdl_trigger();
  if (warp == 0) {
    // ---- TMA producer (the embedding does not depend on the previous kernel) ----
    int st = 0, ph = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&s_empty[st], ph ^ 1);
        if (lane == 0) {
          mbar_arrive_expect_tx(&e_full[st], kLmE);
          tma_load_2d(smem + st * kLmStage, &tmE, &e_full[st], kb * kLmK, tile * kLmRows);
          tma_load_2d(smem + st * kLmStage + kLmE / 2, &tmE, &e_full[st], kb * kLmK + 32, tile * kLmRows);
        }
        __syncwarp();
        if (++st == kLmS) st = 0, ph ^= 1;
      }
  } else if (warp == 1) {
    // ---- MMA issuer ----
    pdl_wait();
    const uint32_t idesc = (1u << 4) | ((uint32_t)(kLmTok >> 3) << 17) | ((uint32_t)(kLmRows >> 4) << 24);
    int st = 0, ph = 0, acc = 0, aph = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      mbar_wait(&t_empty[acc], aph ^ 1);
      tc_fence_after();
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&c_full[st], ph);
        tc_fence_after();
        if (lane == 0) {
          uint8_t* o = smem + st * kLmStage;
          const uint64_t dEh = make_sw128_desc(smem_u32(o)), dEl = make_sw128_desc(smem_u32(o + kLmE / 2));
          const uint64_t dXh = make_sw128_desc(smem_u32(o + kLmE));
          const uint64_t dXl = make_sw128_desc(smem_u32(o + kLmE + kLmX));
#pragma unroll
          for (int t3 = 0; t3 < 3; ++t3)
#pragma unroll
            for (int ks = 0; ks < kLmK / 16; ++ks)
              mma_f16_ss(tmem + acc * 16, (t3 == 2 ? dEl : dEh) + 2 * ks, (t3 == 1 ? dXl : dXh) + 2 * ks, idesc,
                         (kb | ks | t3) != 0);
          mma_commit(&s_empty[st]);
        }
        __syncwarp();
        if (++st == kLmS) st = 0, ph ^= 1;
      }
      if (lane == 0) mma_commit(&t_full[acc]);
      __syncwarp();
      if (++acc == 2) acc = 0, aph ^= 1;
    }
  } else {
    // ---- converters (row r = thread - 64) and epilogue ----
    pdl_wait();
    const int r = threadIdx.x - 64, quarter = warp & 3;
    int st = 0, ph = 0, acc = 0, aph = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&e_full[st], ph);
        uint8_t* o = smem + st * kLmStage;
        uint32_t hi[32], lo[32];
#pragma unroll
        for (int c = 0; c < 16; ++c) {  // 16 float4 chunks: box c / 8, chunk c % 8 (row r only)
          const float4 v = *reinterpret_cast<const float4*>(o + (c >> 3) * (kLmE / 2) + r * 128 +
                                                             (((c & 7) ^ (r & 7)) << 4));
          lm_split(__fmul_rn(v.x, fe), __fmul_rn(v.y, fe), hi[2 * c], lo[2 * c]);
          lm_split(__fmul_rn(v.z, fe), __fmul_rn(v.w, fe), hi[2 * c + 1], lo[2 * c + 1]);
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) {  // row r of box 0 <- hi, of box 1 <- lo (128 B each)
          const uint32_t off = r * 128 + ((c ^ (r & 7)) << 4);
          *reinterpret_cast<uint4*>(o + off) = make_uint4(hi[4 * c], hi[4 * c + 1], hi[4 * c + 2], hi[4 * c + 3]);
          *reinterpret_cast<uint4*>(o + kLmE / 2 + off) =
              make_uint4(lo[4 * c], lo[4 * c + 1], lo[4 * c + 2], lo[4 * c + 3]);
        }
        {  // the tokens' f16 k-block: 16 rows x 8 chunks = 128 threads x 16 B each
          const int xr = r >> 3, c = r & 7;
          const uint32_t off = xr * 128 + ((c ^ (xr & 7)) << 4);
          const int64_t src = (int64_t)xr * dim + kb * kLmK + 8 * c;
          *reinterpret_cast<uint4*>(o + kLmE + off) = *reinterpret_cast<const uint4*>(xh + src);
          *reinterpret_cast<uint4*>(o + kLmE + kLmX + off) = *reinterpret_cast<const uint4*>(xl + src);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&c_full[st]);
        if (++st == kLmS) st = 0, ph ^= 1;
      }
      // ---- epilogue: 16 logits per vocabulary row -> per-token (max, lowest index) ----
      mbar_wait(&t_full[acc], aph);
      tc_fence_after();
      uint32_t lg[16];
      tmem_ld16(tmem + ((uint32_t)(quarter * 32) << 16) + acc * 16, lg);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&t_empty[acc]);
      if (++acc == 2) acc = 0, aph ^= 1;
      const int64_t v = (int64_t)tile * kLmRows + quarter * 32 + lane;
#pragma unroll
      for (int t = 0; t < kLmTok; ++t) {
        if (t >= ntok) break;
        const float val = __fmul_rn(__fmul_rn(__uint_as_float(lg[t]), inv_fe), xinv[t]);
        uint32_t u = __float_as_uint(val);
        u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
        unsigned long long key = v < vocab ? (((unsigned long long)u << 32) | (0xFFFFFFFFull - (uint64_t)v)) : 0ull;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          const unsigned long long o2 = __shfl_xor_sync(0xffffffffu, key, off);
          key = o2 > key ? o2 : key;
        }
        if (lane == 0 && key) atomicMax(keys + t, key);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 32);
}

// Pre-split variant: the embedding's f16 hi / lo terms (scaled by the same
// global power of two) are computed once (zq_lm_embed_split) and streamed by
// TMA straight into SWIZZLE_128B tiles, so no CUDA-core conversion sits between
// HBM and the tensor core (4 B per weight element either way).  The tokens'
// f16 hi / lo k-blocks are TMA-loaded too (after the grid dependency: the prep
// kernel writes them); the first stages' embedding tiles go out before it.
// Warps: 0 TMA, 1 MMA, 2-5 epilogue (TMEM logits -> per-token argmax keys).
constexpr int kLs16 = kLmRows * kLmK * 2;   // one f16 embedding term tile: 16 KB
constexpr int kLsStage = 2 * kLs16 + 2 * kLmX;
constexpr int kLsS = 6;
constexpr int kLsSmem = kLsS * kLsStage + 256;

__global__ void __launch_bounds__(192, 1)
    lm_head_split_kernel(const __grid_constant__ CUtensorMap tmEh, const __grid_constant__ CUtensorMap tmEl,
                         const __grid_constant__ CUtensorMap tmXh, const __grid_constant__ CUtensorMap tmXl,
                         const float* __restrict__ xinv, int ntok, int64_t vocab, int dim, float inv_fe,
                         unsigned long long* __restrict__ keys) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kLsS * kLsStage);
  uint64_t* full = bars;               // [S] all four tiles landed
  uint64_t* s_empty = bars + kLsS;     // [S]
  uint64_t* t_full = bars + 2 * kLsS;  // [2]
  uint64_t* t_empty = t_full + 2;      // [2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(t_empty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = (int)((vocab + kLmRows - 1) / kLmRows);
  const int nkb = dim / kLmK;
  if (threadIdx.x == 0) {
    if (smem_u32(smem) & 1023) __trap();
    prefetch_tmap(&tmEh);
    prefetch_tmap(&tmEl);
    for (int i = 0; i < kLsS; ++i) mbar_init(&full[i], 1), mbar_init(&s_empty[i], 1);
    for (int i = 0; i < 2; ++i) mbar_init(&t_full[i], 1), mbar_init(&t_empty[i], 4);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tslot, 32);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  pdl_trigger();
  if (warp == 0) {
    if (lane == 0) {
      // embedding tiles of the first stages before the dependency, token tiles after
      const int total = ((ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x) * nkb;
      const int pre = total < kLsS ? total : kLsS;
      for (int i = 0; i < pre; ++i) {
        const int tile = blockIdx.x + (i / nkb) * gridDim.x, kb = i % nkb;
        uint8_t* o = smem + i * kLsStage;
        mbar_arrive_expect_tx(&full[i], kLsStage);
        tma_load_2d(o, &tmEh, &full[i], kb * kLmK, tile * kLmRows);
        tma_load_2d(o + kLs16, &tmEl, &full[i], kb * kLmK, tile * kLmRows);
      }
      pdl_wait();
      for (int i = 0; i < pre; ++i) {
        const int kb = i % nkb;
        uint8_t* o = smem + i * kLsStage;
        tma_load_2d(o + 2 * kLs16, &tmXh, &full[i], kb * kLmK, 0);
        tma_load_2d(o + 2 * kLs16 + kLmX, &tmXl, &full[i], kb * kLmK, 0);
      }
      int st = pre % kLsS, ph = pre / kLsS;
      for (int i = pre; i < total; ++i) {
        const int tile = blockIdx.x + (i / nkb) * gridDim.x, kb = i % nkb;
        mbar_wait(&s_empty[st], ph ^ 1);
        uint8_t* o = smem + st * kLsStage;
        mbar_arrive_expect_tx(&full[st], kLsStage);
        tma_load_2d(o, &tmEh, &full[st], kb * kLmK, tile * kLmRows);
        tma_load_2d(o + kLs16, &tmEl, &full[st], kb * kLmK, tile * kLmRows);
        tma_load_2d(o + 2 * kLs16, &tmXh, &full[st], kb * kLmK, 0);
        tma_load_2d(o + 2 * kLs16 + kLmX, &tmXl, &full[st], kb * kLmK, 0);
        if (++st == kLsS) st = 0, ph ^= 1;
      }
    }
    pdl_wait();
  } else if (warp == 1) {
    pdl_wait();
    const uint32_t idesc = (1u << 4) | ((uint32_t)(kLmTok >> 3) << 17) | ((uint32_t)(kLmRows >> 4) << 24);
    int st = 0, ph = 0, acc = 0, aph = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      mbar_wait(&t_empty[acc], aph ^ 1);
      tc_fence_after();
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&full[st], ph);
        tc_fence_after();
        if (lane == 0) {
          uint8_t* o = smem + st * kLsStage;
          const uint64_t dEh = make_sw128_desc(smem_u32(o)), dEl = make_sw128_desc(smem_u32(o + kLs16));
          const uint64_t dXh = make_sw128_desc(smem_u32(o + 2 * kLs16));
          const uint64_t dXl = make_sw128_desc(smem_u32(o + 2 * kLs16 + kLmX));
#pragma unroll
          for (int t3 = 0; t3 < 3; ++t3)
#pragma unroll
            for (int ks = 0; ks < kLmK / 16; ++ks)
              mma_f16_ss(tmem + acc * 16, (t3 == 2 ? dEl : dEh) + 2 * ks, (t3 == 1 ? dXl : dXh) + 2 * ks, idesc,
                         (kb | ks | t3) != 0);
          mma_commit(&s_empty[st]);
        }
        __syncwarp();
        if (++st == kLsS) st = 0, ph ^= 1;
      }
      if (lane == 0) mma_commit(&t_full[acc]);
      __syncwarp();
      if (++acc == 2) acc = 0, aph ^= 1;
    }
  } else {
    pdl_wait();
    const int quarter = warp & 3;
    int acc = 0, aph = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      mbar_wait(&t_full[acc], aph);
      tc_fence_after();
      uint32_t lg[16];
      tmem_ld16(tmem + ((uint32_t)(quarter * 32) << 16) + acc * 16, lg);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&t_empty[acc]);
      if (++acc == 2) acc = 0, aph ^= 1;
      const int64_t v = (int64_t)tile * kLmRows + quarter * 32 + lane;
#pragma unroll
      for (int t = 0; t < kLmTok; ++t) {
        if (t >= ntok) break;
        const float val = __fmul_rn(__fmul_rn(__uint_as_float(lg[t]), inv_fe), xinv[t]);
        uint32_t u = __float_as_uint(val);
        u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
        unsigned long long key = v < vocab ? (((unsigned long long)u << 32) | (0xFFFFFFFFull - (uint64_t)v)) : 0ull;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          const unsigned long long o2 = __shfl_xor_sync(0xffffffffu, key, off);
          key = o2 > key ? o2 : key;
        }
        if (lane == 0 && key) atomicMax(keys + t, key);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 32);
}

// Embedding -> (hi, lo) f16 terms of emb * fe (fe: the caller's power of two).
__global__ void lm_embed_split_kernel(const float* __restrict__ emb, int64_t n2, float fe, __half* __restrict__ hi,
                                      __half* __restrict__ lo) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x) {
    const float2 v = reinterpret_cast<const float2*>(emb)[i];
    uint32_t h, l;
    lm_split(__fmul_rn(v.x, fe), __fmul_rn(v.y, fe), h, l);
    reinterpret_cast<uint32_t*>(hi)[i] = h;
    reinterpret_cast<uint32_t*>(lo)[i] = l;
  }
}

__global__ void lm_final_kernel(const unsigned long long* __restrict__ keys, int ntok, int64_t* __restrict__ ids) {
  pdl_trigger();
  pdl_wait();
  const int t = threadIdx.x;
  if (t < ntok) ids[t] = (int64_t)(0xFFFFFFFFull - (keys[t] & 0xFFFFFFFFull));
}

}  // namespace zq

using namespace zq;

namespace zq {
int make_tmap_f32(CUtensorMap* tm, const void* base, int64_t rows, int64_t cols, int64_t ld_bytes,
                  int box_cols, int box_rows, CUtensorMapSwizzle sw);
}

extern "C" {

int zq_kv_append(const float* qkv, int64_t ld_qkv, int batch, int rows_per_seq, int dmodel_local,
                 const int32_t* pos, float* kcache, float* vcache, int64_t max_ctx, void* stream) {
  ZQ_CHECK_ARG(batch >= 1 && rows_per_seq >= 1 && dmodel_local >= 4 && dmodel_local % 4 == 0,
               ZQ_ERR_SHAPE, "bad kv append shape");
  ZQ_CHECK_ARG(ld_qkv % 4 == 0 && (reinterpret_cast<uintptr_t>(qkv) & 15) == 0, ZQ_ERR_USAGE,
               "qkv rows must be 16-byte aligned");
  const int64_t total4 = (int64_t)batch * rows_per_seq * (dmodel_local / 4);
  int blocks = (int)((total4 + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  const cudaError_t e = launch_kernel(kv_append_kernel, dim3(blocks), dim3(256), 0,
                                      reinterpret_cast<cudaStream_t>(stream), 1, qkv, ld_qkv,
                                      rows_per_seq, dmodel_local, pos, kcache, vcache, max_ctx, total4);
  if (e != cudaSuccess) {
    set_error("kv append launch: %s", cudaGetErrorString(e));
    return ZQ_ERR_CUDA;
  }
  return ZQ_OK;
}

int zq_lm_head_argmax(const float* x, int64_t ld_x, int ntok, const float* emb, int64_t vocab, int64_t dim,
                      float emb_scale, void* xh_ws, void* xl_ws, float* xinv_ws, unsigned long long* keys_ws,
                      int64_t* ids, void* stream) {
  ZQ_CHECK_ARG(ntok >= 1 && ntok <= kLmTok, ZQ_ERR_UNSUPPORTED, "lm head: 1..16 tokens per step");
  ZQ_CHECK_ARG(dim % kLmK == 0 && vocab >= 1, ZQ_ERR_UNSUPPORTED, "lm head: dim must be a multiple of 64");
  ZQ_CHECK_ARG((reinterpret_cast<uintptr_t>(emb) & 15) == 0 && (reinterpret_cast<uintptr_t>(xh_ws) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(xl_ws) & 15) == 0,
               ZQ_ERR_USAGE, "lm head operands must be 16-byte aligned");
  const int nsm = zq_num_sms();
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  CUtensorMap tm;
  int rc = make_tmap_f32(&tm, emb, vocab, dim, dim * 4, 32, kLmRows, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc != ZQ_OK) return rc;
  static ZqDeviceOnce attr_once;
  attr_once([&](int) {
    cudaFuncSetAttribute(lm_head_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kLmSmem);
  });
  // emb_scale: the power of two the caller chose once for the embedding
  const float fe = emb_scale;
  const float inv_fe = 1.0f / emb_scale;
  cudaError_t e = launch_kernel(lm_prep_kernel, dim3(kLmTok), dim3(256), 0, st, 1, x, ld_x, ntok, (int)dim,
                                reinterpret_cast<__half*>(xh_ws), reinterpret_cast<__half*>(xl_ws), xinv_ws, keys_ws);
  if (e == cudaSuccess) {
    const int ntiles = (int)((vocab + kLmRows - 1) / kLmRows);
    e = launch_kernel(lm_head_kernel, dim3(ntiles < nsm ? ntiles : nsm), dim3(192), kLmSmem, st, 1, tm,
                      reinterpret_cast<const __half*>(xh_ws), reinterpret_cast<const __half*>(xl_ws),
                      (const float*)xinv_ws, ntok, vocab, (int)dim, fe, inv_fe, keys_ws);
  }
  if (e == cudaSuccess) e = launch_kernel(lm_final_kernel, dim3(1), dim3(32), 0, st, 1, (const unsigned long long*)keys_ws, ntok, ids);
  if (e != cudaSuccess) {
    set_error("lm head launch: %s", cudaGetErrorString(e));
    return ZQ_ERR_CUDA;
  }
  return ZQ_OK;
}

static bool dec_tma_enabled() {
  static int use_tma = -1;  // ZQ_DEC_TMA=0: the register-load kernel
  if (use_tma < 0) {
    const char* ev = getenv("ZQ_DEC_TMA");
    use_tma = ev ? atoi(ev) : 1;
  }
  return use_tma != 0;
}

int zq_lm_embed_split(const float* emb, int64_t vocab, int64_t dim, float emb_scale, void* emb_hi, void* emb_lo,
                      void* stream) {
  ZQ_CHECK_ARG(vocab >= 1 && dim >= 2 && dim % 2 == 0, ZQ_ERR_SHAPE, "bad embedding shape");
  const int64_t n2 = vocab * dim / 2;
  const int blocks = (int)std::min<int64_t>((n2 + 255) / 256, (int64_t)zq_num_sms() * 16);
  lm_embed_split_kernel<<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      emb, n2, emb_scale, reinterpret_cast<__half*>(emb_hi), reinterpret_cast<__half*>(emb_lo));
  ZQ_LAUNCH_CHECK("embedding split launch");
  return ZQ_OK;
}

int zq_lm_head_argmax_split(const float* x, int64_t ld_x, int ntok, const void* emb_hi, const void* emb_lo,
                            int64_t vocab, int64_t dim, float emb_scale, void* xh_ws, void* xl_ws, float* xinv_ws,
                            unsigned long long* keys_ws, int64_t* ids, void* stream) {
  ZQ_CHECK_ARG(ntok >= 1 && ntok <= kLmTok, ZQ_ERR_UNSUPPORTED, "lm head: 1..16 tokens per step");
  ZQ_CHECK_ARG(dim % kLmK == 0 && vocab >= 1, ZQ_ERR_UNSUPPORTED, "lm head: dim must be a multiple of 64");
  ZQ_CHECK_ARG((reinterpret_cast<uintptr_t>(emb_hi) & 15) == 0 && (reinterpret_cast<uintptr_t>(emb_lo) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(xh_ws) & 15) == 0 && (reinterpret_cast<uintptr_t>(xl_ws) & 15) == 0,
               ZQ_ERR_USAGE, "lm head operands must be 16-byte aligned");
  const int nsm = zq_num_sms();
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  CUtensorMap teh, tel, txh, txl;
  int rc = make_tmap_2d(&teh, CU_TENSOR_MAP_DATA_TYPE_UINT16, emb_hi, vocab, dim, dim * 2, kLmK, kLmRows,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  if (!rc) rc = make_tmap_2d(&tel, CU_TENSOR_MAP_DATA_TYPE_UINT16, emb_lo, vocab, dim, dim * 2, kLmK, kLmRows,
                             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  if (!rc) rc = make_tmap_2d(&txh, CU_TENSOR_MAP_DATA_TYPE_UINT16, xh_ws, kLmTok, dim, dim * 2, kLmK, kLmTok,
                             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  if (!rc) rc = make_tmap_2d(&txl, CU_TENSOR_MAP_DATA_TYPE_UINT16, xl_ws, kLmTok, dim, dim * 2, kLmK, kLmTok,
                             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  if (rc) return rc;
  static ZqDeviceOnce attr_once;
  attr_once([&](int) {
    cudaFuncSetAttribute(lm_head_split_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kLsSmem);
  });
  cudaError_t e = launch_kernel(lm_prep_kernel, dim3(kLmTok), dim3(256), 0, st, 1, x, ld_x, ntok, (int)dim,
                                reinterpret_cast<__half*>(xh_ws), reinterpret_cast<__half*>(xl_ws), xinv_ws, keys_ws);
  if (e == cudaSuccess) {
    const int ntiles = (int)((vocab + kLmRows - 1) / kLmRows);
    e = launch_kernel(lm_head_split_kernel, dim3(ntiles < nsm ? ntiles : nsm), dim3(192), kLsSmem, st, 1, teh, tel,
                      txh, txl, (const float*)xinv_ws, ntok, vocab, (int)dim, 1.0f / emb_scale, keys_ws);
  }
  if (e == cudaSuccess)
    e = launch_kernel(lm_final_kernel, dim3(1), dim3(32), 0, st, 1, (const unsigned long long*)keys_ws, ntok, ids);
  if (e != cudaSuccess) {
    set_error("lm head (split) launch: %s", cudaGetErrorString(e));
    return ZQ_ERR_CUDA;
  }
  return ZQ_OK;
}

int zq_decode_attention_chunks(int batch, int heads, int64_t max_ctx) {
  // context chunks per (sequence, head), at most 8 (portable cluster).  TMA
  // kernel (measured, tools/dec_attn_bench.py): ~512 CTAs with 2-stage rings,
  // >= 32 keys per chunk.  Register-load kernel: ~1000 CTAs of 4 warps (7 per
  // SM), >= 16 keys per chunk.
  int C = 1;
  if (dec_tma_enabled()) {
    while (C < 8 && (int64_t)batch * heads * C * 2 <= 512 && max_ctx / (2 * C) >= 32) C *= 2;
    return C;
  }
  while (C < 8 && (int64_t)batch * heads * C * 2 <= 7 * 148 && max_ctx / (2 * C) >= 16) C *= 2;
  return C;
}

int zq_decode_attention_f32(const float* q, int64_t ld_q, const float* kcache, const float* vcache,
                            int64_t max_ctx, int batch, int heads, int head_dim,
                            const int32_t* lens, float scale, float* ctx, int64_t ld_ctx,
                            int chunks, void* stream) {
  ZQ_CHECK_ARG(batch >= 1 && heads >= 1 && max_ctx >= 1, ZQ_ERR_SHAPE, "bad decode attention shape");
  ZQ_CHECK_ARG(head_dim % 32 == 0 && head_dim <= 256, ZQ_ERR_UNSUPPORTED,
               "decode attention supports head_dim % 32 == 0 and <= 256");
  ZQ_CHECK_ARG(chunks == 0 || chunks == 1 || chunks == 2 || chunks == 4 || chunks == 8, ZQ_ERR_USAGE,
               "decode attention chunks must be 0 (auto), 1, 2, 4 or 8, got %d", chunks);
  const int C = chunks ? chunks : zq_decode_attention_chunks(batch, heads, max_ctx);
  const int chunk = (int)((max_ctx + C - 1) / C);
  cudaError_t e;
  const int64_t dl = (int64_t)heads * head_dim;
  if (dec_tma_enabled() && (head_dim == 64 || head_dim == 96 || head_dim == 128 || head_dim == 256) &&
      (reinterpret_cast<uintptr_t>(kcache) & 15) == 0 && (reinterpret_cast<uintptr_t>(vcache) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(q) & 15) == 0 && ld_q % 4 == 0 && (int64_t)batch * max_ctx < (1LL << 31)) {
    CUtensorMap tk, tv;
    static int kt64 = -1;  // ZQ_DEC_KT=16: 16-key tiles x 8 stages for head_dim 64 (experiments)
    if (kt64 < 0) {
      const char* ev = getenv("ZQ_DEC_KT");
      kt64 = ev ? atoi(ev) : 32;
    }
    const int kt = head_dim == 64 ? (kt64 == 16 ? 16 : 32) : head_dim == 256 ? 8 : 16;
    static int stg = -1;  // ZQ_DEC_STG: ring stages (2 / 4 / 8)
    if (stg < 0) {
      const char* ev = getenv("ZQ_DEC_STG");
      stg = ev ? atoi(ev) : 2;
    }
    int rc = make_tmap_f32(&tk, kcache, (int64_t)batch * max_ctx, dl, dl * 4, head_dim, kt, CU_TENSOR_MAP_SWIZZLE_NONE);
    if (rc == ZQ_OK)
      rc = make_tmap_f32(&tv, vcache, (int64_t)batch * max_ctx, dl, dl * 4, head_dim, kt, CU_TENSOR_MAP_SWIZZLE_NONE);
    if (rc != ZQ_OK) return rc;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
#define ZQ_DECT(DH_, KT_, LPK_, NF_, STG_)                                                                 \
  {                                                                                                         \
    using Cfg = DecTmaCfg<DH_, KT_, LPK_, NF_, STG_>;                                                       \
    static ZqDeviceOnce attr_once;                                                                          \
    attr_once([&](int) {                                                                                    \
      cudaFuncSetAttribute(decode_attention_tma_kernel<DH_, KT_, LPK_, NF_, STG_>,                          \
                           cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);                         \
    });                                                                                                     \
    e = launch_kernel(decode_attention_tma_kernel<DH_, KT_, LPK_, NF_, STG_>, dim3(batch * heads * C),      \
                      dim3(160), Cfg::SMEM, st, C, tk, tv, q, ld_q, max_ctx, heads, lens, scale, ctx,      \
                      ld_ctx, C);                                                                           \
  }
#define ZQ_DECT_S(DH_, KT_, LPK_, NF_) \
  if (stg == 2) ZQ_DECT(DH_, KT_, LPK_, NF_, 2) else if (stg == 8) ZQ_DECT(DH_, KT_, LPK_, NF_, 8) else ZQ_DECT(DH_, KT_, LPK_, NF_, 4)
    if (head_dim == 64) {
      if (kt == 16) { ZQ_DECT_S(64, 16, 16, 1) } else { ZQ_DECT_S(64, 32, 16, 1) }
    } else if (head_dim == 96) { ZQ_DECT_S(96, 16, 8, 3) }
    else if (head_dim == 128) { ZQ_DECT_S(128, 16, 32, 1) }
    else { ZQ_DECT_S(256, 8, 32, 2) }
#undef ZQ_DECT_S
#undef ZQ_DECT
    if (e != cudaSuccess) {
      set_error("decode attention (tma) launch: %s", cudaGetErrorString(e));
      return ZQ_ERR_CUDA;
    }
    return ZQ_OK;
  }
#define ZQ_DEC(TT, LL, NN, UU)                                                                           \
  e = launch_kernel(decode_attention_kernel<TT, LL, NN, UU>, dim3(batch * heads * C), dim3(TT), 0,      \
                    reinterpret_cast<cudaStream_t>(stream), C, q, ld_q, kcache, vcache, max_ctx, heads,  \
                    head_dim, lens, scale, ctx, ld_ctx, C, chunk)
  const int d4 = head_dim / 4;
  if (d4 <= 8) ZQ_DEC(128, 8, 1, 2);
  else if (d4 <= 16) ZQ_DEC(128, 16, 1, 2);
  else if (d4 <= 24) ZQ_DEC(128, 8, 3, 1);
  else if (d4 <= 32) ZQ_DEC(128, 32, 1, 2);
  else ZQ_DEC(128, 32, 2, 2);
#undef ZQ_DEC
  if (e != cudaSuccess) {
    set_error("decode attention launch: %s", cudaGetErrorString(e));
    return ZQ_ERR_CUDA;
  }
  return ZQ_OK;
}

}  // extern "C"
