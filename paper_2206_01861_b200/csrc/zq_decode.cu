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
#include <string.h>

#include "zq_common.cuh"

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

}  // namespace zq

using namespace zq;

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

int zq_decode_attention_f32(const float* q, int64_t ld_q, const float* kcache, const float* vcache,
                            int64_t max_ctx, int batch, int heads, int head_dim,
                            const int32_t* lens, float scale, float* ctx, int64_t ld_ctx,
                            void* stream) {
  ZQ_CHECK_ARG(batch >= 1 && heads >= 1 && max_ctx >= 1, ZQ_ERR_SHAPE, "bad decode attention shape");
  ZQ_CHECK_ARG(head_dim % 32 == 0 && head_dim <= 256, ZQ_ERR_UNSUPPORTED,
               "decode attention supports head_dim % 32 == 0 and <= 256");
  // context chunks per (sequence, head): split until ~1000 CTAs of 4 warps are in
  // flight (7 per SM), at most 8 (portable cluster), keeping >= 16 keys per chunk
  int C = 1;
  while (C < 8 && (int64_t)batch * heads * C * 2 <= 7 * 148 && max_ctx / (2 * C) >= 16) C *= 2;
  {
    static int force = -1;
    if (force < 0) {
      const char* ev = getenv("ZQ_DEC_C");
      force = ev ? atoi(ev) : 0;
    }
    if (force >= 1 && force <= 8) C = force;
  }
  const int chunk = (int)((max_ctx + C - 1) / C);
  static int wide_env = -1;
  if (wide_env < 0) {
    const char* ev = getenv("ZQ_DEC_WIDE");
    wide_env = ev ? atoi(ev) : 0;
  }
  const bool wide = wide_env == 1;
  cudaError_t e;
#define ZQ_DEC(TT, LL, NN, UU)                                                                           \
  e = launch_kernel(decode_attention_kernel<TT, LL, NN, UU>, dim3(batch * heads * C), dim3(TT), 0,      \
                    reinterpret_cast<cudaStream_t>(stream), C, q, ld_q, kcache, vcache, max_ctx, heads,  \
                    head_dim, lens, scale, ctx, ld_ctx, C, chunk)
  (void)wide;
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
