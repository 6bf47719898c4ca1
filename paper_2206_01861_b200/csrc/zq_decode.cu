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
// keys [c*chunk, (c+1)*chunk) below lens[b] and produces a partial
// (max m_c, sum l_c, unnormalised o_c = sum_j e^(s_j - m_c) v_j); after a cluster
// barrier each CTA combines dims [c*dh/C, (c+1)*dh/C) of all C partials through
// distributed shared memory:  o = sum_c o_c e^(m_c - M) / sum_c l_c e^(m_c - M).
// 256 threads; scores: 8 lanes per key (4 keys per warp step, float4 chunks,
// xor-reduce); P.V: G = 256/(dh/4) key groups of dh/4 threads (float4 of dims).
constexpr int kDecThreads = 256;

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

__global__ void __launch_bounds__(kDecThreads) decode_attention_kernel(
    const float* __restrict__ q, int64_t ld_q, const float* __restrict__ kc,
    const float* __restrict__ vc, int64_t max_ctx, int heads, int dh,
    const int32_t* __restrict__ lens, float scale, float* __restrict__ ctx, int64_t ld_ctx,
    int C, int chunk) {
  extern __shared__ float dsm[];
  __shared__ float red[32];
  __shared__ float stat[2];  // m_c, l_c
  pdl_trigger();
  pdl_wait();
  const int c = (int)cta_rank_in_cluster();
  const int bh = blockIdx.x / C;
  const int b = bh / heads, h = bh % heads;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int dl = heads * dh;
  const int len = lens[b];
  const int j0 = c * chunk, j1 = min(len, j0 + chunk);
  const int G = kDecThreads / (dh >> 2);
  float* sq = dsm;                 // [dh]
  float* sc = dsm + 256;           // [chunk]
  float* po = sc + chunk;          // [G][dh] partial outputs; row 0 = o_c after the reduce
  for (int i = tid; i < dh; i += kDecThreads) sq[i] = q[(int64_t)b * ld_q + h * dh + i];
  __syncthreads();

  const int d4 = dh >> 2;
  const float* kb = kc + (int64_t)b * max_ctx * dl + h * dh;
  const float* vb = vc + (int64_t)b * max_ctx * dl + h * dh;
  {
    const int sub = lane >> 3, l8 = lane & 7;
#pragma unroll 2
    for (int jj = j0 + warp * 4; jj < j1; jj += 4 * (kDecThreads / 32)) {
      const int j = jj + sub;
      float acc = 0.0f;
      if (j < j1) {
        // issue every load of the key row first (dh <= 256: <= 8 float4 per lane)
        const float4* kr = reinterpret_cast<const float4*>(kb + (int64_t)j * dl);
        float4 kv[8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
          kv[i] = (l8 + 8 * i < d4) ? __ldg(kr + l8 + 8 * i) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (l8 + 8 * i < d4) {
            const float4 qv = *reinterpret_cast<const float4*>(sq + 4 * (l8 + 8 * i));
            acc = __fmaf_rn(qv.x, kv[i].x, acc);
            acc = __fmaf_rn(qv.y, kv[i].y, acc);
            acc = __fmaf_rn(qv.z, kv[i].z, acc);
            acc = __fmaf_rn(qv.w, kv[i].w, acc);
          }
        }
      }
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      acc += __shfl_xor_sync(0xffffffffu, acc, 4);
      if (l8 == 0 && j < j1) sc[j - j0] = __fmul_rn(acc, scale);
    }
  }
  __syncthreads();
  float mx = -INFINITY;
  for (int j = tid; j < j1 - j0; j += kDecThreads) mx = fmaxf(mx, sc[j]);
  mx = warp_max(mx);
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  mx = red[0];
#pragma unroll
  for (int w = 1; w < kDecThreads / 32; ++w) mx = fmaxf(mx, red[w]);
  __syncthreads();
  float sum = 0.0f;
  for (int j = tid; j < j1 - j0; j += kDecThreads) {
    const float e = expf(sc[j] - mx);
    sc[j] = e;
    sum += e;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if (lane == 0) red[warp] = sum;
  __syncthreads();
  if (tid == 0) {
    float t = 0.0f;
    for (int w = 0; w < kDecThreads / 32; ++w) t += red[w];
    stat[0] = mx;  // -inf for an empty chunk
    stat[1] = t;
  }
  const int g = tid / d4, cc = tid % d4;
  float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
  if (g < G) {
#pragma unroll 8
    for (int j = j0 + g; j < j1; j += G) {
      const float pj = sc[j - j0];
      const float4 v = __ldg(reinterpret_cast<const float4*>(vb + (int64_t)j * dl) + cc);
      o.x = __fmaf_rn(pj, v.x, o.x);
      o.y = __fmaf_rn(pj, v.y, o.y);
      o.z = __fmaf_rn(pj, v.z, o.z);
      o.w = __fmaf_rn(pj, v.w, o.w);
    }
    *reinterpret_cast<float4*>(po + g * dh + 4 * cc) = o;
  }
  __syncthreads();
  for (int i = tid; i < dh; i += kDecThreads) {
    float t = 0.0f;
    for (int gg = 0; gg < G; ++gg) t += po[gg * dh + i];
    po[i] = t;  // row 0 of po = o_c
  }
  cluster_barrier();
  // combine dims [c*dh/C, (c+1)*dh/C) across the cluster
  const int da = (c * dh) / C, db = ((c + 1) * dh) / C;
  const uint32_t stat_a = smem_u32(stat), po_a = smem_u32(po);
  float M = -INFINITY;
  for (int r = 0; r < C; ++r) M = fmaxf(M, dsm_ld_f32(dsm_map(stat_a, r)));
  float L = 0.0f;
  for (int r = 0; r < C; ++r) {
    const float mr = dsm_ld_f32(dsm_map(stat_a, r));
    if (mr != -INFINITY) L += dsm_ld_f32(dsm_map(stat_a + 4, r)) * expf(mr - M);
  }
  for (int i = da + tid; i < db; i += kDecThreads) {
    float t = 0.0f;
    for (int r = 0; r < C; ++r) {
      const float mr = dsm_ld_f32(dsm_map(stat_a, r));
      if (mr != -INFINITY) t += dsm_ld_f32(dsm_map(po_a + 4 * i, r)) * expf(mr - M);
    }
    ctx[(int64_t)b * ld_ctx + h * dh + i] = t / L;
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
  // context chunks per (sequence, head): split until ~4 CTAs per SM are in flight,
  // at most 8 (portable cluster), keeping >= 32 keys per chunk
  int C = 1;
  while (C < 8 && (int64_t)batch * heads * C < 4 * 148 && max_ctx / (2 * C) >= 32) C *= 2;
  const int chunk = (int)(((max_ctx + C - 1) / C + 3) / 4 * 4);  // keeps the partial-output rows 16-byte aligned
  const int G = kDecThreads / (head_dim / 4);
  const size_t smem = sizeof(float) * (256 + (size_t)chunk + (size_t)G * head_dim);
  ZQ_CHECK_ARG(smem <= 200 * 1024, ZQ_ERR_UNSUPPORTED, "context too long for decode attention");
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(decode_attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    attr = true;
  }
  cudaError_t e = launch_kernel(decode_attention_kernel, dim3(batch * heads * C), dim3(kDecThreads), smem,
                                reinterpret_cast<cudaStream_t>(stream), C, q, ld_q, kcache, vcache,
                                max_ctx, heads, head_dim, lens, scale, ctx, ld_ctx, C, chunk);
  if (e != cudaSuccess) {
    set_error("decode attention launch: %s", cudaGetErrorString(e));
    return ZQ_ERR_CUDA;
  }
  return ZQ_OK;
}

}  // extern "C"
