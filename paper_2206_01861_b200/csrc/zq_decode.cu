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
#include "zq_common.cuh"

namespace zq {

// cache[b, pos[b] + t, c] = qkv[b*rows_per_seq + t, col0 + c] for the k and v blocks
__global__ void kv_append_kernel(const float* __restrict__ qkv, int64_t ld_qkv, int rows_per_seq,
                                 int dl, const int32_t* __restrict__ pos, float* __restrict__ kc,
                                 float* __restrict__ vc, int64_t max_ctx, int64_t total4) {
  const int d4 = dl >> 2;
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

// One CTA (256 threads) per (sequence, head).  dh % 32 == 0, dh <= 256.
//  1. scores: 8 lanes per key (4 keys per warp step), float4 chunks, xor-reduce;
//  2. softmax over lens[b] scores in smem (block max / sum);
//  3. ctx = sum_j p_j v_j: G key groups of dh/4 threads (one float4 of dims
//     each), partial sums combined through smem.
__global__ void __launch_bounds__(256) decode_attention_kernel(
    const float* __restrict__ q, int64_t ld_q, const float* __restrict__ kc,
    const float* __restrict__ vc, int64_t max_ctx, int heads, int dh,
    const int32_t* __restrict__ lens, float scale, float* __restrict__ ctx, int64_t ld_ctx) {
  extern __shared__ float dsm[];
  __shared__ float red[32];
  const int b = blockIdx.x / heads, h = blockIdx.x % heads;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int dl = heads * dh;
  const int len = lens[b];
  float* sq = dsm;            // [dh]
  float* sc = dsm + 256;      // [max_ctx] scores -> probabilities
  float* part = sc + max_ctx; // [G][dh] partial outputs
  for (int i = tid; i < dh; i += 256) sq[i] = q[(int64_t)b * ld_q + h * dh + i];
  __syncthreads();

  const int d4 = dh >> 2;
  const float* kb = kc + (int64_t)b * max_ctx * dl + h * dh;
  const float* vb = vc + (int64_t)b * max_ctx * dl + h * dh;
  {
    const int sub = lane >> 3, l8 = lane & 7;
    for (int j0 = warp * 4; j0 < len; j0 += 32) {
      const int j = j0 + sub;
      float acc = 0.0f;
      if (j < len) {
        const float4* kr = reinterpret_cast<const float4*>(kb + (int64_t)j * dl);
        for (int c = l8; c < d4; c += 8) {
          const float4 kv = __ldg(kr + c);
          const float4 qv = *reinterpret_cast<const float4*>(sq + 4 * c);
          acc = __fmaf_rn(qv.x, kv.x, acc);
          acc = __fmaf_rn(qv.y, kv.y, acc);
          acc = __fmaf_rn(qv.z, kv.z, acc);
          acc = __fmaf_rn(qv.w, kv.w, acc);
        }
      }
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      acc += __shfl_xor_sync(0xffffffffu, acc, 4);
      if (l8 == 0 && j < len) sc[j] = __fmul_rn(acc, scale);
    }
  }
  __syncthreads();
  float mx = -INFINITY;
  for (int j = tid; j < len; j += 256) mx = fmaxf(mx, sc[j]);
  mx = warp_max(mx);
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  mx = red[0];
#pragma unroll
  for (int w = 1; w < 8; ++w) mx = fmaxf(mx, red[w]);
  __syncthreads();
  float sum = 0.0f;
  for (int j = tid; j < len; j += 256) {
    const float e = expf(sc[j] - mx);
    sc[j] = e;
    sum += e;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if (lane == 0) red[warp] = sum;
  __syncthreads();
  sum = 0.0f;
#pragma unroll
  for (int w = 0; w < 8; ++w) sum += red[w];
  const float inv = 1.0f / sum;

  const int G = 256 / d4;  // key groups
  const int g = tid / d4, c = tid % d4;
  float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
  if (g < G) {
    for (int j = g; j < len; j += G) {
      const float p = sc[j];
      const float4 v = __ldg(reinterpret_cast<const float4*>(vb + (int64_t)j * dl) + c);
      o.x = __fmaf_rn(p, v.x, o.x);
      o.y = __fmaf_rn(p, v.y, o.y);
      o.z = __fmaf_rn(p, v.z, o.z);
      o.w = __fmaf_rn(p, v.w, o.w);
    }
    *reinterpret_cast<float4*>(part + g * dh + 4 * c) = o;
  }
  __syncthreads();
  for (int i = tid; i < dh; i += 256) {
    float s = 0.0f;
    for (int gg = 0; gg < G; ++gg) s += part[gg * dh + i];
    ctx[(int64_t)b * ld_ctx + h * dh + i] = s * inv;
  }
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
  kv_append_kernel<<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      qkv, ld_qkv, rows_per_seq, dmodel_local, pos, kcache, vcache, max_ctx, total4);
  ZQ_LAUNCH_CHECK("kv append launch");
  return ZQ_OK;
}

int zq_decode_attention_f32(const float* q, int64_t ld_q, const float* kcache, const float* vcache,
                            int64_t max_ctx, int batch, int heads, int head_dim,
                            const int32_t* lens, float scale, float* ctx, int64_t ld_ctx,
                            void* stream) {
  ZQ_CHECK_ARG(batch >= 1 && heads >= 1 && max_ctx >= 1, ZQ_ERR_SHAPE, "bad decode attention shape");
  ZQ_CHECK_ARG(head_dim % 32 == 0 && head_dim <= 256, ZQ_ERR_UNSUPPORTED,
               "decode attention supports head_dim % 32 == 0 and <= 256");
  const int G = 256 / (head_dim / 4);
  const size_t smem = sizeof(float) * (256 + (size_t)max_ctx + (size_t)G * head_dim);
  ZQ_CHECK_ARG(smem <= 200 * 1024, ZQ_ERR_UNSUPPORTED, "context too long for decode attention");
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(decode_attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    attr = true;
  }
  decode_attention_kernel<<<batch * heads, 256, smem, reinterpret_cast<cudaStream_t>(stream)>>>(
      q, ld_q, kcache, vcache, max_ctx, heads, head_dim, lens, scale, ctx, ld_ctx);
  ZQ_LAUNCH_CHECK("decode attention launch");
  return ZQ_OK;
}

}  // extern "C"
