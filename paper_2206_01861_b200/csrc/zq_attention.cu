// Float attention of the post-LN block (transformer.py:413-440) on tcgen05:
//   S = (Q K^T) * 1/sqrt(dh); causal -> -inf above the diagonal; P = softmax(S);
//   ctx = P V
// The reference computes this in float32 (sequential sums); it is outside the
// bit-exact contract (tolerance parity), but we keep ~fp32 accuracy: every
// operand is split into tf32 hi + lo and each product is formed as
// hi*hi + hi*lo + lo*hi (3 tcgen05 kind::tf32 MMAs into one f32 TMEM
// accumulator) — relative error ~2^-21 instead of tf32's 2^-11.
//
// One CTA per (sequence, head), seq <= 128, head_dim = 64 (BERT-base, GPT-3
// 350M heads).  256 threads:
//   1. all threads stage Q, K (K-major, SWIZZLE_128B atoms) and V^T as hi/lo;
//   2. thread 0 issues 24 MMAs for S (M=128, N=128, K=64) -> TMEM cols [0,128);
//   3. 8 warps softmax: warp w reads TMEM lanes 32*(w%4).. (query rows), column
//      half w/4; row max / sum combined through smem; P hi/lo written to smem
//      over the (now free) Q/K buffers;
//   4. thread 0 issues 48 MMAs for O (M=128, N=64, K=128) -> TMEM cols [128,192);
//   5. 8 warps read O and store ctx rows (f32).
#include "zq_common.cuh"

namespace zq {

constexpr int kAttT = 128;   // max sequence (query rows = MMA M)
constexpr int kAttD = 64;    // head dim
// smem: Qhi Qlo Khi Klo (128 rows x 256 B each, 2 atoms) | Vthi Vtlo (64 rows x 512 B)
constexpr int kQKBytes = kAttT * kAttD * 4;        // 32 KB per operand copy
constexpr int kVBytes = kAttD * kAttT * 4;         // 32 KB
constexpr int kAttSmem = 4 * kQKBytes + 2 * kVBytes + 1024 + 128 + 8 * 2 * 128 * 4;

__device__ __forceinline__ uint32_t make_idesc_tf32(int M, int N) {
  return (1u << 4)                       // c_format F32
         | (2u << 7)                     // a_format TF32
         | (2u << 10)                    // b_format TF32
         | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// tf32 split: hi keeps the top 10 mantissa bits (round to nearest), lo = x - hi
__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  const uint32_t b = __float_as_uint(x);
  hi = __uint_as_float((b + 0x1000u) & 0xFFFFE000u);
  lo = __fsub_rn(x, hi);
}

// byte offset of element (row r, k) in a K-major SWIZZLE_128B operand of `rows`
// rows: atoms of 128 bytes along K, each [rows][128 B], 16-byte chunks XORed
// with (row & 7)
__device__ __forceinline__ uint32_t sw_off(int rows, int r, int k_bytes) {
  const int atom = k_bytes >> 7, wb = k_bytes & 127;
  return atom * rows * 128 + r * 128 + ((((wb >> 4) ^ (r & 7))) << 4) + (wb & 15);
}

__global__ void __launch_bounds__(256, 1) attention_kernel(const float* __restrict__ qkv,
                                                           int64_t ld, int seq, int heads,
                                                           int dmodel, int causal, float scale,
                                                           float* __restrict__ ctx,
                                                           int64_t ld_ctx) {
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQh = sm;
  uint8_t* sQl = sm + kQKBytes;
  uint8_t* sKh = sm + 2 * kQKBytes;
  uint8_t* sKl = sm + 3 * kQKBytes;
  uint8_t* sVh = sm + 4 * kQKBytes;
  uint8_t* sVl = sVh + kVBytes;
  uint8_t* sPh = sQh;                 // P (128 x 128 f32 = 64 KB) overlays Q hi/lo
  uint8_t* sPl = sKh;                 // and K hi/lo
  uint64_t* bar = reinterpret_cast<uint64_t*>(sVl + kVBytes);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 2);
  float* red = reinterpret_cast<float*>(bar + 4);  // [2][128] row partials (max / sum)

  const int b = blockIdx.x / heads, h = blockIdx.x % heads;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const float* base = qkv + (int64_t)b * seq * ld;

  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(tslot, 256);

  // ---- 1. stage Q, K (rows = tokens) and V^T (rows = head dim) as tf32 hi/lo ----
  for (int idx = tid; idx < kAttT * (kAttD / 4); idx += 256) {
    const int r = idx / (kAttD / 4), c4 = idx % (kAttD / 4);
    float4 q = make_float4(0.f, 0.f, 0.f, 0.f), k = q, v = q;
    if (r < seq) {
      const float* rowp = base + (int64_t)r * ld + h * kAttD + 4 * c4;
      q = __ldg(reinterpret_cast<const float4*>(rowp));
      k = __ldg(reinterpret_cast<const float4*>(rowp + dmodel));
      v = __ldg(reinterpret_cast<const float4*>(rowp + 2 * dmodel));
    }
    float4 hq, lq, hk, lk;
    split_tf32(q.x, hq.x, lq.x); split_tf32(q.y, hq.y, lq.y);
    split_tf32(q.z, hq.z, lq.z); split_tf32(q.w, hq.w, lq.w);
    split_tf32(k.x, hk.x, lk.x); split_tf32(k.y, hk.y, lk.y);
    split_tf32(k.z, hk.z, lk.z); split_tf32(k.w, hk.w, lk.w);
    const uint32_t o = sw_off(kAttT, r, 16 * c4);
    *reinterpret_cast<float4*>(sQh + o) = hq;
    *reinterpret_cast<float4*>(sQl + o) = lq;
    *reinterpret_cast<float4*>(sKh + o) = hk;
    *reinterpret_cast<float4*>(sKl + o) = lk;
    const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {  // V^T: row = head-dim index, K = token
      float vh, vl;
      split_tf32(vv[e], vh, vl);
      const uint32_t ov = sw_off(kAttD, 4 * c4 + e, 4 * r);
      *reinterpret_cast<float*>(sVh + ov) = vh;
      *reinterpret_cast<float*>(sVl + ov) = vl;
    }
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  // ---- 2. S = Q K^T (3-term split) ----
  if (tid == 0) {
    const uint32_t idesc = make_idesc_tf32(128, 128);
    const uint8_t* As[3] = {sQh, sQh, sQl};
    const uint8_t* Bs[3] = {sKh, sKl, sKh};
    int first = 1;
    for (int t3 = 0; t3 < 3; ++t3)
      for (int ks = 0; ks < kAttD / 8; ++ks) {  // K step = 8 tf32 = 32 bytes
        const int kb = 32 * ks;
        const uint32_t aoff = (kb >> 7) * kAttT * 128 + (kb & 127);
        mma_tf32(tmem, make_sw128_desc(smem_u32(As[t3]) + aoff), make_sw128_desc(smem_u32(Bs[t3]) + aoff),
                 idesc, first ? 0u : 1u);
        first = 0;
      }
    mma_commit(&bar[0]);
  }
  __syncwarp();

  // ---- 3. softmax rows ----
  const int quarter = warp & 3, half = warp >> 2;
  const int row = quarter * 32 + lane;           // query index (TMEM lane)
  mbar_wait(&bar[0], 0);
  tc_fence_after();
  float s[64];
  {
    uint32_t r0[32], r1[32];
    const uint32_t ta = tmem + ((uint32_t)(quarter * 32) << 16) + half * 64;
    tmem_ld_32x32b_x32(ta, r0);
    tmem_ld_32x32b_x32(ta + 32, r1);
    tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      s[j] = __uint_as_float(r0[j]);
      s[32 + j] = __uint_as_float(r1[j]);
    }
  }
  float mx = -INFINITY;
#pragma unroll
  for (int j = 0; j < 64; ++j) {
    const int key = half * 64 + j;
    float v = __fmul_rn(s[j], scale);                       // scores *= inv (transformer.py:432)
    if (key >= seq || (causal && key > row)) v = -INFINITY;  // mask (transformer.py:433-434)
    s[j] = v;
    mx = fmaxf(mx, v);
  }
  red[half * 128 + row] = mx;
  __syncthreads();
  mx = fmaxf(red[row], red[128 + row]);
  float sum = 0.0f;
#pragma unroll
  for (int j = 0; j < 64; ++j) {
    const float e = (s[j] == -INFINITY) ? 0.0f : expf(__fsub_rn(s[j], mx));
    s[j] = e;
    sum = __fadd_rn(sum, e);
  }
  __syncthreads();
  red[half * 128 + row] = sum;
  __syncthreads();
  sum = __fadd_rn(red[row], red[128 + row]);
  const float inv_sum = 1.0f / sum;
  // P hi/lo -> smem (rows = queries, K = keys), overlaying Q/K (S MMAs are done)
#pragma unroll
  for (int j4 = 0; j4 < 16; ++j4) {
    float4 ph, pl;
    float p0 = __fmul_rn(s[4 * j4], inv_sum), p1 = __fmul_rn(s[4 * j4 + 1], inv_sum);
    float p2 = __fmul_rn(s[4 * j4 + 2], inv_sum), p3 = __fmul_rn(s[4 * j4 + 3], inv_sum);
    split_tf32(p0, ph.x, pl.x); split_tf32(p1, ph.y, pl.y);
    split_tf32(p2, ph.z, pl.z); split_tf32(p3, ph.w, pl.w);
    const uint32_t o = sw_off(kAttT, row, 4 * (half * 64 + 4 * j4));
    *reinterpret_cast<float4*>(sPh + o) = ph;
    *reinterpret_cast<float4*>(sPl + o) = pl;
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  // ---- 4. O = P V (3-term split), N = 64 ----
  if (tid == 0) {
    const uint32_t idesc = make_idesc_tf32(128, kAttD);
    const uint8_t* As[3] = {sPh, sPh, sPl};
    const uint8_t* Bs[3] = {sVh, sVl, sVh};
    int first = 1;
    for (int t3 = 0; t3 < 3; ++t3)
      for (int ks = 0; ks < kAttT / 8; ++ks) {
        const int kb = 32 * ks;
        const uint32_t aoff = (kb >> 7) * kAttT * 128 + (kb & 127);
        const uint32_t boff = (kb >> 7) * kAttD * 128 + (kb & 127);
        mma_tf32(tmem + 128, make_sw128_desc(smem_u32(As[t3]) + aoff),
                 make_sw128_desc(smem_u32(Bs[t3]) + boff), idesc, first ? 0u : 1u);
        first = 0;
      }
    mma_commit(&bar[1]);
  }
  __syncwarp();
  mbar_wait(&bar[1], 0);
  tc_fence_after();
  {
    uint32_t r0[32];
    tmem_ld_32x32b_x32(tmem + ((uint32_t)(quarter * 32) << 16) + 128 + half * 32, r0);
    tmem_ld_wait();
    if (row < seq) {
      float* dst = ctx + ((int64_t)b * seq + row) * ld_ctx + h * kAttD + half * 32;
#pragma unroll
      for (int j = 0; j < 32; j += 4)
        *reinterpret_cast<float4*>(dst + j) =
            make_float4(__uint_as_float(r0[j]), __uint_as_float(r0[j + 1]),
                        __uint_as_float(r0[j + 2]), __uint_as_float(r0[j + 3]));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 256);
}

}  // namespace zq

using namespace zq;

extern "C" int zq_attention_f32(const float* qkv, int64_t ld_qkv, int batch, int seq, int heads,
                                int head_dim, int causal, float scale, float* ctx, int64_t ld_ctx,
                                void* stream) {
  ZQ_CHECK_ARG(batch >= 1 && seq >= 1 && heads >= 1, ZQ_ERR_SHAPE, "bad attention shape");
  ZQ_CHECK_ARG(seq <= kAttT && head_dim == kAttD, ZQ_ERR_UNSUPPORTED,
               "fused attention supports seq <= 128 and head_dim == 64");
  ZQ_CHECK_ARG(ld_qkv % 4 == 0 && ld_ctx % 4 == 0 && (reinterpret_cast<uintptr_t>(qkv) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(ctx) & 15) == 0,
               ZQ_ERR_UNSUPPORTED, "attention operands must be 16-byte aligned");
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kAttSmem);
    attr = true;
  }
  attention_kernel<<<batch * heads, 256, kAttSmem, reinterpret_cast<cudaStream_t>(stream)>>>(
      qkv, ld_qkv, seq, heads, heads * head_dim, causal, scale, ctx, ld_ctx);
  ZQ_LAUNCH_CHECK("attention launch");
  return ZQ_OK;
}
