// Float attention of the post-LN block (transformer.py:413-440) on tcgen05:
//   S = (Q K^T) * 1/sqrt(dh); causal -> -inf above the diagonal; P = softmax(S);
//   ctx = P V
// The reference computes this in float32 (sequential sums); it is outside the
// bit-exact contract (tolerance parity), but we keep ~fp32 accuracy: every
// operand x is split into hi = x with the low 13 mantissa bits cleared (exactly
// representable in tf32) and lo = x - hi (exact in f32), and each product is
// formed as hi*hi + hi*lo + lo*hi (3 tcgen05 kind::tf32 MMAs into one f32 TMEM
// accumulator) — relative error ~2^-21 instead of tf32's 2^-11.  The tensor core
// reads only the top 19 bits of a tf32 operand (measured: feeding the raw f32 as
// "hi" gives the same 3e-6 error as the explicitly truncated value), so the raw
// TMA-staged tiles serve as hi and only lo is written.
//
// One CTA per (sequence, head), seq <= 128, head_dim = 64 (BERT-base, GPT-3
// 350M heads).  256 threads:
//   1. one thread TMA-loads Q, K, V of the head (6 boxes of [128 rows x 32 f32],
//      SWIZZLE_128B) straight from the fused QKV GEMM output: Q and K land in
//      the K-major layout the MMA reads;
//   2. all threads write lo(Q), lo(K) (the same swizzled layout, so a flat
//      elementwise pass) and transpose V into K-major V^T hi / lo (with B
//      MN-major the kind::tf32 MMA returned zeros, so only K-major is used);
//   3. thread 0 issues 24 MMAs for S (M=128, N=128, K=64) -> TMEM cols [0,128);
//   4. 8 warps softmax: warp w reads TMEM lanes 32*(w%4).. (query rows), column
//      half w/4; row max / sum combined through smem; P hi/lo written to smem
//      over the (now free) Q/K buffers;
//   5. thread 0 issues 48 MMAs for O (M=128, N=64, K=128, B = V^T)
//      -> TMEM cols [128,192);
//   6. 8 warps read O and store ctx rows (f32).
#include <cuda.h>

#include "zq_common.cuh"

namespace zq {

constexpr int kAttT = 128;   // max sequence (query rows = MMA M)
constexpr int kAttD = 64;    // head dim
// smem: [Qh | Ql | Kh | Kl | V | VTh | VTl], 32 KB each.  Q/K: 2 K-major atoms
// of [128 rows x 128 B] (32 head-dim columns each), as TMA lands them.  V: the
// same TMA layout (rows = tokens); VTh/VTl: V^T hi/lo as the K-major B operand
// of P.V (64 rows = head dim, 4 atoms of 32 tokens).  P hi / lo (128 x 128 f32,
// 4 K-major atoms each) overlay Qh..Kl once S is computed.
constexpr int kRegion = kAttT * kAttD * 4;         // 32 KB
constexpr int kAttSmem = 7 * kRegion + 128 + 2 * 128 * 4;

__device__ __forceinline__ uint32_t make_idesc_tf32(int M, int N, int b_mn_major) {
  return (1u << 4)                       // c_format F32
         | (2u << 7)                     // a_format TF32
         | (2u << 10)                    // b_format TF32
         | ((uint32_t)b_mn_major << 16)  // B major-ness (1 = MN-major)
         | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// MN-major SWIZZLE_128B operand (kept for reference: with kind::tf32 and B
// MN-major the MMA produced zeros on this B200 build, so V is transposed): 128-byte rows hold 32 consecutive MN elements,
// 8 rows (K) per 1024-byte swizzle atom; LBO = stride between 32-element MN
// blocks, SBO = stride between 8-row K groups.
__device__ __forceinline__ uint64_t make_sw128_mn_desc(uint32_t smem_addr, uint32_t lbo,
                                                       uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr & 0x3FFFFu) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
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

__device__ __forceinline__ float ex2_approx_f(float v) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}

// One elected lane of a converged warp issues the MMA (operands warp-uniform, so
// no per-lane R2UR loops around the instruction).
__device__ __forceinline__ void mma_tf32_elect(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                               uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n"
      ".reg .pred e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
      "}\n" ::"r"(smem_u32(bar))
      : "memory");
}

// hi = x with the low 13 mantissa bits cleared (a tf32 value), lo = x - hi (exact)
__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  hi = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
  lo = __fsub_rn(x, hi);
}

// byte offset of element (row r, k) in a K-major SWIZZLE_128B operand of `rows`
// rows: atoms of 128 bytes along K, each [rows][128 B], 16-byte chunks XORed
// with (row & 7)
__device__ __forceinline__ uint32_t sw_off(int rows, int r, int k_bytes) {
  const int atom = k_bytes >> 7, wb = k_bytes & 127;
  return atom * rows * 128 + r * 128 + ((((wb >> 4) ^ (r & 7))) << 4) + (wb & 15);
}

__global__ void __launch_bounds__(256, 1)
    attention_kernel(const __grid_constant__ CUtensorMap tm, int seq, int heads, int dmodel,
                     int causal, float scale, float* __restrict__ ctx, int64_t ld_ctx, int dbg) {
  // no static smem in this kernel: the dynamic window starts 1024-aligned, and
  // addressing it directly (no integer round trip) keeps every access LDS/STS
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sQh = sm;
  uint8_t* sQl = sm + kRegion;
  uint8_t* sKh = sm + 2 * kRegion;
  uint8_t* sKl = sm + 3 * kRegion;
  uint8_t* sV = sm + 4 * kRegion;
  uint8_t* sVh = sm + 5 * kRegion;
  uint8_t* sVl = sm + 6 * kRegion;
  uint8_t* sPh = sQh;  // P (128 x 128 f32 = 64 KB) overlays Q hi/lo
  uint8_t* sPl = sKh;  // and K hi/lo
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 7 * kRegion);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 3);
  float* red = reinterpret_cast<float*>(bar + 4);  // [2][128] row partials (max / sum)

  const int b = blockIdx.x / heads, h = blockIdx.x % heads;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  unsigned long long ts[8];
  ts[0] = gtime();

  if (tid == 0) {
    if (smem_u32(sm) & 1023) __trap();  // SWIZZLE_128B atoms need 1024-byte alignment
    prefetch_tmap(&tm);
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_init(&bar[2], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(tslot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  ts[1] = gtime();

  // ---- 1. TMA: Q, K, V boxes of this (sequence, head) ----
  pdl_trigger();
  pdl_wait();  // the QKV GEMM output is ready (and the previous ctx reader is done)
  if (tid == 0) {
    mbar_arrive_expect_tx(&bar[0], 6 * 128 * 128);
    const int row0 = b * seq;
#pragma unroll
    for (int part = 0; part < 3; ++part)
#pragma unroll
      for (int j = 0; j < 2; ++j)
        tma_load_2d(sm + (part == 2 ? 4 : 2 * part) * kRegion + j * (kRegion / 2), &tm, &bar[0],
                    part * dmodel + h * kAttD + 32 * j, row0);
  }
  mbar_wait(&bar[0], 0);
  ts[2] = gtime();

  // ---- 2. split Q, K hi / lo in place (flat pass over the swizzled tiles);
  //         V -> V^T hi / lo (lane = head-dim column j, 4 consecutive tokens)
  for (int i = tid; i < 2 * (kRegion / 16); i += 256) {
    const int part = i / (kRegion / 16), off = (i % (kRegion / 16)) * 16;
    const float4 x = *reinterpret_cast<const float4*>(sm + 2 * part * kRegion + off);
    float4 hi, lo;
    split_tf32(x.x, hi.x, lo.x);
    split_tf32(x.y, hi.y, lo.y);
    split_tf32(x.z, hi.z, lo.z);
    split_tf32(x.w, hi.w, lo.w);
    *reinterpret_cast<float4*>(sm + (2 * part + 1) * kRegion + off) = lo;
  }
  {
    const int j = (warp & 1) * 32 + lane;  // head-dim column
    const uint8_t* vcol = sV + (j >> 5) * (kRegion / 2) + (j & 3) * 4;
    const int jc = (j & 31) >> 2;
#pragma unroll 2
    for (int q = warp >> 1; q < kAttT / 4; q += 4) {  // token quad
      float v[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int t = 4 * q + e;
        v[e] = *reinterpret_cast<const float*>(vcol + t * 128 + ((jc ^ (t & 7)) << 4));
      }
      float4 hi, lo;
      split_tf32(v[0], hi.x, lo.x);
      split_tf32(v[1], hi.y, lo.y);
      split_tf32(v[2], hi.z, lo.z);
      split_tf32(v[3], hi.w, lo.w);
      hi = make_float4(v[0], v[1], v[2], v[3]);  // the MMA reads only the tf32 bits
      const uint32_t o = (q >> 3) * (kAttD * 128) + j * 128 + (((q & 7) ^ (j & 7)) << 4);
      *reinterpret_cast<float4*>(sVh + o) = hi;
      *reinterpret_cast<float4*>(sVl + o) = lo;
    }
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  ts[3] = gtime();
  // ---- 3. S = Q K^T (3-term split) ----
  if (warp == 0) {  // whole warp walks the issue loop (uniform descriptors), one lane issues
    const uint32_t idesc = make_idesc_tf32(128, 128, 0);
    const uint64_t dQh = make_sw128_desc(smem_u32(sQh)), dQl = make_sw128_desc(smem_u32(sQl));
    const uint64_t dKh = make_sw128_desc(smem_u32(sKh)), dKl = make_sw128_desc(smem_u32(sKl));
#pragma unroll
    for (int t3 = 0; t3 < 3; ++t3)
#pragma unroll
      for (int ks = 0; ks < kAttD / 8; ++ks) {  // K step = 8 tf32 = 32 bytes
        const int kb = 32 * ks;
        const uint64_t aoff = (uint64_t)(((kb >> 7) * kAttT * 128 + (kb & 127)) >> 4);
        mma_tf32_elect(tmem, (t3 == 2 ? dQl : dQh) + aoff, (t3 == 1 ? dKl : dKh) + aoff, idesc,
                       (t3 | ks) != 0);
      }
    mma_commit_elect(&bar[1]);
  }

  // ---- 4. softmax rows ----
  const int quarter = warp & 3, half = warp >> 2;
  const int row = quarter * 32 + lane;  // query index (TMEM lane)
  mbar_wait(&bar[1], 0);
  tc_fence_after();
  ts[4] = gtime();
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
    float v = __fmul_rn(s[j], scale);                        // scores *= inv (transformer.py:432)
    if (key >= seq || (causal && key > row)) v = -INFINITY;  // mask (transformer.py:433-434)
    s[j] = v;
    mx = fmaxf(mx, v);
  }
  red[half * 128 + row] = mx;
  __syncthreads();
  mx = fmaxf(red[row], red[128 + row]);
  // exp(s - mx) = 2^((s - mx) * log2 e), branch-free: masked scores give 2^-inf = 0
  // (key 0 is never masked, so mx is finite); relative error ~1e-6
  float sum = 0.0f;
#pragma unroll
  for (int j = 0; j < 64; ++j) {
    const float e = ex2_approx_f(__fmul_rn(__fsub_rn(s[j], mx), 1.4426950408889634f));
    s[j] = e;
    sum = __fadd_rn(sum, e);
  }
  __syncthreads();
  red[half * 128 + row] = sum;
  __syncthreads();
  sum = __fadd_rn(red[row], red[128 + row]);
  const float inv_sum = __frcp_rn(sum);
  // P hi/lo -> smem (rows = queries, K = keys), overlaying Q/K (S MMAs are done)
#pragma unroll
  for (int j4 = 0; j4 < 16; ++j4) {
    float4 ph, pl;
    float p0 = __fmul_rn(s[4 * j4], inv_sum), p1 = __fmul_rn(s[4 * j4 + 1], inv_sum);
    float p2 = __fmul_rn(s[4 * j4 + 2], inv_sum), p3 = __fmul_rn(s[4 * j4 + 3], inv_sum);
    split_tf32(p0, ph.x, pl.x);
    split_tf32(p1, ph.y, pl.y);
    split_tf32(p2, ph.z, pl.z);
    split_tf32(p3, ph.w, pl.w);
    const uint32_t o = sw_off(kAttT, row, 4 * (half * 64 + 4 * j4));
    *reinterpret_cast<float4*>(sPh + o) = ph;
    *reinterpret_cast<float4*>(sPl + o) = pl;
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  ts[5] = gtime();
  // ---- 5. O = P V (3-term split), N = 64 ----
  if (warp == 0) {
    const uint32_t idesc = make_idesc_tf32(128, kAttD, 0);
    const uint64_t dPh = make_sw128_desc(smem_u32(sPh)), dPl = make_sw128_desc(smem_u32(sPl));
    const uint64_t dVh = make_sw128_desc(smem_u32(sVh)), dVl = make_sw128_desc(smem_u32(sVl));
#pragma unroll
    for (int t3 = 0; t3 < 3; ++t3)
#pragma unroll
      for (int ks = 0; ks < kAttT / 8; ++ks) {
        const int kb = 32 * ks;
        const uint64_t aoff = (uint64_t)(((kb >> 7) * kAttT * 128 + (kb & 127)) >> 4);
        const uint64_t boff = (uint64_t)(((kb >> 7) * kAttD * 128 + (kb & 127)) >> 4);
        mma_tf32_elect(tmem + 128, (t3 == 2 ? dPl : dPh) + aoff, (t3 == 1 ? dVl : dVh) + boff, idesc,
                       (t3 | ks) != 0);
      }
    mma_commit_elect(&bar[2]);
  }
  mbar_wait(&bar[2], 0);
  tc_fence_after();
  ts[6] = gtime();
  {
    uint32_t r0[32];
    tmem_ld_32x32b_x32(tmem + ((uint32_t)(quarter * 32) << 16) + 128 + half * 32, r0);
    tmem_ld_wait();
    if (row < seq && dbg != 20) {
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
  ts[7] = gtime();
  if (dbg == 20 && tid == 0) {
    unsigned long long* o = reinterpret_cast<unsigned long long*>(ctx) + blockIdx.x * 8;
    for (int k = 0; k < 8; ++k) o[k] = ts[k];
  }
  if (warp == 0) tmem_dealloc(tmem, 256);
}

int make_tmap_f32(CUtensorMap* tm, const void* base, int64_t rows, int64_t cols, int64_t ld_bytes,
                  int box_cols, int box_rows, CUtensorMapSwizzle sw);

}  // namespace zq

using namespace zq;

static int g_att_dbg = 0;
extern "C" int zq_attention_debug(int mode) {
  g_att_dbg = mode;
  return ZQ_OK;
}

extern "C" int zq_attention_f32(const float* qkv, int64_t ld_qkv, int batch, int seq, int heads,
                                int head_dim, int causal, float scale, float* ctx, int64_t ld_ctx,
                                void* stream) {
  ZQ_CHECK_ARG(batch >= 1 && seq >= 1 && heads >= 1, ZQ_ERR_SHAPE, "bad attention shape");
  ZQ_CHECK_ARG(seq <= kAttT && head_dim == kAttD, ZQ_ERR_UNSUPPORTED,
               "fused attention supports seq <= 128 and head_dim == 64");
  ZQ_CHECK_ARG(ld_qkv % 4 == 0 && ld_ctx % 4 == 0 && (reinterpret_cast<uintptr_t>(qkv) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(ctx) & 15) == 0,
               ZQ_ERR_UNSUPPORTED, "attention operands must be 16-byte aligned");
  CUtensorMap tm;
  const int rc = make_tmap_f32(&tm, qkv, (int64_t)batch * seq, 3LL * heads * head_dim, ld_qkv * 4,
                               32, kAttT, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc != ZQ_OK) return rc;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kAttSmem);
    attr = true;
  }
  const cudaError_t e = launch_kernel(attention_kernel, dim3(batch * heads), dim3(256), kAttSmem,
                                      reinterpret_cast<cudaStream_t>(stream), 1, tm, seq, heads,
                                      heads * head_dim, causal, scale, ctx, ld_ctx, g_att_dbg);
  if (e != cudaSuccess) {
    set_error("attention launch: %s", cudaGetErrorString(e));
    return ZQ_ERR_CUDA;
  }
  return ZQ_OK;
}
