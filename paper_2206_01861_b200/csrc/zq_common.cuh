// Shared helpers for the sm_100a kernels: status codes, thread-local error text,
// exact quantization arithmetic, and thin inline-PTX wrappers (mbarrier, TMA,
// tcgen05) used by the GEMM.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <atomic>

#include "zq_b200.h"

// Launcher state is per device: a process may drive several GPUs (and several
// host threads may launch concurrently).  ZqDeviceOnce runs its body once per
// device ordinal (idempotent bodies only: two threads may both run it);
// zq_num_sms() caches the SM count per device.
struct ZqDeviceOnce {
  std::atomic<unsigned long long> done{0};
  template <class F>
  void operator()(F&& body) {
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return;
    body(dev);
    done.fetch_or(bit, std::memory_order_acq_rel);
  }
};

static inline int zq_num_sms() {
  static std::atomic<int> cache[64];
  int dev = 0;
  cudaGetDevice(&dev);
  int v = cache[dev & 63].load(std::memory_order_relaxed);
  if (v <= 0) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    cache[dev & 63].store(v, std::memory_order_relaxed);
  }
  return v;
}

namespace zq {

// ---------------------------------------------------------------------------
// host-side error reporting
// ---------------------------------------------------------------------------
void set_error(const char* fmt, ...);

// ---------------------------------------------------------------------------
// Programmatic dependent launch (PDL).  Every hot-path kernel is launched with
// programmatic stream serialization, calls pdl_trigger() early (the next kernel
// may start its prologue: barrier init, TMEM alloc, tensor-map prefetch, weight
// TMA loads) and pdl_wait() before touching anything a previous kernel writes
// or reads (griddepcontrol.wait returns once the preceding grid has completed
// and its memory is visible).  ZQ_PDL=0 disables the launch attribute.
// ---------------------------------------------------------------------------
bool pdl_enabled();

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_kernel(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                 cudaStream_t st, unsigned cluster_x, Args... args) {
  cudaLaunchConfig_t cfg;
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  unsigned n = 0;
  if (cluster_x > 1) {
    at[n].id = cudaLaunchAttributeClusterDimension;
    at[n].val.clusterDim.x = cluster_x;
    at[n].val.clusterDim.y = 1;
    at[n].val.clusterDim.z = 1;
    ++n;
  }
  if (pdl_enabled()) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.attrs = at;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

#define ZQ_CHECK_ARG(cond, code, ...)     \
  do {                                    \
    if (!(cond)) {                        \
      ::zq::set_error(__VA_ARGS__);       \
      return (code);                      \
    }                                     \
  } while (0)

#define ZQ_LAUNCH_CHECK(what)                                                  \
  do {                                                                         \
    cudaError_t e_ = cudaGetLastError();                                       \
    if (e_ != cudaSuccess) {                                                   \
      ::zq::set_error("%s: %s", (what), cudaGetErrorString(e_));               \
      return ZQ_ERR_CUDA;                                                      \
    }                                                                          \
  } while (0)

inline int qmax_of(int bits) { return (1 << (bits - 1)) - 1; }
inline bool bits_ok(int bits) { return bits == 4 || bits == 8; }

// ---------------------------------------------------------------------------
// device: exact ZeroQuant rounding (pkg/src/lowbit/quant.py:98-113, :229-233)
// ---------------------------------------------------------------------------

// Scale from a row max (quant.py:222-226): f32(f64(maxabs) / qmax), 0 -> 1.0.
// That double rounding equals one correctly rounded f32 division: for f32 a and
// odd qm (127, 7) the exact quotient a/qm is never an f32 rounding midpoint and
// stays >= 2^-32 (relative) away from every midpoint (the numerator
// a*2^k - qm*(2j+1) is a nonzero integer multiple of the midpoint grid), far
// beyond the f64 quotient's 2^-53 error, so RN_f32(RN_f64(a/qm)) = RN_f32(a/qm)
// (also for subnormal a).  The f32 IEEE division keeps the FP64 pipe (slow on
// this part) off every row's critical path.
__device__ __forceinline__ float scale_from_absmax(float amax, int qm) {
  if (amax == 0.0f) return 1.0f;
  return __fdiv_rn(amax, (float)qm);
}

// q = clamp(sign(x) * floor(|x|/s + 1/2), +-qm) for f32 x and f32 s > 0.
// The reference divides in f64; for f32 operands its result equals exact
// round-half-away of the rational |x|/s (the f64 quotient cannot cross a
// half-integer it is not exactly on).  We estimate k from an f32 quotient and
// fix it with an exact boundary test on (k -+ 1/2) * s.
__device__ __forceinline__ int quantize_exact(float x, float s, int qm) {
  float ax = fabsf(x);
  float r = fminf(__fdiv_rn(ax, s), 512.0f);
  int k = __float2int_rd(__fadd_rn(r, 0.5f));
  // (k -+ 1/2) * s - |x| with a single rounding (FMA): its sign is the sign of the
  // exact value (zero stays zero), so the boundary tests are exact in f32
  if (__fmaf_rn((float)k - 0.5f, s, -ax) > 0.0f) {
    k -= 1;
  } else if (__fmaf_rn((float)k + 0.5f, s, -ax) <= 0.0f) {
    k += 1;
  }
  k = min(k, qm);
  return x < 0.0f ? -k : k;
}

// Out-of-line copy for rarely taken fallbacks (keeps hot loops small in I$).
static __device__ __noinline__ int quantize_exact_slow(float x, float s, int qm) {
  return quantize_exact(x, s, qm);
}

// Fast exact variant.  r = |x| * (1/s) with the correctly rounded reciprocal
// is within 2^-15 (absolute, for r < 200) of the true quotient q.  RHAFZ(q) is
// the integer nearest q (ties away), so rint(r) is exact unless q is within
// that error of a half-integer; the magic-number rounding (r + 1.5*2^23 rounds
// to an integer in the FMA pipe) gives rint(r) and the distance to it, and
// near-ties (|d - 1/2| < 2^-14: ~1e-4 of elements, and every planted tie) take
// the exact path above.  `inv` = safe_rcp(s); inv == 0 forces the exact path.
__device__ __forceinline__ int quantize_fast(float x, float s, float inv, int qm) {
  const float r = __fmul_rn(fabsf(x), inv);
  int k;
  if (r >= 200.0f) {
    k = qm;
  } else {
    const float m = __fadd_rn(r, 12582912.0f);        // RN(r) in the low mantissa bits
    const float d = fabsf(__fsub_rn(r, __fsub_rn(m, 12582912.0f)));  // |r - rint(r)|, exact
    if (d > 0.49993896484375f || inv == 0.0f) return quantize_exact_slow(x, s, qm);
    k = min(__float_as_int(m) - 0x4B400000, qm);
  }
  return x < 0.0f ? -k : k;
}

// |x| as a u32 bit pattern: monotone for finite values, and inf/NaN compare
// above every finite value, so one max tracks both the row max and the
// non-finite flag (bits >= 0x7f800000).
__device__ __forceinline__ uint32_t abs_bits(float x) { return __float_as_uint(x) & 0x7fffffffu; }

// Correctly rounded a / b given y = RN(1/b): two Newton corrections with exact
// FMA residuals (q0 = RN(a*y) can be 1.5 ulp off, so one correction is not
// enough; two gave 0 mismatches vs IEEE division on 2e5 random pairs checked
// with exact rationals).  Operands / quotients near the subnormal or overflow
// range take the IEEE division.
__device__ __forceinline__ float div_rn_fast(float a, float b, float y) {
  const float q0 = __fmul_rn(a, y);
  const float aq = fabsf(q0);
  if (!(aq > 1e-30f && aq < 1e30f) || !(fabsf(a) > 1e-30f)) return __fdiv_rn(a, b);
  const float q1 = __fmaf_rn(__fmaf_rn(-b, q0, a), y, q0);
  return __fmaf_rn(__fmaf_rn(-b, q1, a), y, q1);
}

__device__ __forceinline__ float safe_rcp(float s) {
  const float inv = __frcp_rn(s);
  return (inv < 1e30f) ? inv : 0.0f;
}

// Static path with an arbitrary f64 scale: numpy's exact op sequence
// (f64 divide, f64 add 0.5, floor, clip).
__device__ __forceinline__ int quantize_f64(float x, double s, int qm) {
  double v = __ddiv_rn((double)x, s);
  double a = floor(__dadd_rn(fabs(v), 0.5));
  a = fmin(a, (double)qm);
  int k = (int)a;
  return v < 0.0 ? -k : k;
}

__device__ __forceinline__ bool is_finite_f(float x) {
  return (__float_as_uint(x) & 0x7f800000u) != 0x7f800000u;
}

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ---------------------------------------------------------------------------
// Branch-free exact quantization.  With inv = RN(1/s), x*inv is within
// |x/s| * 2^-24 (< 2^-16 for |x/s| <= 127) of the true quotient.  One FMA
// rounds x*inv + 1.5*2^23 to an integer (the magic constant pins the ulp to 1),
// a second FMA gives the residual x*inv - k exactly up to 2^-25, and RHAFZ(x/s)
// equals that k unless the quotient is within the margin of a half-integer, in
// which case `amb` is raised and the caller redoes the element exactly.  No
// clamp is needed: the token scale comes from the row's max, so |x*inv| <= qm
// (1 + 2^-16) < qm + 1/2 (GeLU estimates stay within 2^-17 of that max).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int qbf(float x, float inv, int qm, float margin, bool& amb) {
  (void)qm;
  const float m = __fmaf_rn(x, inv, 12582912.0f);
  const float k = __fsub_rn(m, 12582912.0f);
  amb |= fabsf(__fmaf_rn(x, inv, -k)) > 0.5f - margin;
  return __float_as_int(m) - 0x4B400000;
}

// four signed bytes (low byte of each int) -> one word, in three byte permutes
__device__ __forceinline__ uint32_t pack4(int a, int b, int c, int d) {
  return __byte_perm(__byte_perm((uint32_t)a, (uint32_t)b, 0x0040), __byte_perm((uint32_t)c, (uint32_t)d, 0x0040),
                     0x5410);
}

constexpr float kQMargin = 6.103515625e-05f;  // 2^-14

// Packed f32x2 arithmetic (sm_100 FFMA2 / FMUL2 / FADD2): two IEEE
// round-to-nearest operations per instruction, each bit-identical to __fmaf_rn /
// __fmul_rn / __fadd_rn / __fsub_rn.  The row quantizers are issue-bound.
// CAUTION: ptxas contracts f2mul feeding f2add / f2sub into one FFMA2 (single
// rounding) despite the .rn modifiers; where the product must be rounded, do
// the multiply-add pair with scalar __fmul_rn / __fadd_rn.
__device__ __forceinline__ uint64_t f2pack(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2unpack(uint64_t v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t f2fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t f2mul(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t f2add(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t f2sub(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t f2splat(float a) { return f2pack(a, a); }

// qbf on four elements, two per packed instruction (nk = magic - m = -k exactly;
// the low byte of m's bits is k's byte, all pack4 reads), one
// compare on the largest |residual| (FMNMX3; a NaN residual is never ambiguous,
// as with the per-element compares), then pack4
__device__ __forceinline__ uint32_t qbf4(float4 v, float inv, float margin, bool& amb) {
  const uint64_t inv2 = f2splat(inv);
  const uint64_t xa = f2pack(v.x, v.y), xb = f2pack(v.z, v.w);
  const uint64_t ma = f2fma(xa, inv2, f2splat(12582912.0f)), mb = f2fma(xb, inv2, f2splat(12582912.0f));
  float r0, r1, r2, r3, m0, m1, m2, m3;
  f2unpack(f2fma(xa, inv2, f2sub(f2splat(12582912.0f), ma)), r0, r1);
  f2unpack(f2fma(xb, inv2, f2sub(f2splat(12582912.0f), mb)), r2, r3);
  f2unpack(ma, m0, m1);
  f2unpack(mb, m2, m3);
  amb |= fmaxf(fmaxf(fabsf(r0), fabsf(r1)), fmaxf(fabsf(r2), fabsf(r3))) > 0.5f - margin;
  return pack4(__float_as_int(m0), __float_as_int(m1), __float_as_int(m2), __float_as_int(m3));
}

// Block-wide max of a non-negative float (as its u32 bit pattern — monotone for
// non-negative floats, NaN never reaches here because the finite flag is raised
// separately).  `red` must hold >= 32 words.
__device__ __forceinline__ float block_max_nonneg(float v, uint32_t* red) {
  // redux.sync per warp, one slot per warp, then every warp reduces the slots
  // itself (two barriers; the leading one protects the slots of the last call)
  uint32_t b = __reduce_max_sync(0xffffffffu, __float_as_uint(v));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = b;
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  b = l < nw ? red[l] : 0u;
  return __uint_as_float(__reduce_max_sync(0xffffffffu, b));
}

// ---------------------------------------------------------------------------
// PTX wrappers (sm_100a)
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* smem_dst, const void* tmap, uint64_t* bar,
                                            int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// smem -> global tensor store (bulk async group), clipped to the tensor bounds.
__device__ __forceinline__ void tma_store_2d(const void* tmap, const void* smem_src, int32_t c0,
                                             int32_t c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   tmap),
               "r"(smem_u32(smem_src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__device__ __forceinline__ void prefetch_tmap(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---- tcgen05 ---------------------------------------------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// D[tmem] (+)= A[smem] * B[smem]^T, int8 x int8 -> int32, one elected thread.
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Arrive on an mbarrier once all previously issued tcgen05.mma of this thread complete.
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

// 32 lanes x 32 consecutive 32-bit columns -> 32 registers per thread.
__device__ __forceinline__ void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// ---- CTA pairs (cta_group::2) ---------------------------------------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cta address of the same object in the even (leader) CTA of the pair:
// bit 24 of a shared window address selects the peer CTA.
__device__ __forceinline__ uint32_t leader_addr(const void* p) { return smem_u32(p) & 0xFEFFFFFFu; }

__device__ __forceinline__ void mbar_arrive_cluster(uint32_t addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(addr) : "memory");
}
// TMA load into the issuing CTA's smem, completing bytes on the pair leader's barrier.
__device__ __forceinline__ void tma_load_2d_cg2(void* smem_dst, const void* tmap, uint32_t bar_leader,
                                                int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(tmap), "r"(bar_leader), "r"(c0), "r"(c1)
      : "memory");
}
// The same, multicast: the tile lands at the same offset in every CTA of
// `mask`, and each destination's pair leader barrier receives its bytes.
__device__ __forceinline__ void tma_load_2d_cg2_mc(void* smem_dst, const void* tmap, uint32_t bar_leader,
                                                   int32_t c0, int32_t c1, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(tmap), "r"(bar_leader), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void tmem_alloc_cg2(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_cg2(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
// D[tmem of both CTAs] (+)= A[smem of both CTAs] * B[smem of both CTAs]^T, M = 256.
__device__ __forceinline__ void mma_i8_cg2(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                           uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive (once) on the barrier at this offset in every CTA of `mask` when all
// prior tcgen05.mma of the pair complete.
__device__ __forceinline__ void mma_commit_mc2(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

// Shared-memory matrix descriptor for a K-major, SWIZZLE_128B operand tile whose
// rows are 128 bytes and whose 8-row core groups are 1024 bytes apart
// (SM100 UMMA descriptor: start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46),
// version=1 [46,48), base_offset [49,52), layout SWIZZLE_128B=2 [61,64)).
__device__ __forceinline__ uint64_t make_sw128_desc(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr & 0x3FFFFu) >> 4);
  d |= (uint64_t)(16u >> 4) << 16;   // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024u >> 4) << 32; // SBO: 8 rows x 128 B
  d |= (uint64_t)1 << 46;            // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;            // SWIZZLE_128B
  return d;
}

// Instruction descriptor: kind::i8, A/B signed int8, K-major both, D = s32.
__host__ __device__ constexpr uint32_t make_idesc_i8(int M, int N) {
  return (2u << 4)                       // c_format = S32
         | (1u << 7)                     // a_format = INT8 (signed)
         | (1u << 10)                    // b_format = INT8 (signed)
         | ((uint32_t)(N >> 3) << 17)    // N >> 3
         | ((uint32_t)(M >> 4) << 24);   // M >> 4
}

}  // namespace zq
