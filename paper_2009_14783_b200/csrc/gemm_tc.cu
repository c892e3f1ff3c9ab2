// tcgen05 + TMA + TMEM bf16 GEMM for sm_100a (fp32 accumulation in TMEM).
//
// Persistent, warp-specialized: grid = min(#work units, #SMs); a CTA walks
// work units u = blockIdx.x, += gridDim.x.  A unit is one 128 x BN output tile
// (BN in {128, 192, 256}) over one K range (split-K for the weight-gradient
// GEMMs whose output has too few tiles to fill 148 SMs).
//   warp 0      TMA producer: STAGES-deep ring of (A 128x64, B BNx64) tiles,
//               128B-swizzled, full/empty mbarriers
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (UMMA_K=16)
//               into one of TWO accumulator buffers, so the epilogue of tile i
//               overlaps the MMAs of tile i+1
//   warps 2..17 epilogue: tcgen05.ld 32x32b.x32 -> registers -> bias / GELU /
//               dGELU / residual -> global, staged through a swizzled 2 KB
//               smem tile per warp so every global access is a full row
//               segment (coalesced; split-K uses fp32 vector reductions).
//               Warp w reads TMEM lanes 32*(w%4)..+31, every 4th 32-col chunk.
//
// Operands may be K-major or MN-major (the three GEMMs of a linear layer's
// training step: fwd X.W, dgrad dY.W^T, wgrad X^T.dY all read the canonical
// row-major weight and token-major activations without transposes), and B may
// be "grouped" (the per-head [d x dk] projection blocks wq.0..wv.{h-1} of the
// canonical layout, model.hpp:103-112) through a 3-D tensor map.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <array>
#include <map>
#include <mutex>

#include "hp_common.h"
#include "kernels.h"

namespace hp {

namespace tc {

constexpr int BM = 128;
constexpr int BK = 64;  // one 128-byte swizzle row of bf16
constexpr int STAGES = 4;
constexpr int kEpiWarps = 16;
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr uint32_t kATileBytes = BM * BK * 2;  // 16 KB

struct Params {
  int M, N, K;
  int a_mn;       // A stored MN-major (A^T row-major)
  int b_mn;       // B stored MN-major (row-major K x N)
  int b_grouped;  // B uses the 3-D grouped map (group = 64)
  int m_tiles, n_tiles, splits, kb_per_split, units;
  void* c;
  int64_t ldc;
  int64_t c_group, c_gstride;
  int c_f32;
  float alpha;
  int accumulate;
  const float* bias;
  int act;
  void* aux;
  const void* resid;
  int64_t ld_resid;
  int vec;  // C / aux / resid rows are 16-byte aligned
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_2d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0,
                                       int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_3d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0,
                                       int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// Shared-memory matrix descriptor, SWIZZLE_128B, sm_100 version bit.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accum) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

#define TMEM_LD16(taddr, r)                                                                      \
  asm volatile(                                                                                  \
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14," \
      "%15}, [%16];"                                                                             \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),      \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),  \
        "=r"(r[14]), "=r"(r[15])                                                                 \
      : "r"(taddr))

#define TMEM_LD32(taddr, r)                                                                      \
  asm volatile(                                                                                  \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14," \
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"             \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),      \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),  \
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),            \
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),            \
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])             \
      : "r"(taddr))

__device__ __forceinline__ float gelu_f(float x) {
  return 0.5f * x * (1.f + erff(x * 0.70710678118654752f));
}
__device__ __forceinline__ float dgelu_f(float x) {
  return 0.5f * (1.f + erff(x * 0.70710678118654752f)) +
         x * 0.39894228040143268f * expf(-0.5f * x * x);
}
// Branch-free normal CDF / PDF for the bf16 epilogues: erf by Abramowitz &
// Stegun 7.1.26 (|error| <= 1.5e-7, far below bf16 rounding); exp(-x^2/2) is
// shared between Phi and phi.  2 MUFU ops + ~10 FMA per element.
__device__ __forceinline__ float phi_cdf(float x, float& pdf) {
  const float z = fabsf(x) * 0.70710678118654752f;
  const float t = __frcp_rn(fmaf(0.3275911f, z, 1.f));
  const float e = __expf(-z * z);
  const float poly =
      t * fmaf(t, fmaf(t, fmaf(t, fmaf(t, 1.061405429f, -1.453152027f), 1.421413741f), -0.284496736f),
               0.254829592f);
  const float erf_abs = fmaf(-poly, e, 1.f);
  pdf = e * 0.39894228040143268f;
  return 0.5f * (1.f + copysignf(erf_abs, x));
}
__device__ __forceinline__ float gelu_fast(float x) {
  float pdf;
  return x * phi_cdf(x, pdf);
}
__device__ __forceinline__ float dgelu_fast(float x) {
  float pdf;
  const float c = phi_cdf(x, pdf);
  return fmaf(x, pdf, c);
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ void store8_bf16(__nv_bfloat16* dst, const float* v) {
  *reinterpret_cast<uint4*>(dst) = make_uint4(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]),
                                              pack_bf16(v[4], v[5]), pack_bf16(v[6], v[7]));
}
__device__ __forceinline__ void load8_bf16(const __nv_bfloat16* src, float* v) {
  const uint4 u = *reinterpret_cast<const uint4*>(src);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 f = __bfloat1622float2(h[e]);
    v[2 * e] = f.x;
    v[2 * e + 1] = f.y;
  }
}
__device__ __forceinline__ void red_add_v4(float* dst, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(a), "f"(b), "f"(c),
               "f"(d)
               : "memory");
}

// Epilogue for NC consecutive columns [n, n+NC) of row m.
template <int NC>
__device__ __forceinline__ void epilogue_cols(const Params& p, int m, int n, float* v) {
  if (m >= p.M) return;
  const bool inb = n + NC <= p.N;
  const bool full = inb && p.vec == 1;
#pragma unroll
  for (int i = 0; i < NC; ++i) v[i] *= p.alpha;
  const int64_t co = p.c_group ? (n / p.c_group) * p.c_gstride + (int64_t)m * p.ldc + n % p.c_group
                               : (int64_t)m * p.ldc + n;
  if (p.splits > 1) {  // split-K partial: reduce into the (zeroed) fp32 output
    float* c = static_cast<float*>(p.c) + co;
    if (full) {
#pragma unroll
      for (int q = 0; q < NC / 4; ++q) red_add_v4(c + 4 * q, v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    } else {
#pragma unroll
      for (int i = 0; i < NC; ++i)
        if (n + i < p.N) atomicAdd(c + i, v[i]);
    }
    return;
  }
  if (p.bias) {
    if (inb && (reinterpret_cast<uintptr_t>(p.bias + n) & 15) == 0) {
#pragma unroll
      for (int q = 0; q < NC / 4; ++q) {
        const float4 b = __ldg(reinterpret_cast<const float4*>(p.bias + n) + q);
        v[4 * q] += b.x; v[4 * q + 1] += b.y; v[4 * q + 2] += b.z; v[4 * q + 3] += b.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < NC; ++i) v[i] += (n + i < p.N) ? p.bias[n + i] : 0.f;
    }
  }
  if (p.act == ACT_GELU) {
    // pre-activation kept for the backward pass (same type as C)
    if (p.c_f32) {
      float* a = static_cast<float*>(p.aux) + co;
#pragma unroll
      for (int i = 0; i < NC; ++i)
        if (n + i < p.N) a[i] = v[i];
    } else {
      __nv_bfloat16* a = static_cast<__nv_bfloat16*>(p.aux) + co;
      if (full) {
#pragma unroll
        for (int q = 0; q < NC / 8; ++q) store8_bf16(a + 8 * q, v + 8 * q);
      } else {
#pragma unroll
        for (int i = 0; i < NC; ++i)
          if (n + i < p.N) a[i] = __float2bfloat16_rn(v[i]);
      }
    }
#pragma unroll
    for (int i = 0; i < NC; ++i) v[i] = gelu_fast(v[i]);
  } else if (p.act == ACT_DGELU) {
    if (p.c_f32) {
      const float* a = static_cast<const float*>(p.aux) + co;
#pragma unroll
      for (int i = 0; i < NC; ++i)
        if (n + i < p.N) v[i] *= dgelu_fast(a[i]);
    } else {
      const __nv_bfloat16* a = static_cast<const __nv_bfloat16*>(p.aux) + co;
      if (full) {
#pragma unroll
        for (int q = 0; q < NC / 8; ++q) {
          float f[8];
          load8_bf16(a + 8 * q, f);
#pragma unroll
          for (int e = 0; e < 8; ++e) v[8 * q + e] *= dgelu_fast(f[e]);
        }
      } else {
#pragma unroll
        for (int i = 0; i < NC; ++i)
          if (n + i < p.N) v[i] *= dgelu_fast(__bfloat162float(a[i]));
      }
    }
  }
  if (p.resid) {
    if (p.c_f32) {
      const float* r = static_cast<const float*>(p.resid) + (int64_t)m * p.ld_resid + n;
#pragma unroll
      for (int i = 0; i < NC; ++i)
        if (n + i < p.N) v[i] += r[i];
    } else {
      const __nv_bfloat16* r = static_cast<const __nv_bfloat16*>(p.resid) + (int64_t)m * p.ld_resid + n;
      if (full) {
#pragma unroll
        for (int q = 0; q < NC / 8; ++q) {
          float f[8];
          load8_bf16(r + 8 * q, f);
#pragma unroll
          for (int e = 0; e < 8; ++e) v[8 * q + e] += f[e];
        }
      } else {
#pragma unroll
        for (int i = 0; i < NC; ++i)
          if (n + i < p.N) v[i] += __bfloat162float(r[i]);
      }
    }
  }
  if (p.c_f32) {
    float* c = static_cast<float*>(p.c) + co;
    if (full) {
#pragma unroll
      for (int q = 0; q < NC / 4; ++q) {
        float4 o = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        if (p.accumulate) {
          const float4 old = reinterpret_cast<const float4*>(c)[q];
          o.x += old.x; o.y += old.y; o.z += old.z; o.w += old.w;
        }
        reinterpret_cast<float4*>(c)[q] = o;
      }
    } else if (inb && p.vec == 2 && !p.accumulate) {
      // rows only 8-byte aligned (e.g. d(mlm.w) with ld = V = 30522)
      if ((reinterpret_cast<uintptr_t>(c) & 15) == 0) {
#pragma unroll
        for (int q = 0; q < NC / 4; ++q)
          reinterpret_cast<float4*>(c)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      } else {
        reinterpret_cast<float2*>(c)[0] = make_float2(v[0], v[1]);
#pragma unroll
        for (int q = 0; q < NC / 4 - 1; ++q)
          reinterpret_cast<float4*>(c + 2)[q] =
              make_float4(v[2 + 4 * q], v[3 + 4 * q], v[4 + 4 * q], v[5 + 4 * q]);
        reinterpret_cast<float2*>(c + NC - 2)[0] = make_float2(v[NC - 2], v[NC - 1]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < NC; ++i)
        if (n + i < p.N) c[i] = p.accumulate ? c[i] + v[i] : v[i];
    }
  } else {
    __nv_bfloat16* c = static_cast<__nv_bfloat16*>(p.c) + co;
    if (full) {
#pragma unroll
      for (int q = 0; q < NC / 8; ++q) store8_bf16(c + 8 * q, v + 8 * q);
    } else {
#pragma unroll
      for (int i = 0; i < NC; ++i)
        if (n + i < p.N) c[i] = __float2bfloat16_rn(v[i]);
    }
  }
}

// ---- coalesced epilogue through a per-warp smem staging buffer ------------
// A warp owns 32 output rows (its TMEM lane quarter) x 32 columns per chunk.
// Thread r holds row r in registers; global traffic instead goes row-segment
// by row-segment (4 or 8 lanes per row, full 64/128-byte segments), through a
// swizzled [32 rows][32 x elem] staging tile that is conflict-free both when a
// thread writes its own row and when a warp reads a row segment.
// Staging tile: 32 rows x 64 bytes (32 bf16, or 16 fp32 = half a chunk).
template <int ES>  // element size: 2 (bf16) or 4 (fp32)
struct Stage {
  static constexpr int RB = 64;        // row bytes
  static constexpr int CPR = 4;        // 16-byte pieces per row
  static constexpr int RPI = 8;        // rows per warp instruction
  static constexpr int NE = 64 / ES;   // elements per staged row (32 or 16)
  __device__ static __forceinline__ int off(int r, int j) {
    return r * RB + ((j ^ ((r >> 1) & 3)) * 16);  // conflict-free both ways
  }
};

// thread `lane` writes its NE values (row lane) into the staging tile
template <int ES>
__device__ __forceinline__ void stage_put(uint8_t* st, int lane, const float* v) {
  if constexpr (ES == 2) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      *reinterpret_cast<uint4*>(st + Stage<2>::off(lane, j)) =
          make_uint4(pack_bf16(v[8 * j], v[8 * j + 1]), pack_bf16(v[8 * j + 2], v[8 * j + 3]),
                     pack_bf16(v[8 * j + 4], v[8 * j + 5]), pack_bf16(v[8 * j + 6], v[8 * j + 7]));
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      *reinterpret_cast<float4*>(st + Stage<4>::off(lane, j)) =
          make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
  }
}
// thread `lane` reads its row back as floats
template <int ES>
__device__ __forceinline__ void stage_get(const uint8_t* st, int lane, float* v) {
  if constexpr (ES == 2) {
#pragma unroll
    for (int j = 0; j < 4; ++j) load8_bf16(reinterpret_cast<const __nv_bfloat16*>(st + Stage<2>::off(lane, j)), v + 8 * j);
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float4 q = *reinterpret_cast<const float4*>(st + Stage<4>::off(lane, j));
      v[4 * j] = q.x; v[4 * j + 1] = q.y; v[4 * j + 2] = q.z; v[4 * j + 3] = q.w;
    }
  }
}
// staging tile -> global rows [row0, row0+32) (rows >= M skipped); mode 0
// store, 1 fp32 vector reduction (split-K), 2 fp32 read-add-store (accumulate)
template <int ES>
__device__ __forceinline__ void stage_store(const uint8_t* st, int lane, char* g0, int64_t ld_bytes,
                                            int rows_left, int mode) {
  using S = Stage<ES>;
#pragma unroll
  for (int i = 0; i < S::CPR; ++i) {
    const int r = i * S::RPI + lane / S::CPR, j = lane % S::CPR;
    if (r < rows_left) {
      const uint4 u = *reinterpret_cast<const uint4*>(st + S::off(r, j));
      char* g = g0 + r * ld_bytes + j * 16;
      if (mode == 0) {
        *reinterpret_cast<uint4*>(g) = u;
      } else if (mode == 1) {
        red_add_v4(reinterpret_cast<float*>(g), __uint_as_float(u.x), __uint_as_float(u.y),
                   __uint_as_float(u.z), __uint_as_float(u.w));
      } else {
        float4 o = *reinterpret_cast<float4*>(g);
        o.x += __uint_as_float(u.x); o.y += __uint_as_float(u.y);
        o.z += __uint_as_float(u.z); o.w += __uint_as_float(u.w);
        *reinterpret_cast<float4*>(g) = o;
      }
    }
  }
}
// global rows -> staging tile (coalesced), for the residual / aux operands
template <int ES>
__device__ __forceinline__ void stage_load(uint8_t* st, int lane, const char* g0, int64_t ld_bytes,
                                           int rows_left) {
  using S = Stage<ES>;
#pragma unroll
  for (int i = 0; i < S::CPR; ++i) {
    const int r = i * S::RPI + lane / S::CPR, j = lane % S::CPR;
    uint4 u = make_uint4(0, 0, 0, 0);
    if (r < rows_left) u = *reinterpret_cast<const uint4*>(g0 + r * ld_bytes + j * 16);
    *reinterpret_cast<uint4*>(st + S::off(r, j)) = u;
  }
}

// 32 register values of row `lane` -> 32 columns of rows [row0, row0+32) at
// g (byte address of the first row's first column), via the staging tile.
__device__ __forceinline__ void staged_out(bool f32, uint8_t* st, int lane, const float* v, char* g,
                                           int64_t ld_bytes, int rows_left, int mode) {
  if (f32) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      stage_put<4>(st, lane, v + 16 * h);
      __syncwarp();
      stage_store<4>(st, lane, g + 64 * h, ld_bytes, rows_left, mode);
      __syncwarp();
    }
  } else {
    stage_put<2>(st, lane, v);
    __syncwarp();
    stage_store<2>(st, lane, g, ld_bytes, rows_left, mode);
    __syncwarp();
  }
}
__device__ __forceinline__ void staged_in(bool f32, uint8_t* st, int lane, float* v, const char* g,
                                          int64_t ld_bytes, int rows_left) {
  if (f32) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      stage_load<4>(st, lane, g + 64 * h, ld_bytes, rows_left);
      __syncwarp();
      stage_get<4>(st, lane, v + 16 * h);
      __syncwarp();
    }
  } else {
    stage_load<2>(st, lane, g, ld_bytes, rows_left);
    __syncwarp();
    stage_get<2>(st, lane, v);
    __syncwarp();
  }
}

// Full 32-column chunk [n, n+32) of the warp's 32 rows starting at row0.
// Preconditions (checked by the caller): n + 32 <= N, p.vec == 1.
__device__ __forceinline__ void epilogue_staged(const Params& p, uint8_t* st, int lane, int row0,
                                                int n, float* v) {
  const int rows_left = p.M - row0;
  const int64_t co0 = p.c_group ? (n / p.c_group) * p.c_gstride + (int64_t)row0 * p.ldc + n % p.c_group
                                : (int64_t)row0 * p.ldc + n;
  const bool f32 = p.c_f32;
  const int cs = f32 ? 4 : 2;
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] *= p.alpha;
  if (p.splits > 1) {
    staged_out(true, st, lane, v, static_cast<char*>(p.c) + co0 * 4, p.ldc * 4, rows_left, 1);
    return;
  }
  if (p.bias) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float4 b = __ldg(reinterpret_cast<const float4*>(p.bias + n) + q);
      v[4 * q] += b.x; v[4 * q + 1] += b.y; v[4 * q + 2] += b.z; v[4 * q + 3] += b.w;
    }
  }
  if (p.act == ACT_GELU) {  // pre-activation to aux (same type and layout as C)
    staged_out(f32, st, lane, v, static_cast<char*>(p.aux) + co0 * cs, p.ldc * cs, rows_left, 0);
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = gelu_fast(v[i]);
  } else if (p.act == ACT_DGELU) {
    float a[32];
    staged_in(f32, st, lane, a, static_cast<const char*>(p.aux) + co0 * cs, p.ldc * cs, rows_left);
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] *= dgelu_fast(a[i]);
  }
  if (p.resid) {
    float r[32];
    const int64_t ro = (int64_t)row0 * p.ld_resid + n;
    staged_in(f32, st, lane, r, static_cast<const char*>(p.resid) + ro * cs, p.ld_resid * cs,
              rows_left);
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] += r[i];
  }
  staged_out(f32, st, lane, v, static_cast<char*>(p.c) + co0 * cs, p.ldc * cs, rows_left,
             f32 && p.accumulate ? 2 : 0);
}

__device__ __forceinline__ void decode_unit(const Params& p, int u, int& m0, int& n0, int& kb0,
                                            int& kb1) {
  const int s = u % p.splits;
  const int r = u / p.splits;
  m0 = (r % p.m_tiles) * BM;
  n0 = (r / p.m_tiles);  // scaled by BN by the caller
  const int num_kb = (p.K + BK - 1) / BK;
  kb0 = s * p.kb_per_split;
  kb1 = min(num_kb, kb0 + p.kb_per_split);
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap map_a,
                   const __grid_constant__ CUtensorMap map_b, const Params p) {
  constexpr uint32_t kBTileBytes = BN * BK * 2;
  constexpr uint32_t kStageBytes = kATileBytes + kBTileBytes;
  constexpr uint32_t kAccStride = BN <= 128 ? 128 : 256;  // TMEM columns per accumulator
  constexpr uint32_t kTmemCols = 2 * kAccStride;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * kStageBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;  // [2]
  uint64_t* tmem_empty = tmem_full + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tmem_full[a], 1);
      mbar_init(&tmem_empty[a], kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      uint32_t it = 0;
      for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
        int m0, nt, kb0, kb1;
        decode_unit(p, u, m0, nt, kb0, kb1);
        const int n0 = nt * BN;
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          mbar_expect_tx(&full[s], kStageBytes);
          uint8_t* sa = smem + s * kStageBytes;
          uint8_t* sb = sa + kATileBytes;
          const int k0 = kb * BK;
          if (p.a_mn) {
            tma_2d(&map_a, &full[s], sa, m0, k0);
            tma_2d(&map_a, &full[s], sa + 8192, m0 + 64, k0);
          } else {
            tma_2d(&map_a, &full[s], sa, k0, m0);
          }
          if (p.b_mn) {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j) {
              if (p.b_grouped)
                tma_3d(&map_b, &full[s], sb + j * 8192, 0, k0, n0 / 64 + j);
              else
                tma_2d(&map_b, &full[s], sb + j * 8192, n0 + 64 * j, k0);
            }
          } else {
            if (p.b_grouped)
              tma_3d(&map_b, &full[s], sb, 0, n0, kb);
            else
              tma_2d(&map_b, &full[s], sb, k0, n0);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // kind::f16 instruction descriptor: D f32, A/B bf16, majors, N>>3, M>>4
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) |
                             (static_cast<uint32_t>(p.a_mn) << 15) |
                             (static_cast<uint32_t>(p.b_mn) << 16) |
                             (static_cast<uint32_t>(BN >> 3) << 17) |
                             (static_cast<uint32_t>(BM >> 4) << 24);
      uint32_t it = 0, lt = 0;
      for (int u = blockIdx.x; u < p.units; u += gridDim.x, ++lt) {
        int m0, nt, kb0, kb1;
        decode_unit(p, u, m0, nt, kb0, kb1);
        const uint32_t as = lt & 1, aph = (lt >> 1) & 1;
        mbar_wait(&tmem_empty[as], aph ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t dacc = tmem_base + as * kAccStride;
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&full[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t sa = smem_u32(smem + s * kStageBytes);
          const uint32_t sb = sa + kATileBytes;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // K-major: 128B rows, 8-row groups 1024B apart, +32B per UMMA_K.
            // MN-major: 64-wide MN atoms 8KB apart (LBO), 8-row K groups
            // 1024B apart (SBO), +16 rows (2048B) per UMMA_K.
            const uint64_t ad = p.a_mn ? umma_desc(sa + k * 2048, 8192, 1024)
                                       : umma_desc(sa + k * 32, 16, 1024);
            const uint64_t bd = p.b_mn ? umma_desc(sb + k * 2048, 8192, 1024)
                                       : umma_desc(sb + k * 32, 16, 1024);
            umma_bf16(dacc, ad, bd, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          }
          umma_commit(&empty[s]);
        }
        umma_commit(&tmem_full[as]);
      }
    }
    __syncwarp();
  } else {
    // epilogue warps 2..17: lane quarter = warp % 4 (the TMEM lanes a warp
    // may access); the tile's 32-column chunks are dealt round-robin to the
    // four warps of a quarter; each chunk is staged through the warp's own
    // 2 KB smem tile for coalesced global traffic
    const int quarter = warp & 3;
    const int slice = (warp - 2) >> 2;
    uint8_t* st = smem + STAGES * kStageBytes + 1024 + (warp - 2) * 2048;
    uint32_t lt = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x, ++lt) {
      int m0, nt, kb0, kb1;
      decode_unit(p, u, m0, nt, kb0, kb1);
      const int n0 = nt * BN;
      const uint32_t as = lt & 1, aph = (lt >> 1) & 1;
      mbar_wait(&tmem_full[as], aph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int row0 = m0 + quarter * 32;
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + as * kAccStride;
#pragma unroll 1
      for (int c0 = slice * 32; c0 < BN; c0 += 128) {
        uint32_t r[32];
        TMEM_LD32(taddr + c0, r);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const int n = n0 + c0;
        if (n < p.N && row0 < p.M) {
          float v[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
          if (n + 32 <= p.N && p.vec == 1)
            epilogue_staged(p, st, lane, row0, n, v);
          else
            epilogue_cols<32>(p, row0 + lane, n, v);
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&tmem_empty[as]);
    }
  }
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(kTmemCols));
  }
}

}  // namespace tc

// ---------------------------------------------------------------- host side
namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    HP_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) fail(HP_ECUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

using MapKey = std::array<uint64_t, 11>;
std::mutex g_map_mu;
std::map<MapKey, CUtensorMap> g_maps;

// rank 2 or 3, dims/strides in elements (bf16), box in elements.
CUtensorMap make_map(const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                     const uint32_t* box) {
  MapKey key{reinterpret_cast<uint64_t>(base), (uint64_t)rank, dims[0], dims[1],
             rank > 2 ? dims[2] : 0, strides[0], rank > 2 ? strides[1] : 0, box[0], box[1],
             rank > 2 ? box[2] : 0, 0};
  std::lock_guard<std::mutex> g(g_map_mu);
  auto it = g_maps.find(key);
  if (it != g_maps.end()) return it->second;
  CUtensorMap m;
  cuuint64_t gd[3] = {dims[0], dims[1], rank > 2 ? dims[2] : 1};
  cuuint64_t gs[2] = {strides[0] * 2, rank > 2 ? strides[1] * 2 : 0};
  cuuint32_t bx[3] = {box[0], box[1], rank > 2 ? box[2] : 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), gd, gs,
                           bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(HP_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  if (g_maps.size() > 4096) g_maps.clear();
  g_maps[key] = m;
  return m;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    HP_CUDA(cudaGetDevice(&dev));
    HP_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  }
  return n;
}

int g_force_bn = 0;
int g_force_splits = 0;

}  // namespace

void gemm_tc_set_bn(int bn) { g_force_bn = bn; }
void gemm_tc_set_splits(int s) { g_force_splits = s; }

bool gemm_tc_supported(const GemmArgs& g) {
  if (g.ab != DType::bf16) return false;
  if (g.M < 1 || g.N < 1 || g.K < 16) return false;
  if (!aligned16(g.a.p) || !aligned16(g.b.p)) return false;
  if (g.a.group) return false;
  // TMA: non-innermost strides multiple of 16 bytes
  if ((g.a.ld * 2) % 16) return false;
  if ((g.b.ld * 2) % 16) return false;
  if (g.b.group && (g.b.group != 64 || (g.b.gstride * 2) % 16)) return false;
  if (g.b.group && g.b.trans && g.K % 64) return false;
  if (g.b.group && !g.b.trans && g.N % 64) return false;
  if (g.c_group && g.c_group % 32) return false;
  if (g.accumulate && g.ct != DType::f32) return false;
  return true;
}

// 1: every output row 16-byte aligned (full vector epilogue); 2: fp32 rows
// only 8-byte aligned (float2 + float4 stores, plain stores only); 0: scalar.
static int epilogue_vec_ok(const GemmArgs& g) {
  const int64_t elem = g.ct == DType::f32 ? 4 : 2;
  if (g.resid && ((g.ld_resid * elem) % 16 || !aligned16(g.resid))) return 0;
  if (g.aux && !aligned16(g.aux)) return 0;
  if (g.c_group && (g.c_gstride * elem) % 16) return 0;
  if (aligned16(g.c) && (g.ldc * elem) % 16 == 0) return 1;
  if (g.ct == DType::f32 && !g.c_group && (reinterpret_cast<uintptr_t>(g.c) & 7) == 0 &&
      g.ldc % 2 == 0)
    return 2;
  return 0;
}

template <int BN>
static void launch_tc(const CUtensorMap& ma, const CUtensorMap& mb, const tc::Params& p,
                      cudaStream_t s) {
  // stages + barriers (1 KB) + 16 epilogue staging tiles (2 KB) + alignment slack
  constexpr size_t smem = tc::STAGES * (tc::kATileBytes + BN * tc::BK * 2) + 1024 +
                          tc::kEpiWarps * 2048 + 1024;
  static bool attr = false;
  if (!attr) {
    HP_CUDA(cudaFuncSetAttribute(tc::gemm_tc_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    attr = true;
  }
  const int grid = std::min(p.units, num_sms());
  tc::gemm_tc_kernel<BN><<<grid, tc::kThreads, smem, s>>>(ma, mb, p);
  HP_CUDA(cudaGetLastError());
  count_launch();
}

void gemm_tc(const GemmArgs& g, cudaStream_t s) {
  if (!gemm_tc_supported(g)) fail(HP_ECONFIG, "gemm_tc: unsupported operand layout");
  const int nsm = num_sms();
  const int m_tiles = (g.M + tc::BM - 1) / tc::BM;
  const int num_kb = (g.K + tc::BK - 1) / tc::BK;
  const bool can_split = g.ct == DType::f32 && !g.bias && !g.act && !g.resid && !g.accumulate;
  // Pick the N tile (and split-K factor) maximising SM-wave efficiency;
  // ties go to the wider tile (more reuse per byte staged).
  int bn = 256, splits = 1;
  double best = -1;
  for (int cand : {256, 192, 128}) {
    if (g.b.group && !g.b.trans && cand % 64) continue;
    const int tiles = m_tiles * ((g.N + cand - 1) / cand);
    int sp = 1;
    if (can_split && tiles < nsm) sp = std::max(1, std::min(nsm / tiles, num_kb / 4));
    const int units = tiles * sp;
    const int waves = (units + nsm - 1) / nsm;
    const double eff = static_cast<double>(units) / (waves * nsm) * (cand == 256 ? 1.0 : cand == 192 ? 0.97 : 0.93);
    if (eff > best + 1e-9) {
      best = eff;
      bn = cand;
      splits = sp;
    }
  }
  if (g_force_bn) bn = g_force_bn;
  if (g_force_splits && can_split) splits = g_force_splits;
  if (!can_split) splits = 1;
  const int kb_per_split = (num_kb + splits - 1) / splits;
  splits = (num_kb + kb_per_split - 1) / kb_per_split;  // no empty splits

  CUtensorMap ma, mb;
  {
    uint64_t dims[2], str[1];
    uint32_t box[2];
    if (g.a.trans) {  // memory [K rows][M cols]
      dims[0] = g.M; dims[1] = g.K; str[0] = g.a.ld; box[0] = 64; box[1] = 64;
    } else {          // memory [M rows][K cols]
      dims[0] = g.K; dims[1] = g.M; str[0] = g.a.ld; box[0] = 64; box[1] = tc::BM;
    }
    ma = make_map(g.a.p, 2, dims, str, box);
  }
  {
    uint64_t dims[3], str[2];
    uint32_t box[3];
    int rank = 2;
    if (!g.b.trans) {  // MN-major: memory [K rows][N cols] (or grouped blocks)
      if (g.b.group) {
        rank = 3;
        dims[0] = 64; dims[1] = g.K; dims[2] = g.N / 64;
        str[0] = g.b.ld; str[1] = g.b.gstride;
        box[0] = 64; box[1] = 64; box[2] = 1;
      } else {
        dims[0] = g.N; dims[1] = g.K; str[0] = g.b.ld; box[0] = 64; box[1] = 64;
      }
    } else {           // K-major: memory [N rows][K cols] (or grouped along K)
      if (g.b.group) {
        rank = 3;
        dims[0] = 64; dims[1] = g.N; dims[2] = g.K / 64;
        str[0] = g.b.ld; str[1] = g.b.gstride;
        box[0] = 64; box[1] = (uint32_t)bn; box[2] = 1;
      } else {
        dims[0] = g.K; dims[1] = g.N; str[0] = g.b.ld; box[0] = 64; box[1] = (uint32_t)bn;
      }
    }
    mb = make_map(g.b.p, rank, dims, str, box);
  }
  tc::Params p;
  p.M = g.M; p.N = g.N; p.K = g.K;
  p.a_mn = g.a.trans ? 1 : 0;
  p.b_mn = g.b.trans ? 0 : 1;
  p.b_grouped = g.b.group ? 1 : 0;
  p.m_tiles = m_tiles;
  p.n_tiles = (g.N + bn - 1) / bn;
  p.splits = splits;
  p.kb_per_split = kb_per_split;
  p.units = m_tiles * p.n_tiles * splits;
  p.c = g.c; p.ldc = g.ldc; p.c_group = g.c_group; p.c_gstride = g.c_gstride;
  p.c_f32 = g.ct == DType::f32;
  p.alpha = g.alpha; p.accumulate = g.accumulate; p.bias = g.bias; p.act = g.act;
  p.aux = g.aux; p.resid = g.resid; p.ld_resid = g.ld_resid;
  p.vec = epilogue_vec_ok(g);
  if (splits > 1) {
    // partial sums are reduced into C: clear the output region first
    if (g.c_group) {
      HP_CUDA(cudaMemsetAsync(g.c, 0, sizeof(float) * (size_t)(g.N / g.c_group) * g.c_gstride, s));
    } else {
      HP_CUDA(cudaMemset2DAsync(g.c, sizeof(float) * g.ldc, 0, sizeof(float) * g.N, g.M, s));
    }
  }
  if (bn == 256)
    launch_tc<256>(ma, mb, p, s);
  else if (bn == 192)
    launch_tc<192>(ma, mb, p, s);
  else
    launch_tc<128>(ma, mb, p, s);
}

}  // namespace hp
