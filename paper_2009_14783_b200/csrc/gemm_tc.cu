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
#include <cstdlib>
#include <map>
#include <mutex>

#include "hp_common.h"
#include "kernels.h"
#include "launch.cuh"
#include "tc_common.cuh"

namespace hp {

namespace tc {

constexpr int BM = 128;
constexpr int BK = 64;  // one 128-byte swizzle row of bf16
constexpr int kEpiWarps = 8;
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr uint32_t kATileBytes = BM * BK * 2;  // 16 KB

struct Params {
  int M, N, K;
  int a_mn;       // A stored MN-major (A^T row-major)
  int b_mn;       // B stored MN-major (row-major K x N)
  int b_grouped;  // B uses the 3-D grouped map (group = 64)
  int a_atoms, b_atoms;  // MN-major operand loaded through the 3-D atom map
  int m_tiles, n_tiles, splits, kb_per_split, units;
  int64_t part_stride;  // > 0: split s stores its own partial at c + s * part_stride (no reduction)
  int rs_kb;            // running-sum kinds: k-blocks per accumulation stint
  void* c;
  int64_t ldc;
  int c_group;  // 32-bit: divided per chunk in the epilogue
  int64_t c_gstride;
  int c_f32;
  float alpha;
  int accumulate;
  const float* bias;
  int act;
  void* aux;
  const void* resid;
  int64_t ld_resid;
  int vec;  // C / aux / resid rows are 16-byte aligned
  int debug;  // profiling only: 0 normal, 1 skip TMA loads, 2 skip MMAs, 3 skip epilogue
  unsigned long long* trace;  // profiling only: CTA 0 clock64 timeline (see kTr*)
};
// trace slots (CTA 0): [0] entry, [1] after prologue sync, [2] exit;
// [16+it] producer got empty slot, [16+256+it] MMA got full stage,
// [16+512+it] MMA committed, [16+768+2*t] epilogue tile t start / +1 end
constexpr int kTrP = 16, kTrF = 16 + 256, kTrC = 16 + 512, kTrE = 16 + 768, kTrSlots = 16 + 768 + 64;
constexpr int kTrX = 900;  // tile 0, warp 2: per chunk [before tcgen05.ld, after wait, after epilogue]
// Profiling hooks (timeline trace, debug bits) exist only in builds with
// HP_GEMM_PROFILE defined (HP_GEMM_PROFILE=1 tools/build_native.py); they cost
// registers the production kernels need.
#ifdef HP_GEMM_PROFILE
constexpr bool kProfile = true;
#else
constexpr bool kProfile = false;
#endif
__device__ __forceinline__ void trace_at(const Params& p, int slot, int lim = 1 << 30) {
  if constexpr (kProfile) {
    if (p.trace && blockIdx.x == 0 && slot < lim) p.trace[slot] = clock64();
  }
}
// per-CTA [start, end] globaltimer (ns) at trace[1024 + 2 * blockIdx.x]
__device__ __forceinline__ void trace_cta(const Params& p, int which) {
  if constexpr (kProfile) {
    if (p.trace) {
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      p.trace[1024 + 2 * blockIdx.x + which] = t;
    }
  }
}
__device__ __forceinline__ bool debug_bit(const Params& p, int bit) {
  if constexpr (kProfile) return (p.debug & bit) != 0;
  return false;
}

// bf16 epilogues use the tanh form of GELU, 0.5 x (1 + tanh(sqrt(2/pi) (x +
// 0.044715 x^3))), on the MUFU tanh unit: |GELU_tanh - GELU_erf| <= 4.8e-4,
// under 1/16 of a bf16 half-ulp where it peaks (x ~ 2.7), at ~6 instructions
// per element instead of ~20 for an erf polynomial.  The backward multiplies
// by the exact derivative of the same tanh form, so gradients stay consistent
// with the loss the forward computed.  (The fp32 engine path keeps exact erf,
// kernels.cu.)
__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float gelu_fast(float x) {
  const float u = x * fmaf(0.0356774081363001f, x * x, 0.7978845608028654f);
  const float hx = 0.5f * x;
  return fmaf(hx, tanh_approx(u), hx);
}
__device__ __forceinline__ float dgelu_fast(float x) {
  const float x2 = x * x;
  const float t = tanh_approx(x * fmaf(0.0356774081363001f, x2, 0.7978845608028654f));
  const float du = fmaf(0.1070322244089f, x2, 0.7978845608028654f);
  const float hx = 0.5f * x;
  return fmaf(hx * fmaf(-t, t, 1.f), du, fmaf(0.5f, t, 0.5f));
}

// fp32 outputs (the fp32 parity path's GEMMs, bf16x6 operands) keep the
// exact erf form, as the oracle and the SIMT kernels do
__device__ __forceinline__ float gelu_exact(float x) {
  return 0.5f * x * (1.f + erff(x * 0.70710678118654752f));
}
__device__ __forceinline__ float dgelu_exact(float x) {
  return 0.5f * (1.f + erff(x * 0.70710678118654752f)) + x * 0.39894228040143268f * expf(-0.5f * x * x);
}
__device__ __forceinline__ float gelu_by(bool exact, float x) { return exact ? gelu_exact(x) : gelu_fast(x); }
__device__ __forceinline__ float dgelu_by(bool exact, float x) { return exact ? dgelu_exact(x) : dgelu_fast(x); }

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
__device__ __forceinline__ void epilogue_cols(const Params& p, int m, int n, float* v, int64_t coff) {
  if (m >= p.M) return;
  const bool inb = n + NC <= p.N;
  const bool full = inb && p.vec == 1;
#pragma unroll
  for (int i = 0; i < NC; ++i) v[i] *= p.alpha;
  const int64_t co = (p.c_group ? (n / p.c_group) * p.c_gstride + (int64_t)m * p.ldc + n % p.c_group
                                : (int64_t)m * p.ldc + n) + coff;
  if (p.splits > 1 && !p.part_stride) {  // split-K partial: reduce into the (zeroed) fp32 output
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
    for (int i = 0; i < NC; ++i) v[i] = gelu_by(p.c_f32, v[i]);
  } else if (p.act == ACT_DGELU) {
    if (p.c_f32) {
      const float* a = static_cast<const float*>(p.aux) + co;
#pragma unroll
      for (int i = 0; i < NC; ++i)
        if (n + i < p.N) v[i] *= dgelu_exact(a[i]);
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

// Staging-tile accesses use explicit shared-space instructions on a 32-bit
// shared address: generic (flat) ld/st here would be ordered behind the
// warp's in-flight global stores, serialising every chunk.
__device__ __forceinline__ void sts128(uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(a)
               : "memory");
  return v;
}
__device__ __forceinline__ void unpack8_bf16(const uint4 u, float* v) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 f = __bfloat1622float2(h[e]);
    v[2 * e] = f.x;
    v[2 * e + 1] = f.y;
  }
}

// thread `lane` writes its NE values (row lane) into the staging tile
template <int ES>
__device__ __forceinline__ void stage_put(uint32_t st, int lane, const float* v) {
  if constexpr (ES == 2) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      sts128(st + Stage<2>::off(lane, j),
             make_uint4(pack_bf16(v[8 * j], v[8 * j + 1]), pack_bf16(v[8 * j + 2], v[8 * j + 3]),
                        pack_bf16(v[8 * j + 4], v[8 * j + 5]), pack_bf16(v[8 * j + 6], v[8 * j + 7])));
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      sts128(st + Stage<4>::off(lane, j),
             make_uint4(__float_as_uint(v[4 * j]), __float_as_uint(v[4 * j + 1]),
                        __float_as_uint(v[4 * j + 2]), __float_as_uint(v[4 * j + 3])));
  }
}
// thread `lane` reads its row back as floats
template <int ES>
__device__ __forceinline__ void stage_get(uint32_t st, int lane, float* v) {
  if constexpr (ES == 2) {
#pragma unroll
    for (int j = 0; j < 4; ++j) unpack8_bf16(lds128(st + Stage<2>::off(lane, j)), v + 8 * j);
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint4 q = lds128(st + Stage<4>::off(lane, j));
      v[4 * j] = __uint_as_float(q.x); v[4 * j + 1] = __uint_as_float(q.y);
      v[4 * j + 2] = __uint_as_float(q.z); v[4 * j + 3] = __uint_as_float(q.w);
    }
  }
}
// staging tile -> global rows [row0, row0+32) (rows >= M skipped); mode 0
// store, 1 fp32 vector reduction (split-K), 2 fp32 read-add-store (accumulate)
template <int ES>
__device__ __forceinline__ void stage_store(uint32_t st, int lane, char* g0, int64_t ld_bytes,
                                            int rows_left, int mode) {
  using S = Stage<ES>;
#pragma unroll
  for (int i = 0; i < S::CPR; ++i) {
    const int r = i * S::RPI + lane / S::CPR, j = lane % S::CPR;
    if (r < rows_left) {
      const uint4 u = lds128(st + S::off(r, j));
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
__device__ __forceinline__ void stage_load(uint32_t st, int lane, const char* g0, int64_t ld_bytes,
                                           int rows_left) {
  using S = Stage<ES>;
#pragma unroll
  for (int i = 0; i < S::CPR; ++i) {
    const int r = i * S::RPI + lane / S::CPR, j = lane % S::CPR;
    uint4 u = make_uint4(0, 0, 0, 0);
    if (r < rows_left) u = *reinterpret_cast<const uint4*>(g0 + r * ld_bytes + j * 16);
    sts128(st + S::off(r, j), u);
  }
}

// 32 register values of row `lane` -> 32 columns of rows [row0, row0+32) at
// g (byte address of the first row's first column), via the staging tile.
__device__ __forceinline__ void staged_out(bool f32, uint32_t st, int lane, const float* v, char* g,
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
__device__ __forceinline__ void staged_in(bool f32, uint32_t st, int lane, float* v, const char* g,
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

// Prefetch of a bf16 [32 rows x 32 cols] operand chunk (the dGELU
// pre-activation or the residual) into registers, coalesced like
// stage_load<2>: lane reads 16-byte piece (lane % 4) of rows i*8 + lane/4.
// Issued one chunk ahead (and for a tile's first chunk before its accumulator
// is ready) so the epilogue never waits on global-load latency.
__device__ __forceinline__ void pre_issue(const char* g0, int64_t ld_bytes, int rows_left, int lane,
                                          uint4 (&q)[4]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = i * 8 + lane / 4, j = lane % 4;
    q[i] = r < rows_left ? __ldg(reinterpret_cast<const uint4*>(g0 + r * ld_bytes + j * 16))
                         : make_uint4(0, 0, 0, 0);
  }
}
// prefetched pieces -> staging tile -> row `lane` (32 bf16, kept packed)
__device__ __forceinline__ void pre_consume(uint32_t st, int lane, const uint4 (&q)[4], uint4 (&row)[4]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) sts128(st + Stage<2>::off(i * 8 + lane / 4, lane % 4), q[i]);
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 4; ++j) row[j] = lds128(st + Stage<2>::off(lane, j));
  __syncwarp();
}

// Epilogue kinds: each kernel instantiation carries only its own path (a
// single kernel with every variant behind runtime flags was ~7.5k SASS
// instructions, and its epilogue warps stalled on instruction fetch).
enum EpiKind : int {
  EK_GENERIC = 0,  // any flags; unaligned / partial chunks via epilogue_cols
  EK_BF16 = 1,     // bf16 C (+ bias) (+ residual, prefetched)
  EK_GELU = 2,     // bf16 C = GELU(acc + bias), pre-activation -> aux
  EK_DGELU = 3,    // bf16 C = acc * GELU'(aux), aux prefetched
  EK_F32 = 4,      // fp32 C (+ bias) (accumulate | split-K reduction), grouped C
  // running-sum variants (Params::rs_kb): the unit's K range in stints of
  // rs_kb k-blocks, each its own accumulation chain, summed in stint order in
  // fp32 (round-to-nearest) in a third TMEM region, then the EK_F32 /
  // EK_GENERIC epilogue -- the bf16x6 fp32 path without partials in HBM
  EK_F32_RS = 5,
  EK_GENERIC_RS = 6,
};

// Full 32-column chunk [n, n+32) of the warp's 32 rows starting at row0.
// Preconditions (checked by the caller): n + 32 <= N, p.vec == 1.  `pre`:
// the prefetched aux (pre_kind 1, dGELU) or residual (pre_kind 2) chunk.
template <int EK>
__device__ __forceinline__ void epilogue_staged(const Params& p, uint32_t st, int lane, int row0,
                                                int n, float* v, const uint4 (&pre)[4], int pre_kind,
                                                int64_t coff) {
  constexpr bool kAnyF32 = EK == EK_GENERIC || EK == EK_F32;
  const int rows_left = p.M - row0;
  int64_t co0 = (int64_t)row0 * p.ldc + n;
  if constexpr (kAnyF32) {
    if (p.c_group) co0 = (n / p.c_group) * p.c_gstride + (int64_t)row0 * p.ldc + n % p.c_group;
    co0 += coff;
  }
  const bool f32 = EK == EK_F32 || (EK == EK_GENERIC && p.c_f32);
  const int cs = f32 ? 4 : 2;
  if (p.alpha != 1.f) {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] *= p.alpha;
  }
  if constexpr (kAnyF32) {
    if (p.splits > 1 && !p.part_stride) {
      staged_out(true, st, lane, v, static_cast<char*>(p.c) + co0 * 4, p.ldc * 4, rows_left, 1);
      return;
    }
  }
  if constexpr (EK != EK_DGELU) {
    if (p.bias) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 b = __ldg(reinterpret_cast<const float4*>(p.bias + n) + q);
        v[4 * q] += b.x; v[4 * q + 1] += b.y; v[4 * q + 2] += b.z; v[4 * q + 3] += b.w;
      }
    }
  }
  if (EK == EK_GELU || (EK == EK_GENERIC && p.act == ACT_GELU)) {
    // pre-activation to aux (same type and layout as C)
    staged_out(f32, st, lane, v, static_cast<char*>(p.aux) + co0 * cs, p.ldc * cs, rows_left, 0);
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = gelu_by(EK == EK_GENERIC && p.c_f32, v[i]);
  } else if (EK == EK_DGELU || (EK == EK_GENERIC && p.act == ACT_DGELU)) {
    if (EK == EK_DGELU || pre_kind == 1) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float f[8];
        unpack8_bf16(pre[j], f);
#pragma unroll
        for (int e = 0; e < 8; ++e) v[8 * j + e] *= dgelu_fast(f[e]);
      }
    } else if constexpr (EK == EK_GENERIC) {
      float a[32];
      staged_in(f32, st, lane, a, static_cast<const char*>(p.aux) + co0 * cs, p.ldc * cs, rows_left);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] *= dgelu_by(p.c_f32, a[i]);
    }
  }
  if constexpr (EK == EK_BF16 || EK == EK_GENERIC) {
    if (p.resid) {
      if (pre_kind == 2) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float f[8];
          unpack8_bf16(pre[j], f);
#pragma unroll
          for (int e = 0; e < 8; ++e) v[8 * j + e] += f[e];
        }
      } else if constexpr (EK == EK_GENERIC) {
        float r[32];
        const int64_t ro = (int64_t)row0 * p.ld_resid + n;
        staged_in(f32, st, lane, r, static_cast<const char*>(p.resid) + ro * cs, p.ld_resid * cs,
                  rows_left);
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] += r[i];
      }
    }
  }
  int mode = 0;
  if constexpr (kAnyF32) mode = f32 && p.accumulate ? 2 : 0;
  staged_out(f32, st, lane, v, static_cast<char*>(p.c) + co0 * cs, p.ldc * cs, rows_left, mode);
}

__device__ __forceinline__ void decode_unit(const Params& p, int u, int mt_rows, int& m0, int& n0,
                                            int& kb0, int& kb1) {
  const int s = u % p.splits;
  const int r = u / p.splits;
  m0 = (r % p.m_tiles) * mt_rows;
  n0 = (r / p.m_tiles);  // scaled by BN by the caller
  const int num_kb = (p.K + BK - 1) / BK;
  kb0 = s * p.kb_per_split;
  kb1 = min(num_kb, kb0 + p.kb_per_split);
}

// Shared-memory plan of one (BN, CG) instantiation: as many pipeline stages
// as fit next to the barriers and the epilogue staging tiles (4 for a 128x256
// tile, 6 for 128x128 or a CTA pair's 128x128 half of 256x256).
constexpr int kSmemBudget = 232448;  // 227 KB opt-in per CTA
constexpr int kEpiStageBytes = 2048;  // per epilogue warp
template <int BN, int CG>
struct Tile {
  static constexpr int BNL = BN / CG;  // B columns staged by this CTA
  static constexpr uint32_t kBTileBytes = BNL * BK * 2;
  static constexpr uint32_t kStageBytes = kATileBytes + kBTileBytes;
  static constexpr int kFit = (kSmemBudget - 2048 - kEpiWarps * kEpiStageBytes) / kStageBytes;
  static constexpr int kStages = kFit < 8 ? kFit : 8;
  static constexpr size_t kSmem = kStages * kStageBytes + 1024 + kEpiWarps * kEpiStageBytes + 1024;
  static_assert(kStages >= 3, "pipeline too shallow");
  static_assert(kSmem <= kSmemBudget, "smem plan over budget");
};


// CG = 1: one CTA computes a 128 x BN tile.
// CG = 2: a CTA pair (cluster of 2 on one TPC) computes a 256 x BN tile with
//   tcgen05.mma.cta_group::2 (UMMA M = 256) issued by the leader; each CTA
//   stages its own 128 rows of A and half (BN/2 columns) of B, so per-SM smem
//   traffic per FLOP drops by a third.  Both CTAs' TMA complete on the
//   leader's full barrier; commits multicast to both CTAs' empty / tmem_full
//   barriers; both CTAs' epilogues release the leader's tmem_empty barrier.
template <int BN, int CG, int EK>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap map_a,
                   const __grid_constant__ CUtensorMap map_b, const Params p) {
  using TL = Tile<BN, CG>;
  constexpr int BNL = TL::BNL;
  constexpr int STAGES = TL::kStages;
  constexpr uint32_t kStageBytes = TL::kStageBytes;
  constexpr bool kRS = EK == EK_F32_RS || EK == EK_GENERIC_RS;
  constexpr int EKB = EK == EK_F32_RS ? EK_F32 : (EK == EK_GENERIC_RS ? EK_GENERIC : EK);
  static_assert(!kRS || BN == 128, "running-sum kinds use 128-wide tiles");
  constexpr uint32_t kAccStride = BN <= 128 ? 128 : 256;  // TMEM columns per accumulator
  // two accumulators (+ the running sum at column 256 for the RS kinds)
  constexpr uint32_t kTmemCols = kRS ? 512 : 2 * kAccStride;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * kStageBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;  // [2]
  uint64_t* tmem_empty = tmem_full + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    trace_at(p, 0);
    trace_cta(p, 0);
  }
  constexpr int kClu = CG;  // CTAs per cluster
  const uint32_t rank = kClu > 1 ? cluster_rank() : 0;
  const uint32_t row_rank = CG == 2 ? rank : 0;  // which 128 rows of the tile this CTA owns
  const int unit0 = blockIdx.x / kClu, unit_step = gridDim.x / kClu;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tmem_full[a], 1);
      mbar_init(&tmem_empty[a], CG * kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
  }
  if (warp == 1) {
    if constexpr (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if constexpr (kClu > 1) cluster_sync_all();  // peer barriers initialised before use
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) trace_at(p, 1);

  // Work units: static striding, unit u = blockIdx / CG + i * (gridDim / CG).
  // (A dynamic scheduler -- units claimed from a global counter one unit
  // ahead and handed to the MMA / epilogue warps and the peer CTA through an
  // smem ring -- was measured and removed: ~1 us slower per launch at N=1
  // and no gain at N=4 under concurrent NCCL rings.)
  auto take_unit = [&](uint32_t i) -> int {
    const int u = unit0 + static_cast<int>(i) * unit_step;
    return u < p.units ? u : -1;
  };

  if (warp == 0) {
    // TMA producer (whole warp walks the ring, one elected lane issues).  An
    // MN-major operand tile is BNL/64 (or 2 for A) 8 KB swizzle atoms; with
    // the 3-D "atom" map (64 cols, K, col-block) it is ONE bulk-tensor load.
    uint32_t it = 0;
    for (uint32_t ui = 0;; ++ui) {
      const int u = take_unit(ui);
      if (u < 0) break;
      int m0, nt, kb0, kb1;
      decode_unit(p, u, BM * CG, m0, nt, kb0, kb1);
      const int am0 = m0 + static_cast<int>(row_rank) * BM;       // this CTA's A rows
      const int bn0 = nt * BN + static_cast<int>(row_rank) * BNL;  // this CTA's B columns
      for (int kb = kb0; kb < kb1; ++kb, ++it) {
        const int s = it % STAGES;
        const uint32_t ph = (it / STAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        if (lane == 0) trace_at(p, kTrP + it, kTrF);
        uint8_t* sa = smem + s * kStageBytes;
        uint8_t* sb = sa + kATileBytes;
        const int k0 = kb * BK;
        if (elect_one()) {
          if (debug_bit(p, 1)) {  // profiling mode: no loads, MMA on stale smem
            if (CG == 1 || rank == 0) mbar_arrive(&full[s]);
          } else if constexpr (CG == 1) {
            uint64_t* bar = &full[s];
            mbar_expect_tx(bar, kStageBytes);
            if (!p.a_mn) tma_2d(&map_a, bar, sa, k0, am0);
            else if (p.a_atoms) tma_3d(&map_a, bar, sa, 0, k0, am0 / 64);
            else {
              tma_2d(&map_a, bar, sa, am0, k0);
              tma_2d(&map_a, bar, sa + 8192, am0 + 64, k0);
            }
            if (!p.b_mn) {
              if (p.b_grouped) tma_3d(&map_b, bar, sb, 0, bn0, kb);
              else tma_2d(&map_b, bar, sb, k0, bn0);
            } else if (p.b_atoms) {
              tma_3d(&map_b, bar, sb, 0, k0, bn0 / 64);
            } else {
#pragma unroll
              for (int j = 0; j < BNL / 64; ++j) tma_2d(&map_b, bar, sb + j * 8192, bn0 + 64 * j, k0);
            }
          } else {
            // both CTAs' bytes land on the leader's full barrier
            if (rank == 0) mbar_expect_tx(&full[s], 2 * kStageBytes);
            const uint32_t bar = mapa_shared(smem_u32(&full[s]), 0);
            if (!p.a_mn) tma_2d_cg2(&map_a, bar, sa, k0, am0);
            else if (p.a_atoms) tma_3d_cg2(&map_a, bar, sa, 0, k0, am0 / 64);
            else {
              tma_2d_cg2(&map_a, bar, sa, am0, k0);
              tma_2d_cg2(&map_a, bar, sa + 8192, am0 + 64, k0);
            }
            if (!p.b_mn) {
              if (p.b_grouped) tma_3d_cg2(&map_b, bar, sb, 0, bn0, kb);
              else tma_2d_cg2(&map_b, bar, sb, k0, bn0);
            } else if (p.b_atoms) {
              tma_3d_cg2(&map_b, bar, sb, 0, k0, bn0 / 64);
            } else {
#pragma unroll
              for (int j = 0; j < BNL / 64; ++j) tma_2d_cg2(&map_b, bar, sb + j * 8192, bn0 + 64 * j, k0);
            }
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    // The whole warp walks the pipeline (so every value feeding tcgen05.mma is
    // warp-uniform); one elected lane issues the MMAs and their commit.
    if (CG == 1 || rank == 0) {  // CG 2: the leader issues the pair's MMAs
      // kind::f16 instruction descriptor: D f32, A/B bf16, majors, N>>3, M>>4
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) |
                             (static_cast<uint32_t>(p.a_mn) << 15) |
                             (static_cast<uint32_t>(p.b_mn) << 16) |
                             (static_cast<uint32_t>(BN >> 3) << 17) |
                             (static_cast<uint32_t>((BM * CG) >> 4) << 24);
      // Descriptors of stage 0, k-step 0; stage s / k-step k add plain offsets
      // to the 14-bit start-address field (smem < 256 KB: no carry out).
      // K-major: 128B rows, 8-row groups 1024B apart, +32B per UMMA_K.
      // MN-major: 64-wide MN atoms 8KB apart (LBO), 8-row K groups 1024B
      // apart (SBO), +16 rows (2048B) per UMMA_K.
      const uint32_t s0 = smem_u32(smem);
      const uint64_t da0 = umma_desc(s0, p.a_mn ? 8192 : 16, 1024);
      const uint64_t db0 = umma_desc(s0 + kATileBytes, p.b_mn ? 8192 : 16, 1024);
      const uint64_t dak = p.a_mn ? (2048 >> 4) : (32 >> 4);
      const uint64_t dbk = p.b_mn ? (2048 >> 4) : (32 >> 4);
      uint32_t it = 0, lt = 0;  // lt: accumulation stints (one per unit unless kRS)
      for (uint32_t ui = 0;; ++ui) {
        const int u = take_unit(ui);
        if (u < 0) break;
        int m0, nt, kb0, kb1;
        decode_unit(p, u, BM * CG, m0, nt, kb0, kb1);
        const int kbs = kRS ? p.rs_kb : kb1 - kb0;
        for (int sb = kb0; sb < kb1; sb += kbs, ++lt) {
        const int se = min(kb1, sb + kbs);
        const uint32_t as = lt & 1, aph = (lt >> 1) & 1;
        mbar_wait(&tmem_empty[as], aph ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t dacc = tmem_base + as * kAccStride;
        for (int kb = sb; kb < se; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&full[s], ph);
          if (lane == 0) trace_at(p, kTrF + it, kTrC);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t soff = static_cast<uint64_t>(s) * (kStageBytes >> 4);
          if (elect_one()) {
            if (!debug_bit(p, 2)) {
#pragma unroll
              for (int k = 0; k < BK / 16; ++k) {
                const uint64_t ad = da0 + soff + k * dak, bd = db0 + soff + k * dbk;
                if constexpr (CG == 2)
                  umma_bf16_cg2(dacc, ad, bd, idesc, (kb > sb || k > 0) ? 1u : 0u);
                else
                  umma_bf16(dacc, ad, bd, idesc, (kb > sb || k > 0) ? 1u : 0u);
              }
            }
            if constexpr (CG == 2) umma_commit_cg2(&empty[s]);
            else umma_commit(&empty[s]);
          }
          __syncwarp();
          if (lane == 0) trace_at(p, kTrC + it, kTrE);
        }
        if (elect_one()) {
          if constexpr (CG == 2) umma_commit_cg2(&tmem_full[as]); else umma_commit(&tmem_full[as]);
        }
        __syncwarp();
        }
      }
    }
  } else {
    // epilogue warps 2..kEpiWarps+1: lane quarter = warp % 4 (the TMEM lanes
    // a warp may access); a quarter's 32-column chunks are dealt round-robin
    // to its kEpiWarps/4 warps; each chunk is staged through the warp's own
    // 2 KB smem tile for coalesced global traffic.
    constexpr int kChunkStep = 32 * (kEpiWarps / 4);
    const int ew = warp - 2;
    const int quarter = warp & 3;
    const int first = (ew >> 2) * 32;
    const uint32_t st = smem_u32(smem + STAGES * kStageBytes + 1024 + ew * kEpiStageBytes);
    // operand prefetched a chunk ahead: 1 = dGELU pre-activation, 2 = residual
    int pre_kind = 0;
    if constexpr (EKB == EK_DGELU) pre_kind = 1;
    if constexpr (EKB == EK_BF16) pre_kind = p.resid ? 2 : 0;
    if constexpr (EKB == EK_GENERIC)
      pre_kind = (!p.c_f32 && p.vec == 1 && p.splits == 1) ? (p.act == ACT_DGELU ? 1 : (p.resid ? 2 : 0)) : 0;
    const char* pre_base = static_cast<const char*>(pre_kind == 1 ? p.aux : p.resid);
    const int64_t pre_ld = pre_kind == 1 ? p.ldc : p.ld_resid;
    uint32_t lt = 0;  // accumulation stints, as the MMA warp counts them
    const uint32_t empty_leader[2] = {CG == 2 ? mapa_shared(smem_u32(&tmem_empty[0]), 0) : 0u,
                                      CG == 2 ? mapa_shared(smem_u32(&tmem_empty[1]), 0) : 0u};
    const uint32_t rsum = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + 2 * kAccStride;
    for (uint32_t ui = 0;; ++ui) {
      const int u = take_unit(ui);
      if (u < 0) break;
      int m0, nt, kb0, kb1;
      decode_unit(p, u, BM * CG, m0, nt, kb0, kb1);
      const int n0 = nt * BN;
      const int nst = kRS ? (kb1 - kb0 + p.rs_kb - 1) / p.rs_kb : 1;
      // RS kinds: stints 0 .. nst-2 fold into the running sum, the last one
      // finishes it and runs the epilogue
      for (int j = 0; j + 1 < nst; ++j, ++lt) {
        if constexpr (kRS) {
          const uint32_t as = lt & 1, aph = (lt >> 1) & 1;
          mbar_wait(&tmem_full[as], aph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + as * kAccStride;
#pragma unroll 1
          for (int c = first; c < BN; c += kChunkStep) {
            uint32_t r[32];
            TMEM_LD32(taddr + c, r);
            if (j > 0) {
              uint32_t q[32];
              TMEM_LD32(rsum + c, q);
              asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
              for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(q[i]) + __uint_as_float(r[i]));
            } else {
              asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            }
            TMEM_ST32(rsum + c, r);
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            if constexpr (CG == 2)
              mbar_arrive_cluster(empty_leader[as]);
            else
              mbar_arrive(&tmem_empty[as]);
          }
        }
      }
      const uint32_t as = lt & 1, aph = (lt >> 1) & 1;
      const int row0 = m0 + static_cast<int>(row_rank) * BM + quarter * 32;
      const int rows_left = p.M - row0;
      // chunk at tile column c takes the staged path with a prefetched operand
      auto pre_ok = [&](int c) { return pre_kind != 0 && c < BN && n0 + c + 32 <= p.N && rows_left > 0; };
      auto pre_src = [&](int c) {
        const int n = n0 + c;
        const int64_t o = (EK == EK_GENERIC && pre_kind == 1 && p.c_group)
                              ? (n / p.c_group) * p.c_gstride + (int64_t)row0 * p.ldc + n % p.c_group
                              : (int64_t)row0 * pre_ld + n;
        return pre_base + o * 2;
      };
      uint4 cur[4], nxt[4];
      if (pre_ok(first)) pre_issue(pre_src(first), pre_ld * 2, rows_left, lane, cur);
      mbar_wait(&tmem_full[as], aph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (warp == 2 && lane == 0) trace_at(p, kTrE + 2 * lt, kTrSlots);
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + as * kAccStride;
#pragma unroll 1
      for (int c = first; c < BN; c += kChunkStep) {
        if (pre_ok(c + kChunkStep)) pre_issue(pre_src(c + kChunkStep), pre_ld * 2, rows_left, lane, nxt);
        const bool tr = kProfile && warp == 2 && lane == 0 && lt == 0;
        const int tslot = kTrX + 3 * ((c - first) / kChunkStep);
        if (tr) trace_at(p, tslot, 1024);
        uint32_t r[32];
        TMEM_LD32(taddr + c, r);
        if (kRS && nst > 1) {
          uint32_t q[32];
          TMEM_LD32(rsum + c, q);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(q[i]) + __uint_as_float(r[i]));
        } else {
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        }
        if (tr) trace_at(p, tslot + 1, 1024);
        const int n = n0 + c;
        if (n < p.N && rows_left > 0 && !debug_bit(p, 4)) {
          float v[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
          // specialised kinds are only launched with N % 32 == 0, vec == 1
          if (EKB != EK_GENERIC || (n + 32 <= p.N && p.vec == 1)) {
            uint4 pre[4];
            if (pre_kind) pre_consume(st, lane, cur, pre);
            epilogue_staged<EKB>(p, st, lane, row0, n, v, pre, pre_kind,
                                 p.part_stride ? (u % p.splits) * p.part_stride : 0);
          } else if constexpr (EKB == EK_GENERIC) {
            epilogue_cols<32>(p, row0 + lane, n, v, p.part_stride ? (u % p.splits) * p.part_stride : 0);
          }
        }
        if (tr) trace_at(p, tslot + 2, 1024);
#pragma unroll
        for (int i = 0; i < 4; ++i) cur[i] = nxt[i];
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (warp == 2 && lane == 0) trace_at(p, kTrE + 2 * lt + 1, kTrSlots);
      if (lane == 0) {
        if constexpr (CG == 2)
          mbar_arrive_cluster(empty_leader[as]);
        else
          mbar_arrive(&tmem_empty[as]);
      }
      ++lt;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    trace_at(p, 2);
    trace_cta(p, 1);
  }
  // both CTAs done before the pair frees TMEM
  if constexpr (kClu > 1) cluster_sync_all();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if constexpr (CG == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"(kTmemCols));
    else
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

}  // namespace

// rank 2 or 3, dims/strides in elements (bf16), box in elements; cached by
// (base, shape, box) -- tensor maps are built on the host once per operand.
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

namespace {

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

int g_sm_budget = 0;  // 0: every SM (gemm_tc_set_sm_budget)
int num_sms_hw();
int num_sms() {
  const int n = num_sms_hw();
  return g_sm_budget > 0 ? std::min(n, g_sm_budget) : n;
}
int num_sms_hw() {
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
int g_debug_mode = 0;
unsigned long long* g_trace = nullptr;

}  // namespace

void gemm_tc_set_bn(int bn) { g_force_bn = bn; }
void gemm_tc_set_sm_budget(int n) { g_sm_budget = n; }
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

template <int BN, int CG, int EK>
static void launch_tc(const CUtensorMap& ma, const CUtensorMap& mb, const tc::Params& p,
                      cudaStream_t s) {
  // stages + barriers (1 KB) + epilogue staging tiles + alignment slack
  constexpr size_t smem = tc::Tile<BN, CG>::kSmem;
  static bool attr = false;
  if (!attr) {
    HP_CUDA(cudaFuncSetAttribute(tc::gemm_tc_kernel<BN, CG, EK>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  const int grid = CG * std::min(p.units, num_sms() / CG);
  launch_ex(tc::gemm_tc_kernel<BN, CG, EK>, dim3(grid), dim3(tc::kThreads), smem, s,
             CG, ma, mb, p);
  HP_CUDA(cudaGetLastError());
  count_launch();
}

namespace {
int g_force_cg = 0;
int g_generic_only = 0;

}
void gemm_tc_set_generic(int on) { g_generic_only = on; }

template <int EK>
static void launch_ek(int cg, int bn, const CUtensorMap& ma, const CUtensorMap& mb,
                      const tc::Params& p, cudaStream_t s) {
  if (cg == 2) {
    if (bn == 256) launch_tc<256, 2, EK>(ma, mb, p, s);
    else if (bn == 192) launch_tc<192, 2, EK>(ma, mb, p, s);
    else launch_tc<128, 2, EK>(ma, mb, p, s);
  } else {
    if (bn == 256) launch_tc<256, 1, EK>(ma, mb, p, s);
    else if (bn == 192) launch_tc<192, 1, EK>(ma, mb, p, s);
    else launch_tc<128, 1, EK>(ma, mb, p, s);
  }
}
void gemm_tc_set_cg(int cg) { g_force_cg = cg; }
void gemm_tc_set_debug(int mode) { g_debug_mode = mode; }
void gemm_tc_set_trace(unsigned long long* buf) { g_trace = buf; }

void gemm_tc(const GemmArgs& g, cudaStream_t s) {
  if (!gemm_tc_supported(g)) fail(HP_ECONFIG, "gemm_tc: unsupported operand layout");
  const int nsm = num_sms();
  const int num_kb = (g.K + tc::BK - 1) / tc::BK;
  const bool can_split = g.ct == DType::f32 && !g.bias && !g.act && !g.resid && !g.accumulate;
  // Pick (CTA group, N tile, split-K) maximising SM-wave efficiency weighted
  // by the tile's operand reuse: a CTA pair with a 256-wide tile stages the
  // fewest bytes per FLOP, one CTA with a 128-wide tile the most.
  int bn = 256, cg = 2, splits = 1;
  double best = -1;
  // (weights ~ FLOP per staged byte: 128 / 87 / 87 / 77 / 65).  A CTA pair
  // with a 256 x 192 tile (K-major B only) exists for forced use; measured
  // slower than one CTA's 128 x 192 on the N = 768 data gradients (dX 18.5 vs
  // 16.5 us, dX1 20.6 vs 19.9), so it is not a heuristic candidate.
  const int cands[5][3] = {{2, 256, 118}, {2, 128, 100}, {1, 256, 100}, {1, 192, 97}, {1, 128, 90}};
  for (const auto& c : cands) {
    const int ccg = c[0], cbn = c[1];
    if (g_force_cg && ccg != g_force_cg) continue;
    if (g_force_bn && cbn != g_force_bn) continue;
    if (g.rs_kc > 0 && cbn != 128) continue;  // running sum: a third 128-column TMEM region
    if (g.b.group && !g.b.trans && (cbn / ccg) % 64) continue;
    // a 96-column half of B per CTA: only as a K-major operand (rows of the
    // box); an MN-major B tile is whole 64-column swizzle atoms
    if (!g.b.trans && (cbn / ccg) % 64) continue;
    const int mt = (g.M + tc::BM * ccg - 1) / (tc::BM * ccg);
    const int tiles = mt * ((g.N + cbn - 1) / cbn);
    const int slots = nsm / ccg;
    int sp = 1;
    if (can_split && tiles < slots) sp = std::max(1, std::min(slots / tiles, num_kb / 4));
    if (g.part_chunks > 1) sp = g.part_chunks;  // chunk partials: the split count is given
    // at most two K halves: their fp32 partials reduce into the zeroed output
    // in either order to the same bits (a + b == b + a), so every GEMM of the
    // step is run-to-run deterministic; deeper splits would not be
    if (g.part_chunks <= 1) sp = std::min(sp, 2);
    if (g.max_splits > 0) sp = std::min(sp, g.max_splits);
    const int units = tiles * sp;
    const int waves = (units + slots - 1) / slots;
    const double eff = static_cast<double>(units) / (waves * slots) * c[2] / 100.0;
    if (eff > best + 1e-9) {
      best = eff;
      bn = cbn;
      cg = ccg;
      splits = sp;
    }
  }
  if (g_force_splits && can_split) splits = g_force_splits;
  if (!can_split || g.rs_kc > 0) splits = 1;
  const int m_tiles = (g.M + tc::BM * cg - 1) / (tc::BM * cg);
  int kb_per_split = (num_kb + splits - 1) / splits;
  if (g.part_chunks > 1) {  // chunk partials: K-chunk boundaries as given
    if (!can_split || g.part_kc % tc::BK || g.max_splits == 1)
      fail(HP_ECONFIG, "gemm_tc: K-chunk partials need an fp32 C without epilogue, part_kc % 64 == 0");
    kb_per_split = g.part_kc / tc::BK;
  }
  splits = (num_kb + kb_per_split - 1) / kb_per_split;  // no empty splits
  if (g.part_chunks > 1 && splits != g.part_chunks)
    fail(HP_ECONFIG, "gemm_tc: K-chunk count does not match K / part_kc");
  const int bnl = bn / cg;  // B columns per CTA

  // MN-major operands: "atom" maps view the row-major [K][MN] matrix as
  // (64 cols, K rows, MN/64 col-blocks) so one box brings every 8 KB swizzle
  // atom of a tile.  The last col-block may read past column MN (garbage in
  // discarded output rows / cols) but never past the row pitch.
  const int a_blocks = (g.M + 63) / 64, b_blocks = (g.N + 63) / 64;
  const bool a_atoms = g.a.trans && 64LL * a_blocks <= g.a.ld;
  const bool b_atoms = !g.b.trans && (g.b.group || 64LL * b_blocks <= g.b.ld);
  CUtensorMap ma, mb;
  {
    uint64_t dims[3], str[2];
    uint32_t box[3];
    int rank = 2;
    if (g.a.trans && a_atoms) {  // memory [K rows][M cols], atom view
      rank = 3;
      dims[0] = 64; dims[1] = g.K; dims[2] = a_blocks;
      str[0] = g.a.ld; str[1] = 64;
      box[0] = 64; box[1] = 64; box[2] = tc::BM / 64;
    } else if (g.a.trans) {
      dims[0] = g.M; dims[1] = g.K; str[0] = g.a.ld; box[0] = 64; box[1] = 64;
    } else {          // memory [M rows][K cols]
      dims[0] = g.K; dims[1] = g.M; str[0] = g.a.ld; box[0] = 64; box[1] = tc::BM;
    }
    ma = make_map(g.a.p, rank, dims, str, box);
  }
  {
    uint64_t dims[3], str[2];
    uint32_t box[3];
    int rank = 2;
    if (!g.b.trans) {  // MN-major: memory [K rows][N cols] (or grouped blocks)
      rank = 3;
      box[0] = 64; box[1] = 64; box[2] = (uint32_t)(bnl / 64);
      if (g.b.group) {
        dims[0] = 64; dims[1] = g.K; dims[2] = g.N / 64;
        str[0] = g.b.ld; str[1] = g.b.gstride;
      } else if (b_atoms) {
        dims[0] = 64; dims[1] = g.K; dims[2] = b_blocks;
        str[0] = g.b.ld; str[1] = 64;
      } else {
        rank = 2;
        dims[0] = g.N; dims[1] = g.K; str[0] = g.b.ld; box[0] = 64; box[1] = 64;
      }
    } else {           // K-major: memory [N rows][K cols] (or grouped along K)
      if (g.b.group) {
        rank = 3;
        dims[0] = 64; dims[1] = g.N; dims[2] = g.K / 64;
        str[0] = g.b.ld; str[1] = g.b.gstride;
        box[0] = 64; box[1] = (uint32_t)bnl; box[2] = 1;
      } else {
        dims[0] = g.K; dims[1] = g.N; str[0] = g.b.ld; box[0] = 64; box[1] = (uint32_t)bnl;
      }
    }
    mb = make_map(g.b.p, rank, dims, str, box);
  }
  tc::Params p;
  p.M = g.M; p.N = g.N; p.K = g.K;
  p.a_mn = g.a.trans ? 1 : 0;
  p.b_mn = g.b.trans ? 0 : 1;
  p.b_grouped = g.b.group ? 1 : 0;
  p.a_atoms = a_atoms ? 1 : 0;
  p.b_atoms = b_atoms ? 1 : 0;
  p.m_tiles = m_tiles;
  p.n_tiles = (g.N + bn - 1) / bn;
  p.splits = splits;
  p.kb_per_split = kb_per_split;
  p.units = m_tiles * p.n_tiles * splits;
  p.part_stride = g.part_chunks > 1 ? g.part_stride : 0;
  p.rs_kb = g.rs_kc > 0 ? g.rs_kc / tc::BK : 0;
  if (g.rs_kc > 0 && (g.rs_kc % tc::BK || g.ct != DType::f32 || bn != 128))
    fail(HP_ECONFIG, "gemm_tc: running-sum stints need fp32 C, 128-wide tiles, rs_kc % 64 == 0");
  p.c = g.c; p.ldc = g.ldc; p.c_group = static_cast<int>(g.c_group); p.c_gstride = g.c_gstride;
  p.c_f32 = g.ct == DType::f32;
  p.alpha = g.alpha; p.accumulate = g.accumulate; p.bias = g.bias; p.act = g.act;
  p.aux = g.aux; p.resid = g.resid; p.ld_resid = g.ld_resid;
  p.vec = epilogue_vec_ok(g);
  p.debug = g_debug_mode;
  p.trace = g_trace;

  if (splits > 1 && !p.part_stride) {
    // partial sums are reduced into C: clear the output region first
    if (g.c_group) {
      HP_CUDA(cudaMemsetAsync(g.c, 0, sizeof(float) * (size_t)(g.N / g.c_group) * g.c_gstride, s));
    } else {
      HP_CUDA(cudaMemset2DAsync(g.c, sizeof(float) * g.ldc, 0, sizeof(float) * g.N, g.M, s));
    }
  }
  // epilogue kind (see tc::EpiKind); specialised kinds need whole 32-column
  // chunks and 16-byte aligned rows
  int ek = tc::EK_GENERIC;
  if (p.vec == 1 && g.N % 32 == 0 && !g_generic_only) {
    if (g.ct == DType::bf16 && !g.c_group && splits == 1) {
      if (g.act == ACT_NONE) ek = tc::EK_BF16;
      else if (g.act == ACT_GELU && !g.resid) ek = tc::EK_GELU;
      else if (g.act == ACT_DGELU && !g.resid && !g.bias) ek = tc::EK_DGELU;
    } else if (g.ct == DType::f32 && g.act == ACT_NONE && !g.resid) {
      ek = tc::EK_F32;
    }
  }
  if (p.rs_kb > 0) ek = ek == tc::EK_F32 ? tc::EK_F32_RS : tc::EK_GENERIC_RS;
  switch (ek) {
    case tc::EK_F32_RS:
      if (cg == 2) launch_tc<128, 2, tc::EK_F32_RS>(ma, mb, p, s); else launch_tc<128, 1, tc::EK_F32_RS>(ma, mb, p, s);
      break;
    case tc::EK_GENERIC_RS:
      if (cg == 2) launch_tc<128, 2, tc::EK_GENERIC_RS>(ma, mb, p, s);
      else launch_tc<128, 1, tc::EK_GENERIC_RS>(ma, mb, p, s);
      break;
    case tc::EK_BF16: launch_ek<tc::EK_BF16>(cg, bn, ma, mb, p, s); break;
    case tc::EK_GELU: launch_ek<tc::EK_GELU>(cg, bn, ma, mb, p, s); break;
    case tc::EK_DGELU: launch_ek<tc::EK_DGELU>(cg, bn, ma, mb, p, s); break;
    case tc::EK_F32: launch_ek<tc::EK_F32>(cg, bn, ma, mb, p, s); break;
    default: launch_ek<tc::EK_GENERIC>(cg, bn, ma, mb, p, s); break;
  }
}

}  // namespace hp
