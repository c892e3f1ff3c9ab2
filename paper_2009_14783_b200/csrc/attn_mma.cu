// Tensor-core multi-head self-attention for the bf16 path (dk = 64, varlen
// sequences of <= 128 tokens): one CTA per (instance, head), the whole
// sequence staged in shared memory, bf16 mma.sync m16n8k16 with fp32
// accumulation, softmax in registers (the S accumulator fragments are reused
// as the A operand of P.V).  Semantics: softmax((Q K^T) / sqrt(dk)) V over the
// instance's own tokens (attention.hpp:15-26); backward as tape.hpp:274-286.
//
// Fragment layouts (m16n8k16, lane = 4*g + t):
//   A 16x16: a0 (g, 2t..), a1 (g+8, 2t..), a2 (g, 2t+8..), a3 (g+8, 2t+8..)
//   B 16x8 : b0 (k=2t.., n=g), b1 (k=2t+8.., n=g)
//   C 16x8 : c0,c1 (g, 2t..), c2,c3 (g+8, 2t..)
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cfloat>

#include "hp_common.h"
#include "kernels.h"

namespace hp {
namespace attn {

using bf16 = __nv_bfloat16;
constexpr int DK = 64;
constexpr int MAXN = 128;
constexpr int LDS = DK + 8;     // 144-byte rows: conflict-free ldmatrix
constexpr int LDP = MAXN + 8;   // dS^T rows

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                          uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma16816(float* c, uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// Rows [0, n) of one head's 64 columns -> smem [MAXN][LDS], zero padded to
// np, with cp.async (every 16-byte chunk in flight at once; rows >= n are
// zero-filled by a 0-byte source).  Caller commits / waits.
__device__ __forceinline__ void load_tile(bf16* dst, const bf16* src, int64_t ld, int n, int np) {
  for (int e = threadIdx.x; e < np * (DK / 8); e += blockDim.x) {
    const int r = e / (DK / 8), c8 = e % (DK / 8);
    const bf16* g = src + (int64_t)min(r, n - 1) * ld + 8 * c8;
    const uint32_t bytes = r < n ? 16u : 0u;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(su32(dst + r * LDS + 8 * c8)),
                 "l"(g), "r"(bytes)
                 : "memory");
  }
}
__device__ __forceinline__ void load_wait() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

// A fragment (16 rows x 16 k) from a row-major [rows][LDS] tile at (r0, k0).
__device__ __forceinline__ void lda_rows(const bf16* base, int r0, int k0, int lane, uint32_t* a) {
  const int r = r0 + (lane & 7) + ((lane >> 3) & 1) * 8;
  const int c = k0 + ((lane >> 4) & 1) * 8;
  ldsm_x4(su32(base + r * LDS + c), a[0], a[1], a[2], a[3]);
}
// Two B fragments (n-tiles n0, n0+8; k0..k0+15) when B^T is stored
// row-major [n][LDS] (i.e. B[k][n] = base[n][k]).
__device__ __forceinline__ void ldb_nk(const bf16* base, int n0, int k0, int lane, uint32_t* b) {
  const int r = n0 + (lane & 7) + ((lane >> 4) & 1) * 8;
  const int c = k0 + ((lane >> 3) & 1) * 8;
  ldsm_x4(su32(base + r * LDS + c), b[0], b[1], b[2], b[3]);
}
// Two B fragments (n-tiles n0, n0+8; k0..k0+15) when B is stored row-major
// [k][LDS] (B[k][n] = base[k][n]).
__device__ __forceinline__ void ldb_kn(const bf16* base, int ld, int k0, int n0, int lane,
                                       uint32_t* b) {
  const int r = k0 + (lane & 7) + ((lane >> 3) & 1) * 8;
  const int c = n0 + ((lane >> 4) & 1) * 8;
  ldsm_x4_t(su32(base + r * ld + c), b[0], b[1], b[2], b[3]);
}

__global__ void __launch_bounds__(256, 1)
    attn_fwd_mma(const int* __restrict__ cu, int H, const bf16* __restrict__ qkv,
                 bf16* __restrict__ o, float* __restrict__ lse, int T_total) {
  extern __shared__ __align__(16) uint8_t fsm[];
  bf16* Qs = reinterpret_cast<bf16*>(fsm);
  bf16* Ks = Qs + MAXN * LDS;
  bf16* Vs = Ks + MAXN * LDS;
  const int b = blockIdx.x, h = blockIdx.y;
  const int row0 = cu[b], n = cu[b + 1] - row0;
  if (n <= 0) return;
  const int np = (n + 15) & ~15;
  const int d = H * DK;
  const int64_t ldq = 3 * (int64_t)d;
  const bf16* base = qkv + (int64_t)row0 * ldq;
  load_tile(Qs, base + h * DK, ldq, n, np);
  load_tile(Ks, base + d + h * DK, ldq, n, np);
  load_tile(Vs, base + 2 * d + h * DK, ldq, n, np);
  load_wait();
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int m0 = warp * 16;
  if (m0 >= np) return;
  float s[16][4];
#pragma unroll
  for (int j = 0; j < 16; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
  for (int kk = 0; kk < DK / 16; ++kk) {
    uint32_t a[4];
    lda_rows(Qs, m0, 16 * kk, lane, a);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (16 * j < np) {
        uint32_t bb[4];
        ldb_nk(Ks, 16 * j, 16 * kk, lane, bb);
        mma16816(s[2 * j], a[0], a[1], a[2], a[3], bb[0], bb[1]);
        mma16816(s[2 * j + 1], a[0], a[1], a[2], a[3], bb[2], bb[3]);
      }
    }
  }
  // softmax over the instance's keys; scale folded into exp2
  const float scale = rsqrtf((float)DK);
  const float sl2 = scale * 1.4426950408889634f;
  float mx0 = -FLT_MAX, mx1 = -FLT_MAX;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int c = 8 * j + 2 * t;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const bool ok = c + e < n;
      s[j][e] = ok ? s[j][e] : -FLT_MAX;
      s[j][2 + e] = ok ? s[j][2 + e] : -FLT_MAX;
      mx0 = fmaxf(mx0, s[j][e]);
      mx1 = fmaxf(mx1, s[j][2 + e]);
    }
  }
  mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
  mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
  mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
  mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
  float sum0 = 0.f, sum1 = 0.f;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      s[j][e] = exp2f((s[j][e] - mx0) * sl2);
      s[j][2 + e] = exp2f((s[j][2 + e] - mx1) * sl2);
      sum0 += s[j][e];
      sum1 += s[j][2 + e];
    }
  }
  sum0 += __shfl_xor_sync(0xffffffffu, sum0, 1);
  sum0 += __shfl_xor_sync(0xffffffffu, sum0, 2);
  sum1 += __shfl_xor_sync(0xffffffffu, sum1, 1);
  sum1 += __shfl_xor_sync(0xffffffffu, sum1, 2);
  // O = P V
  float acc[8][4];
#pragma unroll
  for (int u = 0; u < 8; ++u) acc[u][0] = acc[u][1] = acc[u][2] = acc[u][3] = 0.f;
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    if (16 * kk < np) {
      const uint32_t a0 = pack2(s[2 * kk][0], s[2 * kk][1]);
      const uint32_t a1 = pack2(s[2 * kk][2], s[2 * kk][3]);
      const uint32_t a2 = pack2(s[2 * kk + 1][0], s[2 * kk + 1][1]);
      const uint32_t a3 = pack2(s[2 * kk + 1][2], s[2 * kk + 1][3]);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        uint32_t bb[4];
        ldb_kn(Vs, LDS, 16 * kk, 16 * u, lane, bb);
        mma16816(acc[2 * u], a0, a1, a2, a3, bb[0], bb[1]);
        mma16816(acc[2 * u + 1], a0, a1, a2, a3, bb[2], bb[3]);
      }
    }
  }
  const float inv0 = 1.f / sum0, inv1 = 1.f / sum1;
  const int r_a = m0 + g, r_b = m0 + g + 8;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int c = h * DK + 8 * u + 2 * t;
    if (r_a < n)
      *reinterpret_cast<uint32_t*>(o + (int64_t)(row0 + r_a) * d + c) =
          pack2(acc[u][0] * inv0, acc[u][1] * inv0);
    if (r_b < n)
      *reinterpret_cast<uint32_t*>(o + (int64_t)(row0 + r_b) * d + c) =
          pack2(acc[u][2] * inv1, acc[u][3] * inv1);
  }
  if (t == 0) {
    if (r_a < n) lse[(int64_t)h * T_total + row0 + r_a] = mx0 * scale + logf(sum0);
    if (r_b < n) lse[(int64_t)h * T_total + row0 + r_b] = mx1 * scale + logf(sum1);
  }
}

struct BwdSmem {
  bf16 Q[MAXN * LDS], K[MAXN * LDS], V[MAXN * LDS], dO[MAXN * LDS];
  union {
    bf16 O[MAXN * LDS];  // only until D is formed
    bf16 dSt[MAXN * LDP];
  };
  float lse[MAXN], D[MAXN];
};

__global__ void __launch_bounds__(256, 1)
    attn_bwd_mma(const int* __restrict__ cu, int H, const bf16* __restrict__ qkv,
                 const bf16* __restrict__ o, const bf16* __restrict__ dO,
                 const float* __restrict__ lse, bf16* __restrict__ dqkv, int T_total) {
  extern __shared__ __align__(16) uint8_t smraw[];
  BwdSmem& sm = *reinterpret_cast<BwdSmem*>(smraw);
  const int b = blockIdx.x, h = blockIdx.y;
  const int row0 = cu[b], n = cu[b + 1] - row0;
  if (n <= 0) return;
  const int np = (n + 15) & ~15;
  const int d = H * DK;
  const int64_t ldq = 3 * (int64_t)d;
  const bf16* base = qkv + (int64_t)row0 * ldq;
  load_tile(sm.Q, base + h * DK, ldq, n, np);
  load_tile(sm.K, base + d + h * DK, ldq, n, np);
  load_tile(sm.V, base + 2 * d + h * DK, ldq, n, np);
  load_tile(sm.dO, dO + (int64_t)row0 * d + h * DK, d, n, np);
  load_tile(sm.O, o + (int64_t)row0 * d + h * DK, d, n, np);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  for (int r = threadIdx.x; r < np; r += blockDim.x)
    sm.lse[r] = r < n ? lse[(int64_t)h * T_total + row0 + r] : 0.f;
  load_wait();
  __syncthreads();
  // D_i = rowsum(dO * O) (padded rows are zero)
  for (int r = warp; r < np; r += 8) {
    const float2 of = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(sm.O + r * LDS)[lane]);
    const float2 gf = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(sm.dO + r * LDS)[lane]);
    float acc = of.x * gf.x + of.y * gf.y;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) sm.D[r] = acc;
  }
  __syncthreads();  // O is dead from here on; its space becomes dS^T
  const float scale = rsqrtf((float)DK);
  const float l2e = 1.4426950408889634f;
  const int k0 = warp * 16;  // this warp's 16 keys
  if (k0 < np) {
    float dv[8][4], dk[8][4];
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int e = 0; e < 4; ++e) dv[u][e] = dk[u][e] = 0.f;
#pragma unroll 1
    for (int qc = 0; qc < np; qc += 64) {
      float st[8][4], dpt[8][4];
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) st[j][e] = dpt[j][e] = 0.f;
#pragma unroll
      for (int kk = 0; kk < DK / 16; ++kk) {
        uint32_t ak[4], av[4];
        lda_rows(sm.K, k0, 16 * kk, lane, ak);
        lda_rows(sm.V, k0, 16 * kk, lane, av);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (qc + 16 * j < np) {
            uint32_t bq[4], bo[4];
            ldb_nk(sm.Q, qc + 16 * j, 16 * kk, lane, bq);
            ldb_nk(sm.dO, qc + 16 * j, 16 * kk, lane, bo);
            mma16816(st[2 * j], ak[0], ak[1], ak[2], ak[3], bq[0], bq[1]);
            mma16816(st[2 * j + 1], ak[0], ak[1], ak[2], ak[3], bq[2], bq[3]);
            mma16816(dpt[2 * j], av[0], av[1], av[2], av[3], bo[0], bo[1]);
            mma16816(dpt[2 * j + 1], av[0], av[1], av[2], av[3], bo[2], bo[3]);
          }
        }
      }
      // P^T and dS^T = P^T (dP^T - D) * scale
      const int ka = k0 + g, kb = k0 + g + 8;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int q = qc + 8 * j + 2 * t + e;
          const bool qok = q < n;
          const float lq = qok ? sm.lse[q] : 0.f;
          const float Dq = qok ? sm.D[q] : 0.f;
          const float pa = (qok && ka < n) ? exp2f((st[j][e] * scale - lq) * l2e) : 0.f;
          const float pb = (qok && kb < n) ? exp2f((st[j][2 + e] * scale - lq) * l2e) : 0.f;
          st[j][e] = pa;
          st[j][2 + e] = pb;
          dpt[j][e] = pa * (dpt[j][e] - Dq) * scale;
          dpt[j][2 + e] = pb * (dpt[j][2 + e] - Dq) * scale;
        }
      }
      // dV += P^T dO ; dK += dS^T Q  (k = queries of this chunk)
#pragma unroll
      for (int kq = 0; kq < 4; ++kq) {
        if (qc + 16 * kq < np) {
          const uint32_t p0 = pack2(st[2 * kq][0], st[2 * kq][1]);
          const uint32_t p1 = pack2(st[2 * kq][2], st[2 * kq][3]);
          const uint32_t p2 = pack2(st[2 * kq + 1][0], st[2 * kq + 1][1]);
          const uint32_t p3 = pack2(st[2 * kq + 1][2], st[2 * kq + 1][3]);
          const uint32_t s0 = pack2(dpt[2 * kq][0], dpt[2 * kq][1]);
          const uint32_t s1 = pack2(dpt[2 * kq][2], dpt[2 * kq][3]);
          const uint32_t s2 = pack2(dpt[2 * kq + 1][0], dpt[2 * kq + 1][1]);
          const uint32_t s3 = pack2(dpt[2 * kq + 1][2], dpt[2 * kq + 1][3]);
          // dS^T -> smem for the dQ pass
          bf16* ds = sm.dSt;
          *reinterpret_cast<uint32_t*>(ds + (k0 + g) * LDP + qc + 16 * kq + 2 * t) = s0;
          *reinterpret_cast<uint32_t*>(ds + (k0 + g + 8) * LDP + qc + 16 * kq + 2 * t) = s1;
          *reinterpret_cast<uint32_t*>(ds + (k0 + g) * LDP + qc + 16 * kq + 8 + 2 * t) = s2;
          *reinterpret_cast<uint32_t*>(ds + (k0 + g + 8) * LDP + qc + 16 * kq + 8 + 2 * t) = s3;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            uint32_t bo[4], bq[4];
            ldb_kn(sm.dO, LDS, qc + 16 * kq, 16 * u, lane, bo);
            ldb_kn(sm.Q, LDS, qc + 16 * kq, 16 * u, lane, bq);
            mma16816(dv[2 * u], p0, p1, p2, p3, bo[0], bo[1]);
            mma16816(dv[2 * u + 1], p0, p1, p2, p3, bo[2], bo[3]);
            mma16816(dk[2 * u], s0, s1, s2, s3, bq[0], bq[1]);
            mma16816(dk[2 * u + 1], s0, s1, s2, s3, bq[2], bq[3]);
          }
        }
      }
    }
    const int ra = k0 + g, rb = k0 + g + 8;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int c = 8 * u + 2 * t;
      if (ra < n) {
        bf16* row = dqkv + (int64_t)(row0 + ra) * ldq;
        *reinterpret_cast<uint32_t*>(row + d + h * DK + c) = pack2(dk[u][0], dk[u][1]);
        *reinterpret_cast<uint32_t*>(row + 2 * d + h * DK + c) = pack2(dv[u][0], dv[u][1]);
      }
      if (rb < n) {
        bf16* row = dqkv + (int64_t)(row0 + rb) * ldq;
        *reinterpret_cast<uint32_t*>(row + d + h * DK + c) = pack2(dk[u][2], dk[u][3]);
        *reinterpret_cast<uint32_t*>(row + 2 * d + h * DK + c) = pack2(dv[u][2], dv[u][3]);
      }
    }
  }
  __syncthreads();
  // dQ = dS K, dS[q][key] = dSt[key][q]
  const int q0 = warp * 16;
  if (q0 >= np) return;
  float dq[8][4];
#pragma unroll
  for (int u = 0; u < 8; ++u) dq[u][0] = dq[u][1] = dq[u][2] = dq[u][3] = 0.f;
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    if (16 * kk < np) {
      uint32_t a[4];
      const int mi = lane >> 3;
      const int key = 16 * kk + (lane & 7) + ((mi >> 1) & 1) * 8;
      const int qq = q0 + (mi & 1) * 8;
      ldsm_x4_t(su32(sm.dSt + key * LDP + qq), a[0], a[1], a[2], a[3]);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        uint32_t bk[4];
        ldb_kn(sm.K, LDS, 16 * kk, 16 * u, lane, bk);
        mma16816(dq[2 * u], a[0], a[1], a[2], a[3], bk[0], bk[1]);
        mma16816(dq[2 * u + 1], a[0], a[1], a[2], a[3], bk[2], bk[3]);
      }
    }
  }
  const int ra = q0 + g, rb = q0 + g + 8;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int c = h * DK + 8 * u + 2 * t;
    if (ra < n)
      *reinterpret_cast<uint32_t*>(dqkv + (int64_t)(row0 + ra) * ldq + c) = pack2(dq[u][0], dq[u][1]);
    if (rb < n)
      *reinterpret_cast<uint32_t*>(dqkv + (int64_t)(row0 + rb) * ldq + c) = pack2(dq[u][2], dq[u][3]);
  }
}

}  // namespace attn

bool attention_mma_supported(int dk, int max_seq) { return dk == attn::DK && max_seq <= attn::MAXN; }

void attention_fwd_mma(const DevBatch& b, int H, const void* qkv, void* o, float* lse,
                       cudaStream_t s) {
  if (b.B == 0) return;
  const int sm = 3 * attn::MAXN * attn::LDS * 2;
  static bool attr = false;
  if (!attr) {
    HP_CUDA(cudaFuncSetAttribute(attn::attn_fwd_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    attr = true;
  }
  attn::attn_fwd_mma<<<dim3(b.B, H), 256, sm, s>>>(b.cu, H, (const attn::bf16*)qkv,
                                                  (attn::bf16*)o, lse, b.T);
  HP_CUDA(cudaGetLastError());
  count_launch();
}

void attention_bwd_mma(const DevBatch& b, int H, const void* qkv, const void* o, const void* dO,
                       const float* lse, void* dqkv, cudaStream_t s) {
  if (b.B == 0) return;
  const int sm = (int)sizeof(attn::BwdSmem);
  static bool attr = false;
  if (!attr) {
    HP_CUDA(cudaFuncSetAttribute(attn::attn_bwd_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    attr = true;
  }
  attn::attn_bwd_mma<<<dim3(b.B, H), 256, sm, s>>>(b.cu, H, (const attn::bf16*)qkv,
                                                   (const attn::bf16*)o, (const attn::bf16*)dO,
                                                   lse, (attn::bf16*)dqkv, b.T);
  HP_CUDA(cudaGetLastError());
  count_launch();
}

}  // namespace hp
