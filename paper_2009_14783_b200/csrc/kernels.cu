// sm_100a kernels of the DP step that are not tcgen05 GEMMs: embedding,
// LayerNorm, varlen attention, label-smoothed CE, NSP head, column sums,
// Adam, and the fp32 SIMT GEMM used by the fp32 parity path.
//
// Reference semantics (file:line into the reference's proj/):
//   embedding       model.hpp:354-365, attention.hpp:53-67
//   attention       attention.hpp:15-50, tape.hpp:123-140 / 274-286
//   ls_ce           tape.hpp:180-209 / 302-321
//   gather/scatter  tape.hpp:144-159 / 287-292
//   adam / sgd      kernels_scalar.cpp:71-83, optim.hpp:107-146
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cfloat>
#include <cmath>
#include <type_traits>
#include <map>
#include <mutex>
#include <string>
#include <vector>
#include <cstdlib>

#include "hp_common.h"
#include "kernels.h"
#include "launch.cuh"
#include "tc_common.cuh"

namespace hp {

namespace {
std::atomic<uint64_t> g_launches{0};
}
uint64_t kernel_launch_count() { return g_launches.load(); }
bool pdl_on(int cls) {
  static const int mask = [] {
    const char* e = std::getenv("HP_PDL");
    if (!e || std::string(e) == "0") return 0;  // default off: measured no gain
    if (std::string(e) == "1") return 7;
    const std::string v(e);
    return (v.find("gemm") != std::string::npos ? 1 : 0) |
           (v.find("attn") != std::string::npos ? 2 : 0) | (v.find("ln") != std::string::npos ? 4 : 0);
  }();
  return (mask >> cls) & 1;
}
void count_launch(int n) { g_launches += n; }

#define LAUNCH_CHECK() HP_CUDA(cudaGetLastError())

using bf16 = __nv_bfloat16;

__device__ __forceinline__ float tof(float x) { return x; }
__device__ __forceinline__ float tof(bf16 x) { return __bfloat162float(x); }
template <class T> __device__ __forceinline__ T fromf(float x);
template <> __device__ __forceinline__ float fromf<float>(float x) { return x; }
template <> __device__ __forceinline__ bf16 fromf<bf16>(float x) { return __float2bfloat16_rn(x); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
template <int NT>
__device__ float block_sum(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float r = (threadIdx.x < NT / 32) ? red[threadIdx.x] : 0.f;
  if (w == 0) r = warp_sum(r);
  if (threadIdx.x == 0) red[0] = r;
  __syncthreads();
  return red[0];
}
template <int NT>
__device__ float block_max(float v, float* red) {
  v = warp_max(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float r = (threadIdx.x < NT / 32) ? red[threadIdx.x] : -FLT_MAX;
  if (w == 0) r = warp_max(r);
  if (threadIdx.x == 0) red[0] = r;
  __syncthreads();
  return red[0];
}

__device__ __forceinline__ void unpack8(const uint4& u, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 v = __bfloat1622float2(h[e]);
    f[2 * e] = v.x;
    f[2 * e + 1] = v.y;
  }
}
__device__ __forceinline__ uint4 pack8(const float* f) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int e = 0; e < 4; ++e) h[e] = __floats2bfloat162_rn(f[2 * e], f[2 * e + 1]);
  return u;
}


#define DISPATCH1(dt, T, ...)              \
  if ((dt) == DType::f32) {                \
    using T = float;                       \
    __VA_ARGS__;                           \
  } else {                                 \
    using T = bf16;                        \
    __VA_ARGS__;                           \
  }

// ------------------------------------------------------------------ embedding
template <class WT, class XT>
__global__ void embed_fwd_kernel(int T, int d, const int* __restrict__ tok,
                                 const int* __restrict__ seg, const int* __restrict__ pos,
                                 const WT* __restrict__ E, const WT* __restrict__ s0,
                                 const WT* __restrict__ s1, const float* __restrict__ pe,
                                 XT* __restrict__ x) {
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= T) return;
  const int lane = threadIdx.x & 31;
  const WT* e = E + (int64_t)tok[t] * d;
  const WT* sg = seg[t] == 0 ? s0 : s1;
  const float* p = pe + (int64_t)pos[t] * d;
  // tape order: (E[tok] + (on0 s0 + on1 s1)) + PE  (model.hpp:361-365)
  for (int c = lane; c < d; c += 32)
    x[(int64_t)t * d + c] = fromf<XT>((tof(e[c]) + tof(sg[c])) + p[c]);
}

// seq2seq extension: x[t] = scale * E[tok] + PE[pos] (fairseq's embed_scale
// = sqrt(d), no segment rows)
template <class WT, class XT>
__global__ void embed_scaled_kernel(int T, int d, const int* __restrict__ tok,
                                    const int* __restrict__ pos, const WT* __restrict__ E,
                                    float scale, const float* __restrict__ pe, XT* __restrict__ x) {
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= T) return;
  const int lane = threadIdx.x & 31;
  const WT* e = E + (int64_t)tok[t] * d;
  const float* p = pe + (int64_t)pos[t] * d;
  for (int c = lane; c < d; c += 32) x[(int64_t)t * d + c] = fromf<XT>(scale * tof(e[c]) + p[c]);
}

void embed_scaled_fwd(int T, int d, const int* tok, const int* pos, const void* E, DType wt,
                      float scale, const float* pe, void* x, DType xt, cudaStream_t s) {
  if (T == 0) return;
  DISPATCH1(wt, W, DISPATCH1(xt, X,
      embed_scaled_kernel<W, X><<<(T + 7) / 8, 256, 0, s>>>(T, d, tok, pos, (const W*)E, scale, pe,
                                                            (X*)x)));
  LAUNCH_CHECK();
  count_launch();
}

void embed_fwd(const DevBatch& b, int d, const void* E, const void* seg0,
               const void* seg1, DType wt, const float* pe, void* x, DType xt,
               cudaStream_t s) {
  if (b.T == 0) return;
  const int wpb = 8;
  dim3 grid((b.T + wpb - 1) / wpb);
  DISPATCH1(wt, W, DISPATCH1(xt, X,
      embed_fwd_kernel<W, X><<<grid, 256, 0, s>>>(b.T, d, b.tok, b.seg, b.pos,
          (const W*)E, (const W*)seg0, (const W*)seg1, pe, (X*)x)));
  LAUNCH_CHECK();
  count_launch();
}

// dE rows of the batch's distinct token ids: row id = sum of dx over the
// tokens with that id -- no atomics, fixed summation order, so the round is
// deterministic.  Engine::stage_batch groups token positions by id (perm,
// useg) and lists the ids with <= kEmbHot tokens first (ulist[0, n_small)),
// the hot ones (e.g. [MASK], [CLS]) after (ulist[n_small, n_small + n_hot)).
//   small id: one warp, rows summed in position order (the reference's
//             accumulation order), loads issued 8 rows ahead
//   hot id:   one 1024-thread CTA; warp w sums rows w, w+32, ... in order,
//             the 32 partials are added in warp order through smem
// Fixed grids, counts read on the device (CUDA-graph stable).
constexpr int kEmbHot = 32;

template <class XT>
__device__ __forceinline__ void emb_load8(const XT* p, float* f) {
  if constexpr (std::is_same<XT, bf16>::value) {
    unpack8(*reinterpret_cast<const uint4*>(p), f);
  } else {
    const float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
    f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
  }
}

// small ids: warp `gw` of `nw` warps (across the blocks taking this role)
template <class XT>
__device__ __forceinline__ void embed_grad_small_warps(int gw, int nw, const int* __restrict__ counts,
                                                       const int* __restrict__ ulist,
                                                       const int* __restrict__ uid,
                                                       const int* __restrict__ useg,
                                                       const int* __restrict__ perm, int d,
                                                       const XT* __restrict__ dx,
                                                       float* __restrict__ dE, int64_t ostride,
                                                       int by_slot) {
  const int n_small = counts[0];
  const int lane = threadIdx.x & 31;
  const int d8 = d / 8;
  for (int i = gw; i < n_small; i += nw) {
    const int u = ulist[i];
    const int k0 = useg[u], cnt = useg[u + 1] - k0;  // <= kEmbHot = 32: one position per lane
    const int mine = lane < cnt ? perm[k0 + lane] : 0;
    float* o = dE + (int64_t)(by_slot ? u : uid[u]) * ostride;
    for (int cb = 0; cb < d8; cb += 32) {  // warp-uniform trip count (shuffles below)
      const int c8 = cb + lane;
      const bool act = c8 < d8;
      float acc[8] = {};
      for (int k = 0; k < cnt; k += 4) {  // positions in order: fixed summation order
        float f[4][8];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int t = __shfl_sync(0xffffffffu, mine, (k + j) & 31);
          if (act && k + j < cnt) emb_load8(dx + (int64_t)t * d + 8 * c8, f[j]);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (k + j < cnt)
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[e] += f[j][e];
      }
      if (act) {
        reinterpret_cast<float4*>(o + 8 * c8)[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
        reinterpret_cast<float4*>(o + 8 * c8)[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
      }
    }
  }
}

// hot ids: block `hb` of `nhb` (1024 threads: 32 warps)
template <class XT>
__device__ __forceinline__ void embed_grad_hot_block(int hb, int nhb, float* part,
                                                     const int* __restrict__ counts,
                                                     const int* __restrict__ ulist,
                                                     const int* __restrict__ uid,
                                                     const int* __restrict__ useg,
                                                     const int* __restrict__ perm, int d,
                                                     const XT* __restrict__ dx,
                                                     float* __restrict__ dE, int64_t ostride,
                                                     int by_slot) {
  const int n_small = counts[0], n_hot = counts[1];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int d8 = d / 8;
  for (int i = hb; i < n_hot; i += nhb) {
    const int u = ulist[n_small + i];
    const int k0 = useg[u], k1 = useg[u + 1];
    for (int c8 = lane; c8 < d8; c8 += 32) {
      float acc[8] = {};
      for (int k = k0 + w; k < k1; k += 32 * 4) {
        float f[4][8];
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (k + 32 * j < k1) emb_load8(dx + (int64_t)perm[k + 32 * j] * d + 8 * c8, f[j]);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (k + 32 * j < k1)
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[e] += f[j][e];
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) part[w * d + 8 * c8 + e] = acc[e];
    }
    __syncthreads();
    float* o = dE + (int64_t)(by_slot ? u : uid[u]) * ostride;
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
      float acc = 0.f;
      for (int j = 0; j < 32; ++j) acc += part[j * d + c];
      o[c] = acc;
    }
    __syncthreads();
  }
}

// One launch for both: blocks [0, kEmbHotBlocks) take the hot ids, the rest
// the small ones -- the two disjoint row sets are summed side by side.
constexpr int kEmbHotBlocks = 64;
template <class XT>
__global__ void __launch_bounds__(1024) embed_grad_kernel(const int* __restrict__ counts,
                                                          const int* __restrict__ ulist,
                                                          const int* __restrict__ uid,
                                                          const int* __restrict__ useg,
                                                          const int* __restrict__ perm, int d,
                                                          const XT* __restrict__ dx,
                                                          float* __restrict__ dE, int64_t ostride,
                                                          int by_slot) {
  extern __shared__ float part[];  // hot blocks: [32 warps][d]
  if (blockIdx.x < kEmbHotBlocks) {
    embed_grad_hot_block<XT>(blockIdx.x, kEmbHotBlocks, part, counts, ulist, uid, useg, perm, d, dx, dE,
                             ostride, by_slot);
  } else {
    const int wpb = blockDim.x >> 5;
    embed_grad_small_warps<XT>((blockIdx.x - kEmbHotBlocks) * wpb + (threadIdx.x >> 5),
                               (gridDim.x - kEmbHotBlocks) * wpb, counts, ulist, uid, useg, perm, d, dx,
                               dE, ostride, by_slot);
  }
}

// column sums over row chunks; sel (optional) keeps rows with sel[r] == want
template <class XT>
__global__ void colsum_partial_kernel(int R, int N, const XT* __restrict__ x, int64_t ld,
                                      const int* __restrict__ sel, int want, int rows_per,
                                      float* __restrict__ part) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  const int r0 = blockIdx.y * rows_per;
  const int r1 = min(R, r0 + rows_per);
  float acc = 0.f;
  for (int r = r0; r < r1; ++r)
    if (!sel || sel[r] == want) acc += tof(x[(int64_t)r * ld + c]);
  part[(int64_t)blockIdx.y * N + c] = acc;
}
// Final stage of every column reduction: out[c] = sum_k part[k*stride + c].
// Block (32 columns x 16 chunk-lanes): each lane sums every 16th chunk, then
// the 16 lane sums are added in a fixed order (deterministic).
constexpr int kFinY = 16;
__device__ __forceinline__ float final_sum(int chunks, int stride, const float* __restrict__ part,
                                           int c, bool ok) {
  __shared__ float red[kFinY][33];
  float acc = 0.f;
  if (ok)
    for (int k = threadIdx.y; k < chunks; k += kFinY) acc += part[(int64_t)k * stride + c];
  red[threadIdx.y][threadIdx.x] = acc;
  __syncthreads();
  float s = 0.f;
  if (threadIdx.y == 0)
#pragma unroll
    for (int j = 0; j < kFinY; ++j) s += red[j][threadIdx.x];
  return s;
}
__global__ void colsum_final_strided(int chunks, int stride, int N, const float* __restrict__ part,
                                     float* __restrict__ out) {
  const int c = blockIdx.x * 32 + threadIdx.x;
  const float s = final_sum(chunks, stride, part, c, c < N);
  if (threadIdx.y == 0 && c < N) out[c] = s;
}
#define FINAL_LAUNCH(N) dim3(((N) + 31) / 32), dim3(32, kFinY)
__global__ void colsum_final_kernel(int chunks, int N, const float* __restrict__ part,
                                    float* __restrict__ out) {
  const int c = blockIdx.x * 32 + threadIdx.x;
  const float s = final_sum(chunks, N, part, c, c < N);
  if (threadIdx.y == 0 && c < N) out[c] = s;
}

static constexpr int kColRows = 64;
constexpr int kLnBwdRows = 32;  // rows per LayerNorm-backward CTA (multiple of 8)

// Segment-embedding gradients in one pass: per 32-row chunk, the column sums
// of the rows with segment 0 and with segment 1 (8 columns per thread), as
// partials [chunk][2 * N8] (segment 0 | segment 1); finalised by
// colsum_final_strided.
template <class XT>
__global__ void segsum_partial_vec(int R, int N8, const XT* __restrict__ x, const int* __restrict__ seg,
                                   int rows_per, float* __restrict__ part) {
  const int c8 = blockIdx.x * blockDim.x + threadIdx.x;
  if (c8 * 8 >= N8) return;
  const int r0 = blockIdx.y * rows_per, r1 = min(R, r0 + rows_per);
  float a0[8] = {}, a1[8] = {};
  for (int r = r0; r < r1; ++r) {
    float f[8];
    emb_load8(x + (int64_t)r * N8 + 8 * c8, f);
    if (seg[r] == 0) {
#pragma unroll
      for (int e = 0; e < 8; ++e) a0[e] += f[e];
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) a1[e] += f[e];
    }
  }
  float4* o = reinterpret_cast<float4*>(part + (int64_t)blockIdx.y * 2 * N8 + 8 * c8);
  o[0] = make_float4(a0[0], a0[1], a0[2], a0[3]);
  o[1] = make_float4(a0[4], a0[5], a0[6], a0[7]);
  o = reinterpret_cast<float4*>(part + (int64_t)blockIdx.y * 2 * N8 + N8 + 8 * c8);
  o[0] = make_float4(a1[0], a1[1], a1[2], a1[3]);
  o[1] = make_float4(a1[4], a1[5], a1[6], a1[7]);
}

// bf16 [R x ld] column sums, 8 columns (one 16-byte load) per thread.
__global__ void colsum_partial_vec(int R, int N8, const bf16* __restrict__ x, int64_t ld,
                                   int rows_per, float* __restrict__ part) {
  const int c8 = blockIdx.x * blockDim.x + threadIdx.x;
  if (c8 * 8 >= N8) return;
  const int r0 = blockIdx.y * rows_per, r1 = min(R, r0 + rows_per);
  float acc[8] = {};
  int r = r0;
  for (; r + 8 <= r1; r += 8) {  // eight independent 16-byte loads in flight
    uint4 u[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) u[q] = *reinterpret_cast<const uint4*>(x + (int64_t)(r + q) * ld + 8 * c8);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float f[8];
      unpack8(u[q], f);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += f[e];
    }
  }
  for (; r < r1; ++r) {
    float f[8];
    unpack8(*reinterpret_cast<const uint4*>(x + (int64_t)r * ld + 8 * c8), f);
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] += f[e];
  }
  float4* o = reinterpret_cast<float4*>(part + (int64_t)blockIdx.y * N8 + 8 * c8);
  o[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
  o[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
}

template <class XT>
static void colsum_launch(int R, int N, const XT* x, int64_t ld, const int* sel,
                          int want, float* out, float* scratch, cudaStream_t s,
                          DeferredFinal* df = nullptr) {
  if constexpr (std::is_same<XT, bf16>::value) {
    const int N8 = (N + 7) & ~7;
    if (!sel && ld % 8 == 0 && ld >= N8 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 && R > 0) {
      const int rows_per = 32;
      const int chunks = (R + rows_per - 1) / rows_per;
      dim3 g1((N8 / 8 + 127) / 128, chunks);
      if (df) {
        colsum_partial_vec<<<g1, 128, 0, s>>>(R, N8, x, ld, rows_per, df->part);
        LAUNCH_CHECK();
        count_launch();
        df->queued = true;
        df->kind = 1;
        df->chunks = chunks;
        df->stride = N8;
        df->n = N;
        df->o0 = out;
        return;
      }
      colsum_partial_vec<<<g1, 128, 0, s>>>(R, N8, x, ld, rows_per, scratch);
      LAUNCH_CHECK();
      colsum_final_strided<<<FINAL_LAUNCH(N), 0, s>>>(chunks, N8, N, scratch, out);
      LAUNCH_CHECK();
      count_launch(2);
      return;
    }
  }
  const int chunks = (R + kColRows - 1) / kColRows;
  if (chunks == 0) {
    HP_CUDA(cudaMemsetAsync(out, 0, sizeof(float) * N, s));
    return;
  }
  dim3 g1((N + 127) / 128, chunks);
  colsum_partial_kernel<XT><<<g1, 128, 0, s>>>(R, N, x, ld, sel, want, kColRows, scratch);
  LAUNCH_CHECK();
  colsum_final_kernel<<<FINAL_LAUNCH(N), 0, s>>>(chunks, N, scratch, out);
  LAUNCH_CHECK();
  count_launch(2);
}

static void embed_bwd_impl(const DevBatch& b, int d, const void* dx, DType xt, float* dE,
                           int64_t ostride, int by_slot, float* dseg0, float* dseg1,
                           float* scratch, cudaStream_t s);
// slot ids of the row-sparse embedding gradient (embed_bwd_rows)
__global__ void emb_slot_ids_kernel(const int* __restrict__ counts, const int* __restrict__ uid,
                                    float* __restrict__ rows, int cap, int64_t stride) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= cap) return;
  const int U = counts[0] + counts[1];
  rows[(int64_t)u * stride] = __int_as_float(u < U ? uid[u] : -1);
}
__global__ void emb_scatter_kernel(const float* __restrict__ rows, int cap, int d,
                                   float* __restrict__ dE, float scale) {
  const int u = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (u >= cap) return;
  const float* r = rows + (int64_t)u * (d + 4);
  const int id = __float_as_int(r[0]);
  if (id < 0) return;
  float* o = dE + (int64_t)id * d;
  for (int c = 4 * lane; c < d; c += 128) {
    const float4 v = *reinterpret_cast<const float4*>(r + 4 + c);
    float4 w = *reinterpret_cast<float4*>(o + c);
    w.x += scale * v.x; w.y += scale * v.y; w.z += scale * v.z; w.w += scale * v.w;
    *reinterpret_cast<float4*>(o + c) = w;
  }
}
void embed_rows_scatter(const float* rows, int cap, int d, float* dE, cudaStream_t s, float scale) {
  if (cap == 0) return;
  if (d % 4) fail(HP_ECONFIG, "embedding rows: d_model must be a multiple of 4");
  emb_scatter_kernel<<<(cap + 7) / 8, 256, 0, s>>>(rows, cap, d, dE, scale);
  LAUNCH_CHECK();
  count_launch();
}

void embed_bwd_rows(const DevBatch& b, int d, const void* dx, DType xt, float* rows, int cap,
                    float* dseg0, float* dseg1, float* scratch, cudaStream_t s) {
  emb_slot_ids_kernel<<<(cap + 255) / 256, 256, 0, s>>>(b.ucount, b.uid, rows, cap, d + 4);
  LAUNCH_CHECK();
  count_launch();
  embed_bwd_impl(b, d, dx, xt, rows + 4, d + 4, 1, dseg0, dseg1, scratch, s);
}

void embed_bwd(const DevBatch& b, int d, const void* dx, DType xt, float* dE,
               float* dseg0, float* dseg1, float* scratch, cudaStream_t s) {
  embed_bwd_impl(b, d, dx, xt, dE, d, 0, dseg0, dseg1, scratch, s);
}

static void embed_bwd_impl(const DevBatch& b, int d, const void* dx, DType xt, float* dE,
                           int64_t ostride, int by_slot, float* dseg0, float* dseg1,
                           float* scratch, cudaStream_t s) {
  if (b.T == 0) return;
  DISPATCH1(xt, X, {
    if (d % 8) fail(HP_ECONFIG, "embedding gradient: d_model must be a multiple of 8");
    {
      const int sm = 32 * d * (int)sizeof(float);
      static int set_for = 0;
      if (sm > 48 * 1024 && sm > set_for) {
        HP_CUDA(cudaFuncSetAttribute(embed_grad_kernel<X>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        set_for = sm;
      }
      // 64 hot-id blocks + 148 blocks of 32 warps for the small ids
      embed_grad_kernel<X><<<kEmbHotBlocks + 148, 1024, sm, s>>>(b.ucount, b.ulist, b.uid, b.useg,
                                                                  b.perm, d, (const X*)dx, dE,
                                                                  ostride, by_slot);
      LAUNCH_CHECK();
    }
    count_launch(1);
    if (dseg0) {
      // both segment rows in one pass over dx (rows of 32, 8 columns a thread)
      const int rows_per = 32, chunks = (b.T + rows_per - 1) / rows_per;
      dim3 g1((d / 8 + 127) / 128, chunks);
      segsum_partial_vec<X><<<g1, 128, 0, s>>>(b.T, d, (const X*)dx, b.seg, rows_per, scratch);
      LAUNCH_CHECK();
      if (dseg1 == dseg0 + d) {  // canonical order: seg0 then seg1, adjacent
        colsum_final_strided<<<FINAL_LAUNCH(2 * d), 0, s>>>(chunks, 2 * d, 2 * d, scratch, dseg0);
        LAUNCH_CHECK();
        count_launch(2);
      } else {
        colsum_final_strided<<<FINAL_LAUNCH(d), 0, s>>>(chunks, 2 * d, d, scratch, dseg0);
        colsum_final_strided<<<FINAL_LAUNCH(d), 0, s>>>(chunks, 2 * d, d, scratch + d, dseg1);
        LAUNCH_CHECK();
        count_launch(3);
      }
    }
  });
}

void col_sum(int R, int N, const void* x, int64_t ld, DType t, float* out,
             float* scratch, cudaStream_t s, DeferredFinal* df) {
  if (df) df->queued = false;
  DISPATCH1(t, X, colsum_launch<X>(R, N, (const X*)x, ld, nullptr, 0, out, scratch, s, df));
}

size_t colsum_part_floats(int R, int N) {
  // LayerNorm-backward partials ([R / kLnBwdRows][3N]) or column-sum partials ([R / 32][N8])
  const size_t ln = (size_t)((R + kLnBwdRows - 1) / kLnBwdRows) * 3 * (size_t)N;
  const size_t cs = (size_t)((R + 31) / 32) * (size_t)((N + 7) & ~7);
  return std::max(ln, cs) + 64;
}

size_t colsum_scratch_floats(int R, int N) {
  const size_t a = (size_t)((R + kColRows - 1) / kColRows) * (N + 8) * 2;   // scalar path (+LN 2d)
  const size_t b = (size_t)((R + 31) / 32) * (((N + 7) & ~7));             // vector path
  const size_t c = (size_t)((R + kLnBwdRows - 1) / kLnBwdRows) * 3 * N;    // LN bwd partials
  return std::max(a, std::max(b, c)) + 3 * (size_t)N + 64;
}

// ------------------------------------------------------------------ LayerNorm
static constexpr float kLnEps = 1e-12f;

template <class XT, class YT>
__global__ void ln_fwd_kernel(int T, int d, const XT* __restrict__ x, const float* __restrict__ g,
                              const float* __restrict__ bta, YT* __restrict__ y,
                              float* __restrict__ mean, float* __restrict__ rstd) {
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= T) return;
  const int lane = threadIdx.x & 31;
  const XT* xr = x + (int64_t)t * d;
  float s = 0.f;
  for (int c = lane; c < d; c += 32) s += tof(xr[c]);
  const float mu = warp_sum(s) / d;
  float v = 0.f;
  for (int c = lane; c < d; c += 32) {
    const float q = tof(xr[c]) - mu;
    v += q * q;
  }
  const float rs = rsqrtf(warp_sum(v) / d + kLnEps);
  for (int c = lane; c < d; c += 32)
    y[(int64_t)t * d + c] = fromf<YT>((tof(xr[c]) - mu) * rs * g[c] + bta[c]);
  if (lane == 0) {
    mean[t] = mu;
    rstd[t] = rs;
  }
}

template <class DYT, class XT, class DXT>
__global__ void ln_bwd_kernel(int T, int d, const DYT* __restrict__ dy, const XT* __restrict__ x,
                              const float* __restrict__ mean, const float* __restrict__ rstd,
                              const float* __restrict__ g, DXT* __restrict__ dx) {
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= T) return;
  const int lane = threadIdx.x & 31;
  const float mu = mean[t], rs = rstd[t];
  const DYT* dyr = dy + (int64_t)t * d;
  const XT* xr = x + (int64_t)t * d;
  float s1 = 0.f, s2 = 0.f;
  for (int c = lane; c < d; c += 32) {
    const float xh = (tof(xr[c]) - mu) * rs;
    const float dxh = tof(dyr[c]) * g[c];
    s1 += dxh;
    s2 += dxh * xh;
  }
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
  const float inv_d = 1.f / d;
  for (int c = lane; c < d; c += 32) {
    const float xh = (tof(xr[c]) - mu) * rs;
    const float dxh = tof(dyr[c]) * g[c];
    dx[(int64_t)t * d + c] = fromf<DXT>(rs * (dxh - (s1 + xh * s2) * inv_d));
  }
}

template <class DYT, class XT>
__global__ void ln_pgrad_partial(int T, int d, const DYT* __restrict__ dy, const XT* __restrict__ x,
                                 const float* __restrict__ mean, const float* __restrict__ rstd,
                                 int rows_per, float* __restrict__ part) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= d) return;
  const int r0 = blockIdx.y * rows_per, r1 = min(T, r0 + rows_per);
  float ag = 0.f, ab = 0.f;
  for (int r = r0; r < r1; ++r) {
    const float g = tof(dy[(int64_t)r * d + c]);
    ag += g * (tof(x[(int64_t)r * d + c]) - mean[r]) * rstd[r];
    ab += g;
  }
  part[(int64_t)blockIdx.y * 2 * d + c] = ag;
  part[(int64_t)blockIdx.y * 2 * d + d + c] = ab;
}

// ---- vectorized bf16 LayerNorm (d = 256 * NV): each lane keeps NV x 8
// elements of its row in registers; 16-byte loads/stores.
template <int NV>
__global__ void __launch_bounds__(256) ln_fwd_vec(int T, const bf16* __restrict__ x,
                                                  const float* __restrict__ g,
                                                  const float* __restrict__ bta, bf16* __restrict__ y,
                                                  float* __restrict__ mean, float* __restrict__ rstd) {
  constexpr int d = 256 * NV;
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= T) return;
  const int lane = threadIdx.x & 31;
  float v[NV * 8];
  const bf16* xr = x + (int64_t)t * d;
  float4 gq[NV * 2], bq[NV * 2];  // gamma/beta issued with the row loads
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    unpack8(*reinterpret_cast<const uint4*>(xr + 8 * lane + 256 * j), v + 8 * j);
    gq[2 * j] = __ldg(reinterpret_cast<const float4*>(g + 8 * lane + 256 * j));
    gq[2 * j + 1] = __ldg(reinterpret_cast<const float4*>(g + 8 * lane + 256 * j) + 1);
    bq[2 * j] = __ldg(reinterpret_cast<const float4*>(bta + 8 * lane + 256 * j));
    bq[2 * j + 1] = __ldg(reinterpret_cast<const float4*>(bta + 8 * lane + 256 * j) + 1);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NV * 8; ++i) s += v[i];
  const float mu = warp_sum(s) * (1.f / d);
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < NV * 8; ++i) q += (v[i] - mu) * (v[i] - mu);
  const float rs = rsqrtf(warp_sum(q) * (1.f / d) + kLnEps);
  bf16* yr = y + (int64_t)t * d;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const int c0 = 8 * lane + 256 * j;
    const float* gg = reinterpret_cast<const float*>(&gq[2 * j]);
    const float* bb = reinterpret_cast<const float*>(&bq[2 * j]);
    float o[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) o[e] = (v[8 * j + e] - mu) * rs * gg[e] + bb[e];
    *reinterpret_cast<uint4*>(yr + c0) = pack8(o);
  }
  if (lane == 0) {
    mean[t] = mu;
    rstd[t] = rs;
  }
}

// dx = LN'(dy) plus per-block partial column sums of dy*xhat (dgamma), dy
// (dbeta) and dx (the bias gradient of the layer that produced x, which the
// residual makes equal to colsum(dx)).  Deterministic: fixed reduction order.
template <int NV>
__global__ void __launch_bounds__(256) ln_bwd_vec(int T, const bf16* __restrict__ dy,
                                                  const bf16* __restrict__ x,
                                                  const float* __restrict__ mean,
                                                  const float* __restrict__ rstd,
                                                  const float* __restrict__ g, bf16* __restrict__ dx,
                                                  float* __restrict__ part) {
  constexpr int d = 256 * NV;
  extern __shared__ float red[];  // [8 warps][3][d]
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float ag[NV * 8], ab[NV * 8], ax[NV * 8];
#pragma unroll
  for (int i = 0; i < NV * 8; ++i) ag[i] = ab[i] = ax[i] = 0.f;
  float gg[NV * 8];
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(g + 8 * lane + 256 * j));
    const float4 b = __ldg(reinterpret_cast<const float4*>(g + 8 * lane + 256 * j) + 1);
    gg[8 * j + 0] = a.x; gg[8 * j + 1] = a.y; gg[8 * j + 2] = a.z; gg[8 * j + 3] = a.w;
    gg[8 * j + 4] = b.x; gg[8 * j + 5] = b.y; gg[8 * j + 6] = b.z; gg[8 * j + 7] = b.w;
  }
  for (int rr = w; rr < kLnBwdRows; rr += 8) {
    const int t = blockIdx.x * kLnBwdRows + rr;
    if (t >= T) break;
    const float mu = mean[t], rs = rstd[t];
    float xh[NV * 8], gy[NV * 8];
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      unpack8(*reinterpret_cast<const uint4*>(x + (int64_t)t * d + 8 * lane + 256 * j), xh + 8 * j);
      unpack8(*reinterpret_cast<const uint4*>(dy + (int64_t)t * d + 8 * lane + 256 * j), gy + 8 * j);
    }
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < NV * 8; ++i) {
      xh[i] = (xh[i] - mu) * rs;
      const float dxh = gy[i] * gg[i];
      s1 += dxh;
      s2 += dxh * xh[i];
      ag[i] += gy[i] * xh[i];
      ab[i] += gy[i];
    }
    s1 = warp_sum(s1) * (1.f / d);
    s2 = warp_sum(s2) * (1.f / d);
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      float o[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int i = 8 * j + e;
        o[e] = rs * (gy[i] * gg[i] - (s1 + xh[i] * s2));
      }
      const uint4 u = pack8(o);
      *reinterpret_cast<uint4*>(dx + (int64_t)t * d + 8 * lane + 256 * j) = u;
      float r[8];
      unpack8(u, r);  // sum what the next kernel will read
#pragma unroll
      for (int e = 0; e < 8; ++e) ax[8 * j + e] += r[e];
    }
  }
#pragma unroll
  for (int j = 0; j < NV; ++j)
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int c = 8 * lane + 256 * j + e;
      red[(w * 3 + 0) * d + c] = ag[8 * j + e];
      red[(w * 3 + 1) * d + c] = ab[8 * j + e];
      red[(w * 3 + 2) * d + c] = ax[8 * j + e];
    }
  __syncthreads();
  for (int c = threadIdx.x; c < 3 * d; c += blockDim.x) {
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) acc += red[k * 3 * d + c];
    part[(int64_t)blockIdx.x * 3 * d + c] = acc;
  }
}

// ---- bulk-fed bf16 LayerNorm (d = 256 * NV).  Each warp owns RPW
// consecutive rows and fetches them with ONE 1-D bulk copy per operand
// (cp.async.bulk, completion on the warp's mbarrier), so a CTA's whole row
// block is in flight at once and the load latency is paid once; the math then
// reads shared memory.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          tc::smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(tc::smem_u32(bar))
      : "memory");
}
// warp-private mbarrier: lane 0 initialises and arms it, every lane waits
__device__ __forceinline__ void warp_bar_init(uint64_t* bar, int lane) {
  if (lane == 0) {
    tc::mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
}

#ifndef HP_LN_FWD_RPW
#define HP_LN_FWD_RPW 2
#endif
constexpr int kLnFwdRpw = HP_LN_FWD_RPW;  // rows per warp (8 warps per CTA)
template <int NV>
__global__ void __launch_bounds__(256) ln_fwd_bulk(int T, const bf16* __restrict__ x,
                                                   const float* __restrict__ g,
                                                   const float* __restrict__ bta, bf16* __restrict__ y,
                                                   float* __restrict__ mean, float* __restrict__ rstd) {
  constexpr int d = 256 * NV;
  extern __shared__ __align__(128) uint8_t lsm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(lsm);
  bf16* xs = reinterpret_cast<bf16*>(lsm + 128);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row0 = (blockIdx.x * 8 + w) * kLnFwdRpw;
  const int nr = min(kLnFwdRpw, T - row0);
  if (nr <= 0) return;
  bf16* xw = xs + w * kLnFwdRpw * d;
  warp_bar_init(&bar[w], lane);
  if (lane == 0) {
    tc::mbar_expect_tx(&bar[w], nr * d * 2);
    bulk_g2s(xw, x + (int64_t)row0 * d, nr * d * 2, &bar[w]);
  }
  float4 gq[NV * 2], bq[NV * 2];  // gamma / beta: loaded once for the warp's rows
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    gq[2 * j] = __ldg(reinterpret_cast<const float4*>(g + 8 * lane + 256 * j));
    gq[2 * j + 1] = __ldg(reinterpret_cast<const float4*>(g + 8 * lane + 256 * j) + 1);
    bq[2 * j] = __ldg(reinterpret_cast<const float4*>(bta + 8 * lane + 256 * j));
    bq[2 * j + 1] = __ldg(reinterpret_cast<const float4*>(bta + 8 * lane + 256 * j) + 1);
  }
  tc::mbar_wait(&bar[w], 0);
  for (int i = 0; i < nr; ++i) {
    const int t = row0 + i;
    float v[NV * 8];
#pragma unroll
    for (int j = 0; j < NV; ++j)
      unpack8(*reinterpret_cast<const uint4*>(xw + i * d + 8 * lane + 256 * j), v + 8 * j);
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < NV * 8; ++k) s += v[k];
    const float mu = warp_sum(s) * (1.f / d);
    float q = 0.f;
#pragma unroll
    for (int k = 0; k < NV * 8; ++k) q += (v[k] - mu) * (v[k] - mu);
    const float rs = rsqrtf(warp_sum(q) * (1.f / d) + kLnEps);
    bf16* yr = y + (int64_t)t * d;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const float* gg = reinterpret_cast<const float*>(&gq[2 * j]);
      const float* bb = reinterpret_cast<const float*>(&bq[2 * j]);
      float o[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = (v[8 * j + e] - mu) * rs * gg[e] + bb[e];
      *reinterpret_cast<uint4*>(yr + 8 * lane + 256 * j) = pack8(o);
    }
    if (lane == 0) {
      mean[t] = mu;
      rstd[t] = rs;
    }
  }
}

// Backward, kLnBwdRows rows per CTA (4 per warp), x and dy bulk-copied; the
// cross-warp partial reduction reuses the row buffers.
template <int NV>
__global__ void __launch_bounds__(256, 1) ln_bwd_bulk(int T, const bf16* __restrict__ dy,
                                                      const bf16* __restrict__ x,
                                                      const float* __restrict__ mean,
                                                      const float* __restrict__ rstd,
                                                      const float* __restrict__ g,
                                                      bf16* __restrict__ dx, float* __restrict__ part) {
  constexpr int d = 256 * NV;
  constexpr int RPW = kLnBwdRows / 8;
  extern __shared__ __align__(128) uint8_t lsm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(lsm);
  bf16* xs = reinterpret_cast<bf16*>(lsm + 128);
  bf16* ys = xs + kLnBwdRows * d;
  float* red = reinterpret_cast<float*>(lsm + 128);  // [8 warps][3][d], after the rows are consumed
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row0 = blockIdx.x * kLnBwdRows + w * RPW;
  const int nr = max(0, min(RPW, T - row0));
  warp_bar_init(&bar[w], lane);
  if (lane == 0 && nr > 0) {
    tc::mbar_expect_tx(&bar[w], 2 * nr * d * 2);
    bulk_g2s(xs + w * RPW * d, x + (int64_t)row0 * d, nr * d * 2, &bar[w]);
    bulk_g2s(ys + w * RPW * d, dy + (int64_t)row0 * d, nr * d * 2, &bar[w]);
  }
  float ag[NV * 8], ab[NV * 8], ax[NV * 8];
#pragma unroll
  for (int i = 0; i < NV * 8; ++i) ag[i] = ab[i] = ax[i] = 0.f;
  float gg[NV * 8];
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(g + 8 * lane + 256 * j));
    const float4 b = __ldg(reinterpret_cast<const float4*>(g + 8 * lane + 256 * j) + 1);
    gg[8 * j + 0] = a.x; gg[8 * j + 1] = a.y; gg[8 * j + 2] = a.z; gg[8 * j + 3] = a.w;
    gg[8 * j + 4] = b.x; gg[8 * j + 5] = b.y; gg[8 * j + 6] = b.z; gg[8 * j + 7] = b.w;
  }
  if (nr > 0) tc::mbar_wait(&bar[w], 0);
  for (int i = 0; i < nr; ++i) {
    const int t = row0 + i;
    const float mu = mean[t], rs = rstd[t];
    float xh[NV * 8], gy[NV * 8];
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      unpack8(*reinterpret_cast<const uint4*>(xs + (w * RPW + i) * d + 8 * lane + 256 * j), xh + 8 * j);
      unpack8(*reinterpret_cast<const uint4*>(ys + (w * RPW + i) * d + 8 * lane + 256 * j), gy + 8 * j);
    }
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int k = 0; k < NV * 8; ++k) {
      xh[k] = (xh[k] - mu) * rs;
      const float dxh = gy[k] * gg[k];
      s1 += dxh;
      s2 += dxh * xh[k];
      ag[k] += gy[k] * xh[k];
      ab[k] += gy[k];
    }
    s1 = warp_sum(s1) * (1.f / d);
    s2 = warp_sum(s2) * (1.f / d);
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      float o[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int k = 8 * j + e;
        o[e] = rs * (gy[k] * gg[k] - (s1 + xh[k] * s2));
      }
      const uint4 u = pack8(o);
      *reinterpret_cast<uint4*>(dx + (int64_t)t * d + 8 * lane + 256 * j) = u;
      float r[8];
      unpack8(u, r);  // sum what the next kernel will read
#pragma unroll
      for (int e = 0; e < 8; ++e) ax[8 * j + e] += r[e];
    }
  }
  __syncthreads();  // every warp is done with the row buffers
#pragma unroll
  for (int j = 0; j < NV; ++j)
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int c = 8 * lane + 256 * j + e;
      red[(w * 3 + 0) * d + c] = ag[8 * j + e];
      red[(w * 3 + 1) * d + c] = ab[8 * j + e];
      red[(w * 3 + 2) * d + c] = ax[8 * j + e];
    }
  __syncthreads();
  for (int c = threadIdx.x; c < 3 * d; c += blockDim.x) {
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) acc += red[k * 3 * d + c];
    part[(int64_t)blockIdx.x * 3 * d + c] = acc;
  }
}

// out0/out1/out2 = column sums of the [chunks x 3d] partials
__global__ void ln_part_final(int chunks, int d, const float* __restrict__ part, float* __restrict__ dg,
                              float* __restrict__ db, float* __restrict__ dbias) {
  const int c = blockIdx.x * 32 + threadIdx.x;
  const float acc = final_sum(chunks, 3 * d, part, c, c < 3 * d);
  if (threadIdx.y != 0 || c >= 3 * d) return;
  if (c < d) dg[c] = acc;
  else if (c < 2 * d) db[c - d] = acc;
  else if (dbias) dbias[c - 2 * d] = acc;
}

void layernorm_fwd(int T, int d, const void* x, DType xt, const float* g,
                   const float* bta, void* y, DType yt, float* mean, float* rstd,
                   cudaStream_t s) {
  if (T == 0) return;
  const int grid = (T + 7) / 8;
  if (xt == DType::bf16 && yt == DType::bf16 && d % 256 == 0 && d <= 1024) {
    const int rows_cta = 8 * kLnFwdRpw;
    const int gb = (T + rows_cta - 1) / rows_cta;
    const size_t sm = 128 + (size_t)rows_cta * d * 2;
    switch (d / 256) {
      case 1: launch_ex(ln_fwd_bulk<1>, dim3(gb), dim3(256), sm, s, 1, T, (const bf16*)x, g, bta, (bf16*)y, mean, rstd); break;
      case 2: launch_ex(ln_fwd_bulk<2>, dim3(gb), dim3(256), sm, s, 1, T, (const bf16*)x, g, bta, (bf16*)y, mean, rstd); break;
      case 3: launch_ex(ln_fwd_bulk<3>, dim3(gb), dim3(256), sm, s, 1, T, (const bf16*)x, g, bta, (bf16*)y, mean, rstd); break;
      default: launch_ex(ln_fwd_bulk<4>, dim3(gb), dim3(256), sm, s, 1, T, (const bf16*)x, g, bta, (bf16*)y, mean, rstd); break;
    }
  } else {
    DISPATCH1(xt, X, DISPATCH1(yt, Y,
        ln_fwd_kernel<X, Y><<<grid, 256, 0, s>>>(T, d, (const X*)x, g, bta, (Y*)y, mean, rstd)));
  }
  LAUNCH_CHECK();
  count_launch();
}

void layernorm_bwd(int T, int d, const void* dy, DType dyt, const void* x,
                   DType xt, const float* mean, const float* rstd, const float* g,
                   void* dx, DType dxt, float* dg, float* db, float* dbias, float* scratch,
                   cudaStream_t s, DeferredFinal* df) {
  if (df) df->queued = false;
  if (T == 0) return;
  float* part = df ? df->part : scratch;
  if (dyt == DType::bf16 && xt == DType::bf16 && dxt == DType::bf16 && d % 256 == 0 && d <= 1024) {
    const int chunks = (T + kLnBwdRows - 1) / kLnBwdRows;
    // rows (x, dy) and, later, the [8][3][d] reduction share the buffer
    const size_t sm = 128 + std::max(sizeof(float) * 8 * 3 * d, (size_t)2 * kLnBwdRows * d * 2);
    switch (d / 256) {
#define LNB(NV)                                                                                 \
  case NV: {                                                                                    \
    static size_t attr_##NV = 0;                                                                \
    if (attr_##NV < sm) {                                                                       \
      HP_CUDA(cudaFuncSetAttribute(ln_bwd_bulk<NV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); \
      attr_##NV = sm;                                                                           \
    }                                                                                           \
    launch_ex(ln_bwd_bulk<NV>, dim3(chunks), dim3(256), sm, s, 1, T, (const bf16*)dy,      \
               (const bf16*)x, mean, rstd, g, (bf16*)dx, part);                                 \
  } break;
      LNB(1) LNB(2) LNB(3) default: LNB(4)
#undef LNB
    }
    LAUNCH_CHECK();
    if (df) {
      count_launch();
      df->queued = true;
      df->kind = 0;
      df->chunks = chunks;
      df->d = d;
      df->o0 = dg;
      df->o1 = db;
      df->o2 = dbias;
      return;
    }
    ln_part_final<<<FINAL_LAUNCH(3 * d), 0, s>>>(chunks, d, scratch, dg, db, dbias);
    LAUNCH_CHECK();
    count_launch(2);
    return;
  }
  DISPATCH1(dyt, DY, DISPATCH1(xt, X, {
    DISPATCH1(dxt, DX, ln_bwd_kernel<DY, X, DX><<<(T + 7) / 8, 256, 0, s>>>(
        T, d, (const DY*)dy, (const X*)x, mean, rstd, g, (DX*)dx));
    LAUNCH_CHECK();
    const int chunks = (T + kColRows - 1) / kColRows;
    ln_pgrad_partial<DY, X><<<dim3((d + 127) / 128, chunks), 128, 0, s>>>(
        T, d, (const DY*)dy, (const X*)x, mean, rstd, kColRows, scratch);
    LAUNCH_CHECK();
    // final: rows of 2d partials -> dg | db
    colsum_final_kernel<<<FINAL_LAUNCH(2 * d), 0, s>>>(chunks, 2 * d, scratch, scratch + (int64_t)chunks * 2 * d);
    LAUNCH_CHECK();
    HP_CUDA(cudaMemcpyAsync(dg, scratch + (int64_t)chunks * 2 * d, sizeof(float) * d, cudaMemcpyDeviceToDevice, s));
    HP_CUDA(cudaMemcpyAsync(db, scratch + (int64_t)chunks * 2 * d + d, sizeof(float) * d, cudaMemcpyDeviceToDevice, s));
    count_launch(3);
    if (dbias)
      DISPATCH1(dxt, DX, colsum_launch<DX>(T, d, (const DX*)dx, d, nullptr, 0, dbias, scratch, s));
  }));
}

void launch_final(const DeferredFinal& f, cudaStream_t s) {
  if (!f.queued) return;
  if (f.kind == 0) {
    ln_part_final<<<FINAL_LAUNCH(3 * f.d), 0, s>>>(f.chunks, f.d, f.part, f.o0, f.o1, f.o2);
  } else {
    colsum_final_strided<<<FINAL_LAUNCH(f.n), 0, s>>>(f.chunks, f.stride, f.n, f.part, f.o0);
  }
  LAUNCH_CHECK();
  count_launch();
}

// ------------------------------------------------------------------ attention
// One CTA per (instance, head); the whole (<=128 token) sequence lives in
// shared memory in fp32.  smem_mm is a register-blocked (8x8 / 8x4) product
// C(i,j) = sum_k A(i,k) B(k,j) over strided smem operands.
struct SMat {
  const float* p;
  int si, sk;  // A: (i,k) ; B: (k,j) strides
};

template <int BR, int BC, class Store>
__device__ __forceinline__ void smem_mm_t(int n1, int n2, int kd, SMat A, SMat B, Store store) {
  const int ti_n = (n1 + BR - 1) / BR, tj_n = (n2 + BC - 1) / BC;
  for (int t = threadIdx.x; t < ti_n * tj_n; t += blockDim.x) {
    const int i0 = (t / tj_n) * BR, j0 = (t % tj_n) * BC;
    float acc[BR][BC];
#pragma unroll
    for (int r = 0; r < BR; ++r)
#pragma unroll
      for (int c = 0; c < BC; ++c) acc[r][c] = 0.f;
    for (int k = 0; k < kd; ++k) {
      float a[BR], bb[BC];
#pragma unroll
      for (int r = 0; r < BR; ++r) a[r] = A.p[(i0 + r) * A.si + k * A.sk];
#pragma unroll
      for (int c = 0; c < BC; ++c) bb[c] = B.p[k * B.si + (j0 + c) * B.sk];
#pragma unroll
      for (int r = 0; r < BR; ++r)
#pragma unroll
        for (int c = 0; c < BC; ++c) acc[r][c] += a[r] * bb[c];
    }
#pragma unroll
    for (int r = 0; r < BR; ++r)
#pragma unroll
      for (int c = 0; c < BC; ++c)
        if (i0 + r < n1 && j0 + c < n2) store(i0 + r, j0 + c, acc[r][c]);
  }
}
// register blocks of 8 x 8 (8 x 4 for the 64-column products): one block per
// thread at 128 x 128 / 128 x 64, a quarter / three eighths of a shared-memory
// load per FMA; every element's k-sum runs in the same order as any blocking.
// Operand rows past n1 / n2 (up to the next multiple of 8) are read but never
// stored: the arrays are packed in an allocation sized for 128-row operands.
template <class Store>
__device__ void smem_mm(int n1, int n2, int kd, SMat A, SMat B, Store store) {
  if (n2 > 64) smem_mm_t<8, 8>(n1, n2, kd, A, B, store);
  else smem_mm_t<8, 4>(n1, n2, kd, A, B, store);
}

template <class T>
__device__ void load_head(float* dst, int ld_dst, int n, int n4, int dk, const T* src,
                          int64_t row0, int64_t ld_src, int col0) {
  for (int e = threadIdx.x; e < n4 * dk; e += blockDim.x) {
    const int i = e / dk, c = e % dk;
    dst[i * ld_dst + c] = i < n ? tof(src[(row0 + i) * ld_src + col0 + c]) : 0.f;
  }
}

template <class T>
__global__ void attn_fwd_kernel(const AttnArgs a) {
  extern __shared__ float sm[];
  const int b = blockIdx.x, h = blockIdx.y, dk = a.dk;
  const int rq = a.cu_q[b], nq = a.cu_q[b + 1] - rq;
  const int rk = a.cu_kv[b], nk = a.cu_kv[b + 1] - rk;
  if (nq <= 0 || nk <= 0) return;
  const int nq4 = (nq + 3) & ~3, nk4 = (nk + 3) & ~3, ldh = dk + 1, lds = nk4 + 1;
  const int d = a.H * dk;
  float* Q = sm;
  float* K = Q + nq4 * ldh;
  float* V = K + nk4 * ldh;
  float* S = V + nk4 * ldh;
  load_head(Q, ldh, nq, nq4, dk, (const T*)a.q, rq, a.ldq, a.qcol + h * dk);
  load_head(K, ldh, nk, nk4, dk, (const T*)a.k, rk, a.ldk, a.kcol + h * dk);
  load_head(V, ldh, nk, nk4, dk, (const T*)a.v, rk, a.ldv, a.vcol + h * dk);
  __syncthreads();
  // scores = (Q K^T) * (1/sqrt(dk))   attention.hpp:21-23; causal: keys j <= i
  const float scale = 1.f / sqrtf((float)dk);
  const int causal = a.causal;
  smem_mm(nq, nk, dk, SMat{Q, ldh, 1}, SMat{K, 1, ldh},
          [&](int i, int j, float v) { S[i * lds + j] = (causal && j > i) ? -FLT_MAX : v * scale; });
  __syncthreads();
  // row softmax with max shift (tape.hpp:129-137)
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int i = w; i < nq; i += nw) {
    float* r = S + i * lds;
    const int nj = causal ? min(nk, i + 1) : nk;
    float mx = -FLT_MAX;
    for (int j = lane; j < nj; j += 32) mx = fmaxf(mx, r[j]);
    mx = warp_max(mx);
    float se = 0.f;
    for (int j = lane; j < nk; j += 32) {
      const float e = j < nj ? expf(r[j] - mx) : 0.f;
      r[j] = e;
      se += e;
    }
    se = warp_sum(se);
    const float inv = 1.f / se;
    for (int j = lane; j < nk; j += 32) r[j] = r[j] * inv;
    if (lane == 0) a.lse[(int64_t)h * a.T_q + rq + i] = mx + logf(se);
  }
  __syncthreads();
  // O = P V -> columns h*dk.. of the concat (concat_cols order)
  T* o = (T*)a.o;
  smem_mm(nq, dk, nk, SMat{S, lds, 1}, SMat{V, ldh, 1}, [&](int i, int c, float v) {
    o[(int64_t)(rq + i) * d + h * dk + c] = fromf<T>(v);
  });
}

template <class T>
__global__ void attn_bwd_kernel(const AttnArgs a) {
  extern __shared__ float sm[];
  const int b = blockIdx.x, h = blockIdx.y, dk = a.dk;
  const int rq = a.cu_q[b], nq = a.cu_q[b + 1] - rq;
  const int rk = a.cu_kv[b], nk = a.cu_kv[b + 1] - rk;
  if (nq <= 0 || nk <= 0) return;
  const int nq4 = (nq + 3) & ~3, nk4 = (nk + 3) & ~3, ldh = dk + 1, lds = nk4 + 1;
  const int d = a.H * dk;
  float* Q = sm;
  float* K = Q + nq4 * ldh;
  float* V = K + nk4 * ldh;
  float* G = V + nk4 * ldh;  // dO
  float* S = G + nq4 * ldh;
  float* D = S + nq4 * lds;  // rowsum(dO * O)
  const T* o = (const T*)a.o;
  load_head(Q, ldh, nq, nq4, dk, (const T*)a.q, rq, a.ldq, a.qcol + h * dk);
  load_head(K, ldh, nk, nk4, dk, (const T*)a.k, rk, a.ldk, a.kcol + h * dk);
  load_head(V, ldh, nk, nk4, dk, (const T*)a.v, rk, a.ldv, a.vcol + h * dk);
  load_head(G, ldh, nq, nq4, dk, (const T*)a.dO, rq, d, h * dk);
  __syncthreads();  // D below reads rows other warps loaded
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int i = w; i < nq; i += nw) {
    float acc = 0.f;
    for (int c = lane; c < dk; c += 32) acc += G[i * ldh + c] * tof(o[(int64_t)(rq + i) * d + h * dk + c]);
    acc = warp_sum(acc);
    if (lane == 0) D[i] = acc;
  }
  __syncthreads();
  const float scale = 1.f / sqrtf((float)dk);
  const int causal = a.causal;
  // P = exp(S*scale - lse); masked keys 0
  smem_mm(nq, nk, dk, SMat{Q, ldh, 1}, SMat{K, 1, ldh}, [&](int i, int j, float v) {
    S[i * lds + j] = (causal && j > i) ? 0.f : expf(v * scale - a.lse[(int64_t)h * a.T_q + rq + i]);
  });
  __syncthreads();
  // dV = P^T dO
  T* dv = (T*)a.dv;
  smem_mm(nk, dk, nq, SMat{S, 1, lds}, SMat{G, ldh, 1}, [&](int j, int c, float v) {
    dv[(int64_t)(rk + j) * a.lddv + a.dvcol + h * dk + c] = fromf<T>(v);
  });
  __syncthreads();
  // dS = P * (dO V^T - D)   (tape.hpp:274-286), in place
  smem_mm(nq, nk, dk, SMat{G, ldh, 1}, SMat{V, 1, ldh}, [&](int i, int j, float v) {
    float* p = S + i * lds + j;
    *p = *p * (v - D[i]) * scale;
  });
  __syncthreads();
  // dQ = dS K ; dK = dS^T Q
  T* dq = (T*)a.dq;
  T* dkk = (T*)a.dk_;
  smem_mm(nq, dk, nk, SMat{S, lds, 1}, SMat{K, ldh, 1}, [&](int i, int c, float v) {
    dq[(int64_t)(rq + i) * a.lddq + a.dqcol + h * dk + c] = fromf<T>(v);
  });
  smem_mm(nk, dk, nq, SMat{S, 1, lds}, SMat{Q, ldh, 1}, [&](int j, int c, float v) {
    dkk[(int64_t)(rk + j) * a.lddk + a.dkcol + h * dk + c] = fromf<T>(v);
  });
}

static size_t attn_smem(int nq4, int nk4, int dk, bool bwd) {
  const int ldh = dk + 1, lds = nk4 + 1;
  return sizeof(float) * ((size_t)(bwd ? 2 : 1) * nq4 * ldh + 2 * (size_t)nk4 * ldh +
                          (size_t)nq4 * lds + (bwd ? nq4 : 0));
}

static constexpr int kAttnMaxSeq = 128;

static void attn_check(const AttnArgs& a) {
  if (a.max_q > kAttnMaxSeq || a.max_kv > kAttnMaxSeq)
    fail(HP_ECONFIG, "attention: sequences longer than 128 need the bf16 blocked kernels");
}

void attention_simt_fwd(const AttnArgs& a, DType t, cudaStream_t s) {
  if (a.B == 0) return;
  attn_check(a);
  const size_t sm = attn_smem(kAttnMaxSeq, kAttnMaxSeq, a.dk, false);
  DISPATCH1(t, X, {
    static size_t set = 0;
    if (set < sm) {
      HP_CUDA(cudaFuncSetAttribute(attn_fwd_kernel<X>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      set = sm;
    }
    attn_fwd_kernel<X><<<dim3(a.B, a.H), 256, sm, s>>>(a);
  });
  LAUNCH_CHECK();
  count_launch();
}

void attention_simt_bwd(const AttnArgs& a, DType t, cudaStream_t s) {
  if (a.B == 0) return;
  attn_check(a);
  const size_t sm = attn_smem(kAttnMaxSeq, kAttnMaxSeq, a.dk, true);
  DISPATCH1(t, X, {
    static size_t set = 0;
    if (set < sm) {
      HP_CUDA(cudaFuncSetAttribute(attn_bwd_kernel<X>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      set = sm;
    }
    attn_bwd_kernel<X><<<dim3(a.B, a.H), 256, sm, s>>>(a);
  });
  LAUNCH_CHECK();
  count_launch();
}

AttnArgs self_attn_args(const DevBatch& b, int H, int dk, int max_seq, const void* qkv, void* o,
                        float* lse, const void* dO, void* dqkv, int causal) {
  AttnArgs a;
  const int d = H * dk;
  a.B = b.B; a.H = H; a.dk = dk;
  a.cu_q = a.cu_kv = b.cu;
  a.T_q = a.T_kv = b.T;
  a.max_q = a.max_kv = max_seq;
  a.q = a.k = a.v = qkv;
  a.ldq = a.ldk = a.ldv = 3 * (int64_t)d;
  a.qcol = 0; a.kcol = d; a.vcol = 2 * d;
  a.o = o; a.lse = lse; a.causal = causal;
  a.dO = dO;
  a.dq = a.dk_ = a.dv = dqkv;
  a.lddq = a.lddk = a.lddv = 3 * (int64_t)d;
  a.dqcol = 0; a.dkcol = d; a.dvcol = 2 * d;
  return a;
}

void attention_fwd(const DevBatch& b, int H, int dk, const void* qkv, void* o,
                   float* lse, DType t, cudaStream_t s) {
  attention_simt_fwd(self_attn_args(b, H, dk, kAttnMaxSeq, qkv, o, lse), t, s);
}

void attention_bwd(const DevBatch& b, int H, int dk, const void* qkv,
                   const void* o, const void* dO, const float* lse, void* dqkv,
                   DType t, cudaStream_t s) {
  attention_simt_bwd(self_attn_args(b, H, dk, kAttnMaxSeq, qkv, const_cast<void*>(o),
                                    const_cast<float*>(lse), dO, dqkv), t, s);
}

bool attention2_tc_ok(const AttnArgs& a, DType t) {
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  return t == DType::bf16 && a.dk == 64 && a.max_q <= 128 && a.max_kv <= 128 &&
         al16(a.q) && al16(a.k) && al16(a.v) && a.ldq % 8 == 0 && a.ldk % 8 == 0 &&
         a.ldv % 8 == 0 && a.qcol % 8 == 0 && a.kcol % 8 == 0 && a.vcol % 8 == 0;
}

void attention2_fwd(const AttnArgs& a, DType t, cudaStream_t s) {
  if (attention2_tc_ok(a, t))
    attention_tc_fwd(a, s);
  else
    attention_simt_fwd(a, t, s);
}

void attention2_bwd(const AttnArgs& a, DType t, cudaStream_t s) {
  if (attention2_tc_ok(a, t))
    attention_tc_bwd(a, s);
  else
    attention_simt_bwd(a, t, s);
}

// ------------------------------------------------------------------ rows
template <class T>
__global__ void gather_kernel(int R, int d, const int* __restrict__ idx, const T* __restrict__ src,
                              T* __restrict__ dst) {
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= R) return;
  const int lane = threadIdx.x & 31;
  const int i = idx[r];
  if (i < 0) {  // padding row (see Engine::stage_batch): zeros
    for (int c = lane; c < d; c += 32) dst[(int64_t)r * d + c] = fromf<T>(0.f);
    return;
  }
  const T* s = src + (int64_t)i * d;
  for (int c = lane; c < d; c += 32) dst[(int64_t)r * d + c] = s[c];
}
template <class T>
__global__ void scatter_kernel(int R, int d, const int* __restrict__ idx, const T* __restrict__ src,
                               T* __restrict__ dst) {
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= R) return;
  const int lane = threadIdx.x & 31;
  if (idx[r] < 0) return;  // padding row
  T* o = dst + (int64_t)idx[r] * d;
  for (int c = lane; c < d; c += 32) o[c] = src[(int64_t)r * d + c];
}
void gather_rows(int R, int d, const int* idx, const void* src, void* dst, DType t,
                 cudaStream_t s) {
  if (R == 0) return;
  DISPATCH1(t, X, gather_kernel<X><<<(R + 7) / 8, 256, 0, s>>>(R, d, idx, (const X*)src, (X*)dst));
  LAUNCH_CHECK();
  count_launch();
}
template <class T>
__global__ void scatter_f32_kernel(int R, int d, const int* __restrict__ idx,
                                   const float* __restrict__ src, T* __restrict__ dst) {
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= R) return;
  const int lane = threadIdx.x & 31;
  if (idx[r] < 0) return;  // padding row
  T* o = dst + (int64_t)idx[r] * d;
  for (int c = lane; c < d; c += 32) o[c] = fromf<T>(src[(int64_t)r * d + c]);
}
void scatter_rows_f32(int R, int d, const int* idx, const float* src, void* dst, DType t,
                      cudaStream_t s) {
  if (R == 0) return;
  DISPATCH1(t, X, scatter_f32_kernel<X><<<(R + 7) / 8, 256, 0, s>>>(R, d, idx, src, (X*)dst));
  LAUNCH_CHECK();
  count_launch();
}
void scatter_rows(int R, int d, const int* idx, const void* src, void* dst,
                  DType t, cudaStream_t s) {
  if (R == 0) return;
  DISPATCH1(t, X, scatter_kernel<X><<<(R + 7) / 8, 256, 0, s>>>(R, d, idx, (const X*)src, (X*)dst));
  LAUNCH_CHECK();
  count_launch();
}

// ------------------------------------------------------------------ ls_ce
template <class DZT>
__global__ void __launch_bounds__(512) ls_ce_kernel(int V, const float* __restrict__ z, int64_t ldz,
                             const int* __restrict__ target, float eps,
                             float* __restrict__ row_loss, DZT* __restrict__ dz, int64_t ld_dz) {
  __shared__ float red[32];
  const int r = blockIdx.x;
  if (target[r] < 0) {  // padding row (see Engine::stage_batch): no loss, no gradient
    if (threadIdx.x == 0) row_loss[r] = 0.f;
    if (dz)
      for (int j = threadIdx.x; j < V; j += blockDim.x) dz[(int64_t)r * ld_dz + j] = fromf<DZT>(0.f);
    return;
  }
  const float* zr = z + (int64_t)r * ldz;
  // one pass: running max, rescaled sum of exp, and the plain sum (for eps)
  // fp32 parity path: accurate expf; bf16 path: fast __expf
  auto ex = [](float x) { return std::is_same<DZT, float>::value ? expf(x) : __expf(x); };
  float mx = -FLT_MAX, se = 0.f, zs = 0.f;
  const int V4 = (reinterpret_cast<uintptr_t>(zr) & 15) == 0 ? (V & ~3) : 0;
  for (int j = 4 * threadIdx.x; j < V4; j += 4 * blockDim.x) {
    const float4 q = *reinterpret_cast<const float4*>(zr + j);
    const float m4 = fmaxf(fmaxf(q.x, q.y), fmaxf(q.z, q.w));
    if (m4 > mx) {
      se *= ex(mx - m4);
      mx = m4;
    }
    se += ex(q.x - mx) + ex(q.y - mx) + ex(q.z - mx) + ex(q.w - mx);
    zs += (q.x + q.y) + (q.z + q.w);
  }
  for (int j = V4 + threadIdx.x; j < V; j += blockDim.x) {
    const float v = zr[j];
    if (v > mx) {
      se *= ex(mx - v);
      mx = v;
    }
    se += ex(v - mx);
    zs += v;
  }
  const float gmx = block_max<512>(mx, red);
  se = block_sum<512>(mx == -FLT_MAX ? 0.f : se * ex(mx - gmx), red);
  zs = block_sum<512>(zs, red);
  mx = gmx;
  const int t = target[r];
  const float invV = eps / (float)V;
  if (threadIdx.x == 0) {
    const float lse = mx + logf(se);
    row_loss[r] = lse - (1.f - eps) * zr[t] - invV * zs;
  }
  if (dz) {
    const float inv_se = 1.f / se;
    DZT* o = dz + (int64_t)r * ld_dz;
    const int V4w = (std::is_same<DZT, bf16>::value && (reinterpret_cast<uintptr_t>(o) & 7) == 0) ? V4 : 0;
    for (int j = 4 * threadIdx.x; j < V4w; j += 4 * blockDim.x) {
      const float4 q = *reinterpret_cast<const float4*>(zr + j);
      float g[4] = {__expf(q.x - mx) * inv_se - invV, __expf(q.y - mx) * inv_se - invV,
                    __expf(q.z - mx) * inv_se - invV, __expf(q.w - mx) * inv_se - invV};
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (j + e == t) g[e] -= 1.f - eps;
      __nv_bfloat162 h0 = __floats2bfloat162_rn(g[0], g[1]), h1 = __floats2bfloat162_rn(g[2], g[3]);
      uint2 u;
      u.x = *reinterpret_cast<uint32_t*>(&h0);
      u.y = *reinterpret_cast<uint32_t*>(&h1);
      *reinterpret_cast<uint2*>(reinterpret_cast<bf16*>(o) + j) = u;
    }
    for (int j = V4w + threadIdx.x; j < V; j += blockDim.x) {
      float g = expf(zr[j] - mx) * inv_se - invV;
      if (j == t) g -= 1.f - eps;
      o[j] = fromf<DZT>(g);
    }
  }
}

void ls_ce(int R, int V, const float* z, int64_t ldz, const int* target,
           float eps, float* row_loss, void* dz, DType dzt, int64_t ld_dz,
           cudaStream_t s) {
  if (R == 0) return;
  DISPATCH1(dzt, X, ls_ce_kernel<X><<<R, 512, 0, s>>>(V, z, ldz, target, eps, row_loss,
                                                     (X*)dz, ld_dz));
  LAUNCH_CHECK();
  count_launch();
}

// ------------------------------------------------------------------ NSP head
// Every CTA recomputes the B x 2 logit gradients (tiny) into smem; CTA 0
// alone writes the row losses and the dH rows; dW's 2d entries are spread
// over the grid, each a fixed-order sum over the batch (deterministic).
template <class HT>
__global__ void __launch_bounds__(1024) nsp_fwd_bwd_kernel(
    int B, int d, const int* __restrict__ cu, const int* __restrict__ label,
    const HT* __restrict__ H, const float* __restrict__ W, const float* __restrict__ bias,
    float* __restrict__ row_loss, float* __restrict__ dW, float* __restrict__ db,
    HT* __restrict__ dH, int grad) {
  extern __shared__ float dzs[];  // [B][2]
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const bool lead = blockIdx.x == 0;
  for (int b = w; b < B; b += nw) {
    const HT* h0 = H + (int64_t)cu[b] * d;
    float z0 = 0.f, z1 = 0.f;
#pragma unroll 8
    for (int c = lane; c < d; c += 32) {
      const float hv = tof(h0[c]);
      z0 += hv * W[c * 2 + 0];
      z1 += hv * W[c * 2 + 1];
    }
    z0 = warp_sum(z0) + bias[0];
    z1 = warp_sum(z1) + bias[1];
    const float mx = fmaxf(z0, z1);
    const float e0 = expf(z0 - mx), e1 = expf(z1 - mx);
    const float se = e0 + e1;
    const int t = label[b];
    const float g0 = e0 / se - (t == 0 ? 1.f : 0.f);
    const float g1 = e1 / se - (t == 1 ? 1.f : 0.f);
    if (lane == 0) {
      if (lead) row_loss[b] = mx + logf(se) - (t == 0 ? z0 : z1);
      dzs[2 * b + 0] = g0;
      dzs[2 * b + 1] = g1;
    }
    if (grad && lead) {
      HT* dh = dH + (int64_t)cu[b] * d;
#pragma unroll 8
      for (int c = lane; c < d; c += 32)
        dh[c] = fromf<HT>(tof(dh[c]) + g0 * W[c * 2 + 0] + g1 * W[c * 2 + 1]);
    }
  }
  if (!grad) return;
  __syncthreads();
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < 2 * d; e += gridDim.x * blockDim.x) {
    const int c = e >> 1, k = e & 1;
    float acc = 0.f;
#pragma unroll 8
    for (int b = 0; b < B; ++b) acc += tof(H[(int64_t)cu[b] * d + c]) * dzs[2 * b + k];
    dW[e] = acc;
  }
  if (lead && threadIdx.x < 2) {
    float acc = 0.f;
    for (int b = 0; b < B; ++b) acc += dzs[2 * b + threadIdx.x];
    db[threadIdx.x] = acc;
  }
}

void nsp_head(const DevBatch& b, int d, const void* H, DType ht, const float* W,
              const float* bias, float* row_loss, float* dW, float* db, void* dH,
              int compute_grad, cudaStream_t s) {
  if (b.B == 0) return;
  const size_t sm = sizeof(float) * 2 * b.B;
  // one warp per row (B <= 32 per CTA pass); dW's 2d sums over 2 CTAs
  const int grid = compute_grad ? 2 : 1;
  DISPATCH1(ht, X, nsp_fwd_bwd_kernel<X><<<grid, 1024, sm, s>>>(b.B, d, b.cu, b.label, (const X*)H, W,
                                                              bias, row_loss, dW, db, (X*)dH,
                                                              compute_grad));
  LAUNCH_CHECK();
  count_launch();
}

// ------------------------------------------------------------------ scalars
__global__ void loss_reduce_kernel(const float* __restrict__ a, int na, const float* __restrict__ b,
                                   int nb, double* __restrict__ out) {
  __shared__ double red[256];
  double acc = 0.0;
  for (int i = threadIdx.x; i < na; i += blockDim.x) acc += (double)a[i];
  for (int i = threadIdx.x; i < nb; i += blockDim.x) acc += (double)b[i];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = red[0];
}
void loss_reduce(const float* a, int na, const float* b, int nb, double* out,
                 cudaStream_t s) {
  loss_reduce_kernel<<<1, 256, 0, s>>>(a, na, b, nb, out);
  LAUNCH_CHECK();
  count_launch();
}

__device__ __forceinline__ unsigned long long round_seq(const float* hyper) {
  return hyper ? (unsigned long long)__float_as_uint(hyper[3]) : 0ull;
}
__global__ void finalize_weight_kernel(const double* lw, float* inv_w, double* inv_w64,
                                       unsigned long long* err, const float* hyper) {
  const double l = lw[0], w = lw[1];
  unsigned long long f = 0;
  if (!isfinite(l)) f |= 1;
  if (!(w > 0.0)) f |= 2;
  if (f && err[0] == 0) err[1] = round_seq(hyper);  // the first failing round
  err[0] |= f;
  *inv_w64 = w > 0.0 ? 1.0 / w : 0.0;
  *inv_w = (float)(*inv_w64);
}
void finalize_weight(const double* lw, float* inv_w, double* inv_w64, unsigned long long* err,
                     const float* hyper, cudaStream_t s) {
  finalize_weight_kernel<<<1, 1, 0, s>>>(lw, inv_w, inv_w64, err, hyper);
  LAUNCH_CHECK();
  count_launch();
}

__global__ void fill_add_kernel_scalar(float* __restrict__ acc, const float* __restrict__ g, uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) acc[i] += g[i];
}
// K > 1 (Accumulator, optim.hpp:154-202): the round's [loss, weight] joins the
// running totals; on the K-th round the totals become the report (lw[4..5])
// and 1/total weight the update's scale, and the totals restart.
__global__ void accumulate_weight_kernel(const double* lw, double* acc, double* out,
                                         double* inv_w64, int final_round) {
  acc[0] += lw[0];
  acc[1] += lw[1];
  if (final_round) {
    out[0] = acc[0];
    out[1] = acc[1];
    *inv_w64 = acc[1] > 0.0 ? 1.0 / acc[1] : 0.0;
    acc[0] = 0.0;
    acc[1] = 0.0;
  }
}
void accumulate_weight(const double* lw, double* acc, double* out, double* inv_w64, int final_round,
                       cudaStream_t s) {
  accumulate_weight_kernel<<<1, 1, 0, s>>>(lw, acc, out, inv_w64, final_round);
  LAUNCH_CHECK();
  count_launch();
}
// acc[lo, lo+n) += g[lo, lo+n) (a reduced gradient bucket of a non-final round)
__global__ void accumulate_grad_kernel(float* __restrict__ acc, const float* __restrict__ g, uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * 4;
  for (uint64_t i = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; i < n; i += stride) {
    if (i + 4 <= n) {
      float4 a = *reinterpret_cast<const float4*>(acc + i);
      const float4 b = *reinterpret_cast<const float4*>(g + i);
      a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
      *reinterpret_cast<float4*>(acc + i) = a;
    } else {
      for (uint64_t j = i; j < n; ++j) acc[j] += g[j];
    }
  }
}
void accumulate_grad(float* acc, const float* g, uint64_t n, cudaStream_t s) {
  if (n == 0) return;
  // float4 path needs 16-byte alignment of both ranges
  if (((reinterpret_cast<uintptr_t>(acc) | reinterpret_cast<uintptr_t>(g)) & 15) == 0) {
    accumulate_grad_kernel<<<148 * 8, 256, 0, s>>>(acc, g, n);
  } else {
    fill_add_kernel_scalar<<<148 * 8, 256, 0, s>>>(acc, g, n);
  }
  LAUNCH_CHECK();
  count_launch();
}

// ------------------------------------------------------------------ Adam
__device__ __forceinline__ uint64_t shadow_index(const uint64_t* seg, int nseg, uint64_t i) {
  int lo = 0, hi = nseg - 1;
  while (lo < hi) {  // last segment with offset <= i
    const int mid = (lo + hi + 1) >> 1;
    if (seg[4 * mid] <= i) lo = mid; else hi = mid - 1;
  }
  const uint64_t off = seg[4 * lo], cols = seg[4 * lo + 1], soff = seg[4 * lo + 2],
                 pcols = seg[4 * lo + 3];
  const uint64_t local = i - off;
  return cols == pcols ? soff + local : soff + (local / cols) * pcols + local % cols;
}

#ifdef HP_ADAM_STREAMING
__device__ __forceinline__ float4 adam_ld4(const float* p) { return __ldcs(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ void adam_st4(float* p, float4 v) { __stcs(reinterpret_cast<float4*>(p), v); }
#else
__device__ __forceinline__ float4 adam_ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void adam_st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
#endif

__device__ __forceinline__ void adam_one(const AdamArgs& a, float& p, float& m, float& v, float g) {
  if (a.sgd) {
    p = __fsub_rn(p, __fmul_rn(a.lr, g));
    return;
  }
  // AdamW (extension): decoupled decay p -= (lr wd) p before the Adam step
  if (a.wd != 0.f) p = __fsub_rn(p, __fmul_rn(__fmul_rn(a.lr, a.wd), p));
  // explicit round-to-nearest ops: no FMA contraction, matching the
  // reference's -ffp-contract=off scalar loop bit for bit
  m = __fadd_rn(__fmul_rn(a.b1, m), __fmul_rn(__fsub_rn(1.f, a.b1), g));
  v = __fadd_rn(__fmul_rn(a.b2, v), __fmul_rn(__fsub_rn(1.f, a.b2), __fmul_rn(g, g)));
  const float mh = __fmul_rn(m, a.c1);
  const float vh = __fmul_rn(v, a.c2);
  p = __fsub_rn(p, __fmul_rn(a.lr, __fdiv_rn(mh, __fadd_rn(__fsqrt_rn(vh), a.eps))));
}

// One CTA per work item.  float4 I/O when the item is 16-byte aligned.
// Memory-bound: 6 CTAs (48 warps) per SM keep enough loads in flight, so the
// register budget is pinned (<= 42).
// the update is skipped when this round's loss / weight check failed, or an
// earlier unsynced round's did (pipelined rounds stop at the first error)
__device__ __forceinline__ bool skip_update(const AdamArgs& a) {
  if (!a.err) return false;
  return a.err[0] != 0 || a.err[3] < round_seq(a.hyper);
}
// a non-finite f64 gradient element (optim.hpp:131-133): skipped, recorded
__device__ __forceinline__ void note_bad(const AdamArgs& a, uint64_t idx, unsigned long long& bad) {
  bad = min(bad, (unsigned long long)idx);
}
__device__ __forceinline__ void flush_bad(const AdamArgs& a, unsigned long long bad) {
  if (bad != ~0ull && a.err) {
    atomicMin(&a.err[2], bad);
    atomicMin(&a.err[3], round_seq(a.hyper));
  }
}

template <bool ACC>  // ACC: add (then zero) the K > 1 accumulator a.g2
__global__ void __launch_bounds__(256, 6) adam_kernel(const AdamArgs a0) {
  if (skip_update(a0)) return;  // numeric error: leave parameters untouched
  AdamArgs a = a0;
  if (a.hyper) {  // per-step scalars from device memory (graph replays)
    a.lr = a.hyper[0];
    a.c1 = a.hyper[1];
    a.c2 = a.hyper[2];
  }
  const bool scale = a.inv_w64 != nullptr;
  const double sc = scale ? *a.inv_w64 : 1.0;
  bf16* sh = (bf16*)a.shadow;
  unsigned long long bad = ~0ull;
  // grid-stride over the work items
  for (int item = blockIdx.x; item < a.nitems; item += gridDim.x) {
    const uint64_t* it = a.items + 5 * (uint64_t)item;
    const uint64_t lo = it[0], n = it[1], slo = it[2], cols = it[3], pcols = it[4];
    const bool contig = cols == pcols;
    auto sidx = [&](uint64_t local) {
      return contig ? slo + local : slo + (local / cols) * pcols + local % cols;
    };
    if ((lo & 3) == 0 && (!sh || !contig || (slo & 3) == 0)) {
      const uint64_t n4 = n & ~uint64_t(3);
      for (uint64_t i = 4 * threadIdx.x; i < n4; i += 4 * blockDim.x) {
        // (streaming / evict-first hints for these once-per-step streams,
        // -DHP_ADAM_STREAMING, measured 7449 vs 7564 samples/s: plain wins)
        float4 p = adam_ld4(a.p + lo + i);
        float4 m = adam_ld4(a.m + lo + i);
        float4 v = adam_ld4(a.v + lo + i);
        float4 g = adam_ld4(a.g + lo + i);
        float* pp = &p.x; float* mm = &m.x; float* vv = &v.x; const float* gg = &g.x;
        // g /= total weight in f64, then cast to T (engine.hpp:151, optim.hpp:135)
        float gs[4];
        bool ok[4];
        if constexpr (ACC) {  // K > 1: earlier rounds' sums, consumed (zeroed) here
          const float4 q = *reinterpret_cast<const float4*>(a.g2 + lo + i);
          *reinterpret_cast<float4*>(a.g2 + lo + i) = make_float4(0.f, 0.f, 0.f, 0.f);
          const float* qq = &q.x;
  #pragma unroll
          for (int e = 0; e < 4; ++e) {
            const double gd = scale ? ((double)gg[e] + (double)qq[e]) * sc : (double)gg[e] + (double)qq[e];
            gs[e] = (float)gd;
            ok[e] = isfinite(gd);
            if (!ok[e]) note_bad(a, lo + i + e, bad);
          }
        } else {
  #pragma unroll
          for (int e = 0; e < 4; ++e) {
            const double gd = scale ? (double)gg[e] * sc : (double)gg[e];
            gs[e] = (float)gd;
            ok[e] = isfinite(gd);
            if (!ok[e]) note_bad(a, lo + i + e, bad);
          }
        }
  #pragma unroll
        for (int e = 0; e < 4; ++e)
          if (ok[e]) adam_one(a, pp[e], mm[e], vv[e], gs[e]);
        adam_st4(a.p + lo + i, p);
        adam_st4(a.m + lo + i, m);
        adam_st4(a.v + lo + i, v);
        if (sh) {
          if (contig) {
            __nv_bfloat162 h0 = __floats2bfloat162_rn(p.x, p.y), h1 = __floats2bfloat162_rn(p.z, p.w);
            uint2 u;
            u.x = *reinterpret_cast<uint32_t*>(&h0);
            u.y = *reinterpret_cast<uint32_t*>(&h1);
            *reinterpret_cast<uint2*>(sh + slo + i) = u;
          } else {
  #pragma unroll
            for (int e = 0; e < 4; ++e) sh[sidx(i + e)] = __float2bfloat16_rn(pp[e]);
          }
        }
      }
      for (uint64_t i = n4 + threadIdx.x; i < n; i += blockDim.x) {
        double gd;
        if constexpr (ACC) {
          gd = (double)a.g[lo + i] + (double)a.g2[lo + i];
          a.g2[lo + i] = 0.f;
        } else {
          gd = (double)a.g[lo + i];
        }
        if (scale) gd *= sc;
        if (!isfinite(gd)) { note_bad(a, lo + i, bad); continue; }
        const float ge = (float)gd;
        float p = a.p[lo + i], m = a.m[lo + i], v = a.v[lo + i];
        adam_one(a, p, m, v, ge);
        a.p[lo + i] = p; a.m[lo + i] = m; a.v[lo + i] = v;
        if (sh) sh[sidx(i)] = __float2bfloat16_rn(p);
      }
    } else {
      for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) {
        double gd;
        if constexpr (ACC) {
          gd = (double)a.g[lo + i] + (double)a.g2[lo + i];
          a.g2[lo + i] = 0.f;
        } else {
          gd = (double)a.g[lo + i];
        }
        if (scale) gd *= sc;
        if (!isfinite(gd)) { note_bad(a, lo + i, bad); continue; }
        const float ge = (float)gd;
        float p = a.p[lo + i], m = a.m[lo + i], v = a.v[lo + i];
        adam_one(a, p, m, v, ge);
        a.p[lo + i] = p; a.m[lo + i] = m; a.v[lo + i] = v;
        if (sh) sh[sidx(i)] = __float2bfloat16_rn(p);
      }
    }
  }
  flush_bad(a, bad);
}
void adam_update(const AdamArgs& a, cudaStream_t s) {
  if (a.nitems == 0) return;
  const int grid = a.nitems;
  if (a.g2)
    adam_kernel<true><<<grid, 256, 0, s>>>(a);
  else
    adam_kernel<false><<<grid, 256, 0, s>>>(a);
  LAUNCH_CHECK();
  count_launch();
}

// Word-embedding rows of a K = 1 update, split around the round's distinct
// token ids: nl sorted id lists (one per rank, list l = uids[l * stride ..],
// length ucnts[2 l] + ucnts[2 l + 1]); only rows in their union receive a
// gradient (embed_bwd, then the exchange), every other row's is exactly 0.
// mode 0 updates the rows in NO list with g = 0 -- no gradient read, so it
// runs while backward is still producing dE; mode 1 updates the union's rows
// (each once: a row is skipped in list l when an earlier list holds it) once
// dE is final. Per element the arithmetic is adam_kernel's (g * (1 / Σw) in
// f64, then adam_one), so the split update is bit-identical to the dense one.
// One warp per row, float4 I/O (d % 4 == 0, lo % 4 == 0).
__device__ __forceinline__ bool in_sorted(const int* __restrict__ u, int n, int r) {
  int l = 0, h = n;
  while (l < h) {
    const int mid = (l + h) >> 1;
    if (u[mid] < r) l = mid + 1; else h = mid;
  }
  return l < n && u[l] == r;
}
__global__ void __launch_bounds__(256) adam_rows_kernel(const AdamArgs a0, int mode,
                                                        const int* __restrict__ uids,
                                                        const int* __restrict__ ucnts, int nl,
                                                        int stride, int V, int d, uint64_t lo,
                                                        uint64_t slo, uint64_t pcols) {
  if (skip_update(a0)) return;
  AdamArgs a = a0;
  if (a.hyper) {
    a.lr = a.hyper[0];
    a.c1 = a.hyper[1];
    a.c2 = a.hyper[2];
  }
  const bool scale = a.inv_w64 != nullptr;
  const double sc = scale ? *a.inv_w64 : 1.0;
  const float g0 = scale ? (float)(0.0 * sc) : 0.f;  // what adam_kernel makes of a zero
  bf16* sh = (bf16*)a.shadow;
  int total = 0;
  for (int l = 0; l < nl; ++l) total += ucnts[2 * l] + ucnts[2 * l + 1];
  const int nrows = mode ? total : V;
  const int lane = threadIdx.x & 31;
  unsigned long long bad = ~0ull;
  for (int i = blockIdx.x * 8 + (threadIdx.x >> 5); i < nrows; i += gridDim.x * 8) {
    int r = i;
    bool skip = false;
    if (mode) {  // i-th entry of the concatenated lists; first list holding it wins
      int l = 0, j = i;
      while (j >= ucnts[2 * l] + ucnts[2 * l + 1]) { j -= ucnts[2 * l] + ucnts[2 * l + 1]; ++l; }
      r = uids[(int64_t)l * stride + j];
      for (int k = 0; k < l && !skip; ++k)
        skip = in_sorted(uids + (int64_t)k * stride, ucnts[2 * k] + ucnts[2 * k + 1], r);
    } else {  // warp-uniform binary searches
      for (int k = 0; k < nl && !skip; ++k)
        skip = in_sorted(uids + (int64_t)k * stride, ucnts[2 * k] + ucnts[2 * k + 1], r);
    }
    if (skip) continue;
    const uint64_t base = lo + (uint64_t)r * d;
    for (int c = 4 * lane; c < d; c += 128) {
      float4 p = adam_ld4(a.p + base + c);
      float4 m = adam_ld4(a.m + base + c);
      float4 v = adam_ld4(a.v + base + c);
      float gs[4] = {g0, g0, g0, g0};
      bool ok[4] = {true, true, true, true};
      if (mode) {
        const float4 g = adam_ld4(a.g + base + c);
        const float* gg = &g.x;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const double gd = scale ? (double)gg[e] * sc : (double)gg[e];
          gs[e] = (float)gd;
          ok[e] = isfinite(gd);
          if (!ok[e]) note_bad(a, base + c + e, bad);
        }
      }
      float* pp = &p.x; float* mm = &m.x; float* vv = &v.x;
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (ok[e]) adam_one(a, pp[e], mm[e], vv[e], gs[e]);
      adam_st4(a.p + base + c, p);
      adam_st4(a.m + base + c, m);
      adam_st4(a.v + base + c, v);
      if (sh) {
        const uint64_t so = slo + (uint64_t)r * pcols + c;
#pragma unroll
        for (int e = 0; e < 4; ++e) sh[so + e] = __float2bfloat16_rn(pp[e]);
      }
    }
  }
  flush_bad(a, bad);
}
void adam_rows(const AdamArgs& a, int mode, const int* uids, const int* ucnts, int nl, int stride,
               int V, int d, uint64_t lo, uint64_t slo, uint64_t pcols, cudaStream_t s) {
  adam_rows_kernel<<<148 * 6, 256, 0, s>>>(a, mode, uids, ucnts, nl, stride, V, d, lo, slo, pcols);
  LAUNCH_CHECK();
  count_launch();
}

__global__ void shadow_kernel(const float* p, bf16* sh, const uint64_t* seg, int nseg, uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    sh[shadow_index(seg, nseg, i)] = __float2bfloat16_rn(p[i]);
}
void refresh_shadow(const float* p, void* shadow, const uint64_t* seg_table,
                    int nseg, uint64_t n, cudaStream_t s) {
  if (n == 0) return;
  shadow_kernel<<<148 * 8, 256, 0, s>>>(p, (bf16*)shadow, seg_table, nseg, n);
  LAUNCH_CHECK();
  count_launch();
}

__global__ void fill_kernel(float* p, uint64_t n, float v) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) p[i] = v;
}
void fill_f32(float* p, uint64_t n, float v, cudaStream_t s) {
  if (n == 0) return;
  fill_kernel<<<148 * 4, 256, 0, s>>>(p, n, v);
  LAUNCH_CHECK();
  count_launch();
}

__global__ void fnv_kernel(const uint8_t* p, uint64_t n, uint64_t* out) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (uint64_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ull;
  }
  *out = h;
}
// FNV-1a of each `chunk`-byte block (one thread per block, bytes in order)
__global__ void fnv_chunks_kernel(const uint8_t* __restrict__ p, uint64_t n, uint64_t chunk,
                                  uint64_t nchunks, uint64_t* __restrict__ out) {
  const uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nchunks) return;
  const uint8_t* q = p + c * chunk;
  const uint64_t m = min(chunk, n - c * chunk);
  uint64_t h = 0xcbf29ce484222325ull;
  uint64_t i = 0;
  for (; i + 16 <= m; i += 16) {
    const uint4 v = *reinterpret_cast<const uint4*>(q + i);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        h ^= (w[k] >> (8 * b)) & 0xffu;
        h *= 0x100000001b3ull;
      }
  }
  for (; i < m; ++i) {
    h ^= q[i];
    h *= 0x100000001b3ull;
  }
  out[c] = h;
}
__global__ void digest_mismatch_kernel(const uint64_t* d, double* bad) {
  *bad = d[0] == d[1] ? 0.0 : 1.0;
}
void fnv1a_chunked(const void* p, uint64_t n, uint64_t* scratch, uint64_t* out, cudaStream_t s) {
  constexpr uint64_t kChunk = 65536;
  const uint64_t nchunks = (n + kChunk - 1) / kChunk;
  fnv_chunks_kernel<<<(unsigned)((nchunks + 127) / 128), 128, 0, s>>>(
      static_cast<const uint8_t*>(p), n, kChunk, nchunks, scratch);
  LAUNCH_CHECK();
  count_launch();
  fnv1a(reinterpret_cast<const uint8_t*>(scratch), nchunks * 8, out, s);
}
size_t fnv1a_chunked_scratch(uint64_t n) { return (n + 65535) / 65536; }
void digest_mismatch(const uint64_t* d, double* bad, cudaStream_t s) {
  digest_mismatch_kernel<<<1, 1, 0, s>>>(d, bad);
  LAUNCH_CHECK();
  count_launch();
}

void fnv1a(const uint8_t* p, uint64_t n, uint64_t* out, cudaStream_t s) {
  fnv_kernel<<<1, 1, 0, s>>>(p, n, out);
  LAUNCH_CHECK();
  count_launch();
}

// ------------------------------------------------------------------ SIMT GEMM
template <class T>
__device__ __forceinline__ float ld_op(const Operand& o, int64_t off) {
  return tof(static_cast<const T*>(o.p)[off]);
}
__device__ __forceinline__ int64_t a_off(const Operand& o, int64_t m, int64_t k) {
  return o.trans ? k * o.ld + m : m * o.ld + k;
}
__device__ __forceinline__ int64_t b_off(const Operand& o, int64_t k, int64_t n) {
  if (!o.trans) {
    return o.group ? (n / o.group) * o.gstride + k * o.ld + n % o.group : k * o.ld + n;
  }
  return o.group ? (k / o.group) * o.gstride + n * o.ld + k % o.group : n * o.ld + k;
}

__device__ __forceinline__ float gelu_f(float x) {
  return 0.5f * x * (1.f + erff(x * 0.70710678118654752f));
}
__device__ __forceinline__ float dgelu_f(float x) {
  return 0.5f * (1.f + erff(x * 0.70710678118654752f)) +
         x * 0.39894228040143268f * expf(-0.5f * x * x);
}

template <class CT>
__device__ __forceinline__ void epi_store(const GemmArgs& g, int m, int n, float acc) {
  float v = acc * g.alpha;
  if (g.bias) v += g.bias[n];
  const int64_t co = g.c_group ? (n / g.c_group) * g.c_gstride + (int64_t)m * g.ldc + n % g.c_group
                               : (int64_t)m * g.ldc + n;
  if (g.act == ACT_GELU) {
    static_cast<CT*>(g.aux)[co] = fromf<CT>(v);
    v = gelu_f(v);
  } else if (g.act == ACT_DGELU) {
    v *= dgelu_f(tof(static_cast<const CT*>(g.aux)[co]));
  }
  if (g.resid) v += tof(static_cast<const CT*>(g.resid)[(int64_t)m * g.ld_resid + n]);
  CT* c = static_cast<CT*>(g.c);
  if (g.accumulate) v += tof(c[co]);
  c[co] = fromf<CT>(v);
}

template <class ABT, class CT>
__global__ void __launch_bounds__(256) gemm_simt_kernel(GemmArgs g) {
  constexpr int BM = 64, BN = 64, BK = 16;
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < g.K; k0 += BK) {
    for (int e = threadIdx.x; e < BM * BK; e += 256) {
      // trans A: m fastest for coalescing, else k fastest
      int mm, kk;
      if (g.a.trans) { mm = e % BM; kk = e / BM; } else { kk = e % BK; mm = e / BK; }
      const int m = m0 + mm, k = k0 + kk;
      As[kk][mm] = (m < g.M && k < g.K) ? ld_op<ABT>(g.a, a_off(g.a, m, k)) : 0.f;
    }
    for (int e = threadIdx.x; e < BK * BN; e += 256) {
      int kk, nn;
      if (g.b.trans) { kk = e % BK; nn = e / BK; } else { nn = e % BN; kk = e / BN; }
      const int k = k0 + kk, n = n0 + nn;
      Bs[kk][nn] = (n < g.N && k < g.K) ? ld_op<ABT>(g.b, b_off(g.b, k, n)) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] += a[i] * b[j];
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int m = m0 + ty * 4 + i, n = n0 + tx * 4 + j;
      if (m < g.M && n < g.N) epi_store<CT>(g, m, n, acc[i][j]);
    }
}

void gemm_simt(const GemmArgs& g, cudaStream_t s) {
  if (g.M == 0 || g.N == 0) return;
  dim3 grid((g.N + 63) / 64, (g.M + 63) / 64);
  DISPATCH1(g.ab, AB, DISPATCH1(g.ct, C, gemm_simt_kernel<AB, C><<<grid, 256, 0, s>>>(g)));
  LAUNCH_CHECK();
  count_launch();
}

// ---- fp32-accurate GEMMs on the bf16 tensor cores ("bf16x6") -------------
// Every fp32 operand element splits exactly into three bf16 terms,
// x = x0 + x1 + x2 (x0 = bf16(x), x1 = bf16(x - x0), x2 = bf16(x - x0 - x1),
// 24 significant bits), and
//   a b ~= a0 b0 + a0 b1 + a1 b0 + a0 b2 + a2 b0 + a1 b1
// (the dropped terms a1 b2, a2 b1, a2 b2 are O(2^-24) of |a||b|, below fp32
// rounding) -- i.e. ONE bf16 GEMM with fp32 accumulation over K' = 6K of
//   A' = [a0 | a0 | a1 | a0 | a2 | a1],  B' = [b0 ; b1 ; b0 ; b2 ; b0 ; b1]
// on the same tcgen05 kernel (and epilogues) as the bf16 path.  The split
// kernel writes A' / B' dense in the operand's own major-ness (grouped per-head
// operands are ungrouped on the way); six bf16 UMMAs per product cost what
// three TF32 ones would (TF32 runs at half the bf16 rate).
__constant__ int kX6PatA[6] = {0, 0, 1, 0, 2, 1};
__constant__ int kX6PatB[6] = {0, 1, 0, 2, 0, 1};

// logical A (m, k) / B (k, n): r = m or n, K the contracted extent
__device__ __forceinline__ void split3(float v, bf16* p) {
  p[0] = __float2bfloat16_rn(v);
  const float r1 = v - __bfloat162float(p[0]);
  p[1] = __float2bfloat16_rn(r1);
  p[2] = __float2bfloat16_rn(r1 - __bfloat162float(p[1]));
}
__global__ void split6_kernel(Operand src, int is_b, int R, int K, bf16* __restrict__ dst, int64_t ldd) {
  const float* x = static_cast<const float*>(src.p);
  // walk the source's contiguous dimension fastest; the destination's
  // contiguous dimension is the same one, so two neighbours along it leave as
  // one bf16x2 per term
  const bool kfast = is_b ? src.trans != 0 : src.trans == 0;
  const int F = kfast ? K : R;  // fast dimension
  auto dst_off = [&](int64_t r, int64_t kk) -> int64_t {
    // A: trans -> [K'][M] else [M][K'];  B: trans -> [N][K'] else [K'][N]
    return is_b ? (src.trans ? r * ldd + kk : kk * ldd + r) : (src.trans ? kk * ldd + r : r * ldd + kk);
  };
  auto src_val = [&](int64_t r, int64_t k) { return x[is_b ? b_off(src, k, r) : a_off(src, r, k)]; };
  const int* pat = is_b ? kX6PatB : kX6PatA;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (F % 2 == 0) {
    const int64_t total2 = (int64_t)R * K / 2;
    for (int64_t e2 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e2 < total2; e2 += stride) {
      const int64_t e = 2 * e2;
      const int64_t slow = e / F, fast = e - slow * F;
      const int64_t r = kfast ? slow : fast, k = kfast ? fast : slow;
      const int64_t r1 = kfast ? r : r + 1, k1 = kfast ? k + 1 : k;
      bf16 p0[3], p1[3];
      split3(src_val(r, k), p0);
      split3(src_val(r1, k1), p1);
#pragma unroll
      for (int j = 0; j < 6; ++j) {
        __nv_bfloat162 h;
        h.x = p0[pat[j]];
        h.y = p1[pat[j]];
        *reinterpret_cast<__nv_bfloat162*>(dst + dst_off(r, (int64_t)j * K + k)) = h;
      }
    }
    return;
  }
  const int64_t total = (int64_t)R * K;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
    const int64_t r = kfast ? e / K : e % R, k = kfast ? e % K : e / R;
    bf16 part[3];
    split3(src_val(r, k), part);
#pragma unroll
    for (int j = 0; j < 6; ++j) dst[dst_off(r, (int64_t)j * K + k)] = part[pat[j]];
  }
}

namespace {
int g_tc_mode = 0;
// per-stream split buffers, grown on demand; superseded buffers stay alive
// (CUDA graphs captured with them keep their addresses)
struct X6Buf {
  void* p = nullptr;
  size_t cap = 0;
};
std::mutex g_x6_mu;
std::map<std::pair<cudaStream_t, int>, X6Buf> g_x6;
std::vector<void*> g_x6_old;
void* x6_buffer(cudaStream_t s, int which, size_t bytes) {
  std::lock_guard<std::mutex> l(g_x6_mu);
  X6Buf& b = g_x6[{s, which}];
  if (b.cap < bytes) {
    if (b.p) g_x6_old.push_back(b.p);
    const size_t cap = std::max(bytes, b.cap * 3 / 2);
    HP_CUDA(cudaMalloc(&b.p, cap));
    b.cap = cap;
  }
  return b.p;
}
int64_t pad8i(int64_t v) { return (v + 7) & ~int64_t(7); }
bool x6_rs_on() {  // HP_X6_RS=0: always partials + reduction (A/B)
  static const bool on = [] {
    const char* e = std::getenv("HP_X6_RS");
    return !(e && std::string(e) == "0");
  }();
  return on;
}
bool f32_x6() {
  static const bool on = [] {
    const char* e = std::getenv("HP_F32_GEMM");  // "simt": the fp32 SIMT kernel (A/B, parity checks)
    return !(e && std::string(e) == "simt");
  }();
  return on;
}
}  // namespace
void gemm_tc_force(int mode) { g_tc_mode = mode; }

// sum of the K-chunk partials (fixed order, fp32 round-to-nearest), then the
// GEMM's own epilogue (alpha, bias, GELU / dGELU, residual, accumulate,
// grouped C) -- the SIMT kernel's epi_store
template <class CT>
__global__ void x6_reduce_kernel(const float* __restrict__ part, int chunks, GemmArgs g) {
  const int64_t MN = (int64_t)g.M * g.N;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (g.N % 4 == 0) {  // four neighbours of one row per thread, float4 partial reads
    const int64_t MN4 = MN / 4;
    const float4* p4 = reinterpret_cast<const float4*>(part);
    for (int64_t e4 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e4 < MN4; e4 += stride) {
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      int c = 0;
      for (; c + 4 <= chunks; c += 4) {  // four loads in flight, added in chunk order
        float4 q[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) q[u] = __ldcs(p4 + (c + u) * MN4 + e4);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          acc.x += q[u].x; acc.y += q[u].y; acc.z += q[u].z; acc.w += q[u].w;
        }
      }
      for (; c < chunks; ++c) {
        const float4 q = __ldcs(p4 + c * MN4 + e4);
        acc.x += q.x; acc.y += q.y; acc.z += q.z; acc.w += q.w;
      }
      const int64_t e = 4 * e4;
      const int m = static_cast<int>(e / g.N), n = static_cast<int>(e - (int64_t)m * g.N);
      epi_store<CT>(g, m, n, acc.x);
      epi_store<CT>(g, m, n + 1, acc.y);
      epi_store<CT>(g, m, n + 2, acc.z);
      epi_store<CT>(g, m, n + 3, acc.w);
    }
    return;
  }
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < MN; e += stride) {
    float acc = 0.f;
    for (int c = 0; c < chunks; ++c) acc += part[c * MN + e];
    epi_store<CT>(g, static_cast<int>(e / g.N), static_cast<int>(e % g.N), acc);
  }
}

bool gemm_x6(const GemmArgs& g, cudaStream_t s) {
  if (g.M == 0 || g.N == 0) return true;
  const int64_t K6 = 6LL * g.K;
  const int64_t lda = g.a.trans ? pad8i(g.M) : pad8i(K6);
  const int64_t ldb = g.b.trans ? pad8i(K6) : pad8i(g.N);
  const size_t abytes = (size_t)(g.a.trans ? K6 * lda : (int64_t)g.M * lda) * 2;
  const size_t bbytes = (size_t)(g.b.trans ? (int64_t)g.N * ldb : K6 * ldb) * 2;
  bf16* A = static_cast<bf16*>(x6_buffer(s, 0, abytes));
  bf16* B = static_cast<bf16*>(x6_buffer(s, 1, bbytes));
  // The tensor core's fp32 accumulation is not round-to-nearest across the
  // MMA chain (its error grows with the chain, not with its square root), so
  // K' is cut into chunks of <= 1024 (at most 48 chunks; whole split terms,
  // K' = 6K: 6 chunks of K, when K <= 1024), each accumulated into its own
  // fp32 partial -- all chunks in ONE launch (split-K units that store their
  // partials side by side) -- and the partials are summed in a fixed order
  // with RN: deterministic, no atomics.
  int64_t kc = 1024;
  if ((K6 + kc - 1) / kc > 48) kc = ((K6 + 47) / 48 + 63) / 64 * 64;
  if (g.K <= 1024 && g.K % 64 == 0) kc = g.K;
  const int chunks = static_cast<int>((K6 + kc - 1) / kc);
  GemmArgs h;
  h.M = g.M;
  h.N = g.N;
  h.ab = DType::bf16;
  h.ct = DType::f32;
  Operand a{A, lda, g.a.trans, 0, 0}, b{B, ldb, g.b.trans, 0, 0};
  h.a = a;
  h.b = b;
  h.K = static_cast<int>(K6);
  if (!gemm_tc_supported(h)) return false;
  const int grid = 148 * 8;
  split6_kernel<<<grid, 256, 0, s>>>(g.a, 0, g.M, g.K, A, lda);
  LAUNCH_CHECK();
  split6_kernel<<<grid, 256, 0, s>>>(g.b, 1, g.N, g.K, B, ldb);
  LAUNCH_CHECK();
  count_launch(2);
  const int64_t MN = (int64_t)g.M * g.N;
  // Enough 128-wide tiles to fill the GPU: the chunks are summed on chip
  // (running-sum stints, same order) and the GEMM applies the epilogue --
  // no partials in HBM, no reduction launch.  Otherwise each chunk is a
  // split-K unit of its own (more parallelism) and x6_reduce_kernel sums them.
  const int64_t tiles128 = ((g.M + 127) / 128) * ((g.N + 127) / 128);
  if (chunks > 1 && g.ct == DType::f32 && tiles128 >= 148 && x6_rs_on()) {
    GemmArgs r = g;
    r.ab = DType::bf16;
    r.a = a;
    r.b = b;
    r.K = static_cast<int>(K6);
    r.rs_kc = static_cast<int>(kc);
    r.max_splits = 1;
    if (gemm_tc_supported(r)) {
      gemm_tc(r, s);
      return true;
    }
  }
  float* part = static_cast<float*>(x6_buffer(s, 2, (size_t)chunks * MN * 4));
  h.c = part;
  h.ldc = g.N;
  if (chunks > 1) {
    h.part_chunks = chunks;
    h.part_kc = static_cast<int>(kc);
    h.part_stride = MN;
  } else {
    h.max_splits = 1;  // one chunk: one accumulation chain, no reduction
  }
  gemm_tc(h, s);
  DISPATCH1(g.ct, CT, x6_reduce_kernel<CT><<<148 * 8, 256, 0, s>>>(part, chunks, g));
  LAUNCH_CHECK();
  count_launch();
  return true;
}

int gemm(const GemmArgs& g, cudaStream_t s) {
  if (g_tc_mode == 0 && g.ab == DType::bf16 && gemm_tc_supported(g)) {
    gemm_tc(g, s);
    return 1;
  }
  if (g_tc_mode == 0 && g.ab == DType::f32 && f32_x6() && gemm_x6(g, s)) return 2;
  gemm_simt(g, s);
  return 0;
}

}  // namespace hp
