// The reference's operator table (hetpar::kern, include/hetpar/kernels.hpp:44-68,
// src/kernels_scalar.cpp) on device pointers: the same results, bit for bit.
//
// Elementwise kernels are grid-stride loops with explicitly rounded
// operations (no FMA contraction, as the reference builds with
// -ffp-contract=off); sqrt and divide are IEEE correctly rounded.
// Reductions follow the reference's accumulation contract: L lanes (8 for
// f32, 4 for f64) accumulate the leading multiple-of-L prefix, lane j taking
// elements j, j+L, j+2L, ... in order, the lanes fold left to right, then the
// tail is appended in order.  That order is sequential per lane by
// definition, so a reduction runs L threads wide; the training step's own
// reductions (kernels.cu) are parallel and tolerance-matched instead.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "hetpar_b200.h"
#include "hp_common.h"
#include "kernels.h"

namespace hp {
namespace kern {

template <class T> __device__ __forceinline__ T add_rn(T a, T b);
template <class T> __device__ __forceinline__ T mul_rn(T a, T b);
template <class T> __device__ __forceinline__ T sub_rn(T a, T b);
template <class T> __device__ __forceinline__ T div_rn(T a, T b);
template <class T> __device__ __forceinline__ T sqrt_rn(T a);
template <> __device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
template <> __device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
template <> __device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
template <> __device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }
template <> __device__ __forceinline__ float sqrt_rn(float a) { return __fsqrt_rn(a); }
template <> __device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
template <> __device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
template <> __device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
template <> __device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }
template <> __device__ __forceinline__ double sqrt_rn(double a) { return __dsqrt_rn(a); }

template <class T>
constexpr int lanes() {
  return sizeof(T) == 8 ? 4 : 8;
}

// kind 0: dot, 1: sum, 2: max
template <class T, int KIND>
__global__ void reduce_kernel(const T* __restrict__ a, const T* __restrict__ b, uint64_t n,
                              T* __restrict__ out) {
  constexpr int L = lanes<T>();
  __shared__ T acc[L];
  const int j = threadIdx.x;
  const uint64_t n0 = n - n % L;
  T s = KIND == 2 ? -INFINITY : T(0);
  for (uint64_t i = j; i < n0; i += L) {
    if constexpr (KIND == 0) s = add_rn(s, mul_rn(a[i], b[i]));
    else if constexpr (KIND == 1) s = add_rn(s, a[i]);
    else s = a[i] > s ? a[i] : s;
  }
  acc[j] = s;
  __syncthreads();
  if (j == 0) {
    T r = acc[0];
    for (int k = 1; k < L; ++k) {
      if constexpr (KIND == 2) r = acc[k] > r ? acc[k] : r;
      else r = add_rn(r, acc[k]);
    }
    for (uint64_t i = n0; i < n; ++i) {
      if constexpr (KIND == 0) r = add_rn(r, mul_rn(a[i], b[i]));
      else if constexpr (KIND == 1) r = add_rn(r, a[i]);
      else r = a[i] > r ? a[i] : r;
    }
    *out = r;
  }
}

// op 0 add, 1 scale, 2 axpy, 3 relu, 4 relu_bwd, 5 sgd_update
template <class T, int OP>
__global__ void elementwise_kernel(const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ y,
                                   uint64_t n, T s) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    if constexpr (OP == 0) y[i] = add_rn(a[i], b[i]);                       // out = a + b
    else if constexpr (OP == 1) y[i] = mul_rn(a[i], s);                     // out = a * s
    else if constexpr (OP == 2) y[i] = add_rn(y[i], mul_rn(s, a[i]));       // y += alpha x
    else if constexpr (OP == 3) y[i] = a[i] > T(0) ? a[i] : T(0);           // relu
    else if constexpr (OP == 4) y[i] = add_rn(y[i], a[i] > T(0) ? b[i] : T(0));  // da += relu'(a) g
    else y[i] = sub_rn(y[i], mul_rn(s, a[i]));                              // p -= lr g
  }
}

template <class T>
__global__ void adam_kernel_ref(T* __restrict__ p, T* __restrict__ m, T* __restrict__ v,
                                const T* __restrict__ g, uint64_t n, T lr, T b1, T b2, T eps, T c1,
                                T c2) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const T gi = g[i];
    const T mi = add_rn(mul_rn(b1, m[i]), mul_rn(sub_rn(T(1), b1), gi));
    const T vi = add_rn(mul_rn(b2, v[i]), mul_rn(sub_rn(T(1), b2), mul_rn(gi, gi)));
    m[i] = mi;
    v[i] = vi;
    const T mh = mul_rn(mi, c1), vh = mul_rn(vi, c2);
    p[i] = sub_rn(p[i], mul_rn(lr, div_rn(mh, add_rn(sqrt_rn(vh), eps))));
  }
}

inline unsigned grid_for(uint64_t n) {
  const uint64_t g = (n + 255) / 256;
  return static_cast<unsigned>(g < 148 * 8 ? (g ? g : 1) : 148 * 8);
}

template <class T, int KIND>
void reduce(const T* a, const T* b, uint64_t n, T* out, cudaStream_t s) {
  reduce_kernel<T, KIND><<<1, lanes<T>(), 0, s>>>(a, b, n, out);
  HP_CUDA(cudaGetLastError());
  count_launch();
}
template <class T, int OP>
void elementwise(const T* a, const T* b, T* y, uint64_t n, T sc, cudaStream_t s) {
  if (n == 0) return;
  elementwise_kernel<T, OP><<<grid_for(n), 256, 0, s>>>(a, b, y, n, sc);
  HP_CUDA(cudaGetLastError());
  count_launch();
}
template <class T>
void adam(T* p, T* m, T* v, const T* g, uint64_t n, T lr, T b1, T b2, T eps, T c1, T c2,
          cudaStream_t s) {
  if (n == 0) return;
  adam_kernel_ref<T><<<grid_for(n), 256, 0, s>>>(p, m, v, g, n, lr, b1, b2, eps, c1, c2);
  HP_CUDA(cudaGetLastError());
  count_launch();
}

}  // namespace kern
}  // namespace hp

#define ST(x) static_cast<cudaStream_t>(x)
#define HP_KERN_ABI(T, SFX)                                                                       \
  hp_status hp_kern_dot_##SFX(const T* a, const T* b, uint64_t n, T* out, void* s) {              \
    HP_API_BEGIN hp::kern::reduce<T, 0>(a, b, n, out, ST(s));                                     \
    HP_API_END                                                                                    \
  }                                                                                               \
  hp_status hp_kern_sum_##SFX(const T* a, uint64_t n, T* out, void* s) {                          \
    HP_API_BEGIN hp::kern::reduce<T, 1>(a, nullptr, n, out, ST(s));                               \
    HP_API_END                                                                                    \
  }                                                                                               \
  hp_status hp_kern_maxv_##SFX(const T* a, uint64_t n, T* out, void* s) {                         \
    HP_API_BEGIN hp::kern::reduce<T, 2>(a, nullptr, n, out, ST(s));                               \
    HP_API_END                                                                                    \
  }                                                                                               \
  hp_status hp_kern_add_##SFX(const T* a, const T* b, T* out, uint64_t n, void* s) {              \
    HP_API_BEGIN hp::kern::elementwise<T, 0>(a, b, out, n, T(0), ST(s));                          \
    HP_API_END                                                                                    \
  }                                                                                               \
  hp_status hp_kern_scale_##SFX(const T* a, T sc, T* out, uint64_t n, void* s) {                  \
    HP_API_BEGIN hp::kern::elementwise<T, 1>(a, nullptr, out, n, sc, ST(s));                      \
    HP_API_END                                                                                    \
  }                                                                                               \
  hp_status hp_kern_axpy_##SFX(T alpha, const T* x, T* y, uint64_t n, void* s) {                  \
    HP_API_BEGIN hp::kern::elementwise<T, 2>(x, nullptr, y, n, alpha, ST(s));                     \
    HP_API_END                                                                                    \
  }                                                                                               \
  hp_status hp_kern_relu_##SFX(const T* a, T* out, uint64_t n, void* s) {                         \
    HP_API_BEGIN hp::kern::elementwise<T, 3>(a, nullptr, out, n, T(0), ST(s));                    \
    HP_API_END                                                                                    \
  }                                                                                               \
  hp_status hp_kern_relu_bwd_##SFX(const T* a, const T* g, T* da, uint64_t n, void* s) {          \
    HP_API_BEGIN hp::kern::elementwise<T, 4>(a, g, da, n, T(0), ST(s));                           \
    HP_API_END                                                                                    \
  }                                                                                               \
  hp_status hp_kern_sgd_update_##SFX(T* p, const T* g, uint64_t n, T lr, void* s) {               \
    HP_API_BEGIN hp::kern::elementwise<T, 5>(g, nullptr, p, n, lr, ST(s));                        \
    HP_API_END                                                                                    \
  }                                                                                               \
  hp_status hp_kern_adam_update_##SFX(T* p, T* m, T* v, const T* g, uint64_t n, T lr, T b1, T b2, \
                                      T eps, T c1, T c2, void* s) {                               \
    HP_API_BEGIN hp::kern::adam<T>(p, m, v, g, n, lr, b1, b2, eps, c1, c2, ST(s));                \
    HP_API_END                                                                                    \
  }

extern "C" {
HP_KERN_ABI(float, f32)
HP_KERN_ABI(double, f64)
}
