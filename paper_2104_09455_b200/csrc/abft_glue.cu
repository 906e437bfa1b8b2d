// abft_glue.cu — the non-linear glue between the protected layers of a CNN forward (config C5),
// plus the per-CTA partial reduction the batch-sharded verification all-reduces.
//
// The reference protects linear layers only and models a network as its linear-layer list
// (shapes.py:198-212, model_to_gemm_sequence); the layers in between (pooling, channel shuffle)
// are not checked, here as in the paper (overhead over the linear layers).  They
// run on the NHWC activations the protected kernels produce, into buffers planned once, so a
// whole forward is one stream of launches that a CUDA graph captures.  All are HBM-bound:
// 16-byte (8-channel) vectors per thread where the layout allows it.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <string>
#include <vector>

#include "abft_common.cuh"

namespace abft {

template <typename T>
struct Max2;
template <>
struct Max2<__half> {
  static __device__ __forceinline__ uint32_t op(uint32_t a, uint32_t b) {
    __half2 r = __hmax2(*reinterpret_cast<__half2*>(&a), *reinterpret_cast<__half2*>(&b));
    return *reinterpret_cast<uint32_t*>(&r);
  }
  static constexpr uint32_t lowest = 0xFC00FC00u;   // -inf, -inf
};
template <>
struct Max2<__nv_bfloat16> {
  static __device__ __forceinline__ uint32_t op(uint32_t a, uint32_t b) {
    __nv_bfloat162 r = __hmax2(*reinterpret_cast<__nv_bfloat162*>(&a), *reinterpret_cast<__nv_bfloat162*>(&b));
    return *reinterpret_cast<uint32_t*>(&r);
  }
  static constexpr uint32_t lowest = 0xFF80FF80u;
};

template <typename T>
struct Unpack2;
template <>
struct Unpack2<__half> {
  static __device__ __forceinline__ float2 f(uint32_t u) { return __half22float2(*reinterpret_cast<__half2*>(&u)); }
};
template <>
struct Unpack2<__nv_bfloat16> {
  static __device__ __forceinline__ float2 f(uint32_t u) {
    return __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&u));
  }
};

// out[n][p][q][c] = max over the window (padding never wins), one 8-channel vector per thread.
// I: the index type of the (pixel, vector) decomposition — 32-bit whenever the tensor allows (the
// 64-bit divisions made the kernel instruction-bound, ~2/3 of HBM bandwidth)
template <typename T, typename I>
__global__ void __launch_bounds__(256) maxpool_nhwc_kernel(const T* __restrict__ x, int H, int W, int C, long long ldx,
                                                           int P, int Q, int k, int s, int pad, T* __restrict__ out,
                                                           long long ldo, long long total_vec) {
  const I cv = (I)(C / 8);
  const I total = (I)total_vec;
  for (I i = (I)(blockIdx.x * blockDim.x + threadIdx.x); i < total; i += (I)(gridDim.x * blockDim.x)) {
    const int c8 = (int)(i % cv);
    I pix = i / cv;
    const int q = (int)(pix % (I)Q);
    pix /= (I)Q;
    const int p = (int)(pix % (I)P);
    const long long n = (long long)(pix / (I)P);
    uint4 m = make_uint4(Max2<T>::lowest, Max2<T>::lowest, Max2<T>::lowest, Max2<T>::lowest);
    const int h0 = p * s - pad, w0 = q * s - pad;
    for (int dh = 0; dh < k; ++dh) {
      const int hh = h0 + dh;
      if (hh < 0 || hh >= H) continue;
      for (int dw = 0; dw < k; ++dw) {
        const int ww = w0 + dw;
        if (ww < 0 || ww >= W) continue;
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(x + ((n * H + hh) * W + ww) * ldx + c8 * 8));
        m.x = Max2<T>::op(m.x, u.x);
        m.y = Max2<T>::op(m.y, u.y);
        m.z = Max2<T>::op(m.z, u.z);
        m.w = Max2<T>::op(m.w, u.w);
      }
    }
    *reinterpret_cast<uint4*>(out + ((n * P + p) * Q + q) * ldo + c8 * 8) = m;
  }
}

// The same pooling, and the column sums of its output (bucket 0 of the window sums; a 3x3
// consumer's border buckets come from border_sums): a thread keeps one 8-channel vector and
// strides over output pixels, summing the stored (rounded) maxima in registers; one smem
// reduction and one global atomic per channel and CTA
template <typename T>
__global__ void __launch_bounds__(256) maxpool_ws_kernel(const T* __restrict__ x, int H, int W, int C, long long ldx,
                                                         int P, int Q, int k, int s, int pad, T* __restrict__ out,
                                                         long long ldo, int npix, float* __restrict__ wsum) {
  extern __shared__ float wsm[];          // [C]
  const int cv = C / 8;
  const int lanes_p = blockDim.x / cv;    // pixels in flight per CTA
  for (int i = threadIdx.x; i < C; i += blockDim.x) wsm[i] = 0.f;
  __syncthreads();
  const int c8 = threadIdx.x % cv, lp = threadIdx.x / cv;
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.f;
  if (lp < lanes_p) {
    // two output pixels per iteration: twice the loads in flight (the loop is latency-bound)
    const int step = gridDim.x * lanes_p;
    auto pool = [&](int pix, uint4& m) {
      const int q = pix % Q;
      const int pq = pix / Q;
      const int p = pq % P;
      const long long n = pq / P;
      m = make_uint4(Max2<T>::lowest, Max2<T>::lowest, Max2<T>::lowest, Max2<T>::lowest);
      const int h0 = p * s - pad, w0 = q * s - pad;
      for (int dh = 0; dh < k; ++dh) {
        const int hh = h0 + dh;
        if (hh < 0 || hh >= H) continue;
        for (int dw = 0; dw < k; ++dw) {
          const int ww = w0 + dw;
          if (ww < 0 || ww >= W) continue;
          const uint4 u = __ldg(reinterpret_cast<const uint4*>(x + ((n * H + hh) * W + ww) * ldx + c8 * 8));
          m.x = Max2<T>::op(m.x, u.x);
          m.y = Max2<T>::op(m.y, u.y);
          m.z = Max2<T>::op(m.z, u.z);
          m.w = Max2<T>::op(m.w, u.w);
        }
      }
      *reinterpret_cast<uint4*>(out + (long long)pix * ldo + c8 * 8) = m;
    };
    auto add = [&](const uint4& m) {
      const uint32_t w4[4] = {m.x, m.y, m.z, m.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = Unpack2<T>::f(w4[e]);
        acc[2 * e] += f.x;
        acc[2 * e + 1] += f.y;
      }
    };
    int pix = blockIdx.x * lanes_p + lp;
    for (; pix + step < npix; pix += 2 * step) {
      uint4 m0, m1;
      pool(pix, m0);
      pool(pix + step, m1);
      add(m0);
      add(m1);
    }
    if (pix < npix) {
      uint4 m0;
      pool(pix, m0);
      add(m0);
    }
#pragma unroll
    for (int e = 0; e < 8; ++e)
      if (acc[e] != 0.f) atomicAdd(&wsm[c8 * 8 + e], acc[e]);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < C; i += blockDim.x)
    if (wsm[i] != 0.f) atomicAdd(&wsum[i], wsm[i]);
}

// out[n][c] = mean over the H*W pixels of image n (fp32 sum, rounded once); CTA = (image, 256-vector slab)
template <typename T>
__global__ void __launch_bounds__(256) avgpool_nhwc_kernel(const T* __restrict__ x, int HW, int C, long long ldx,
                                                           T* __restrict__ out, long long ldo) {
  __shared__ float part[8][8 * 32];
  const int cv = C / 8;
  const long long n = blockIdx.x;
  const int v0 = blockIdx.y * 32;
  const int vi = threadIdx.x & 31, rg = threadIdx.x >> 5;   // 32 vectors x 8 pixel groups
  const int v = v0 + vi;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (v < cv) {
    for (int px = rg; px < HW; px += 8) {
      const uint4 u = __ldg(reinterpret_cast<const uint4*>(x + (n * HW + px) * ldx + v * 8));
      const T* e = reinterpret_cast<const T*>(&u);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += (float)e[j];
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) part[rg][vi * 8 + j] = acc[j];
  __syncthreads();
  const int c = threadIdx.x;   // 256 channels of this slab
  if (v0 * 8 + c < C) {
    float s = 0.f;
#pragma unroll
    for (int g = 0; g < 8; ++g) s += part[g][c];
    out[n * ldo + v0 * 8 + c] = (T)(s / (float)HW);
  }
}

// ShuffleNet v2 unit output: channel_shuffle(cat(x1, b), 2) — logical channel 2i + g is x1[i]
// (g = 0) or b[i] (g = 1); stored in the "halves" layout (logical channels [0, C/2) at physical
// [0, C/2), [C/2, C) at physical [half_pad, half_pad + C/2)) so the next unit's chunk(2) halves
// are 16-byte aligned channel slices.  One (x1[i], b[i]) pair -> one 4-byte store per thread.
template <typename T, typename I>
__global__ void __launch_bounds__(256) interleave2_kernel(const T* __restrict__ x1, long long ld1,
                                                          const T* __restrict__ b, long long ld2, int half,
                                                          T* __restrict__ out, long long ldo, int half_pad,
                                                          long long total) {
  // one thread: channels (2j, 2j+1) of both sources (one 4-byte load each) -> output channels
  // 4j .. 4j+3 as two 4-byte pairs (a pair never straddles the half boundary: half is even)
  const I hp = (I)(half / 2);
  const I tot = (I)(total / 2);
  for (I t = (I)(blockIdx.x * blockDim.x + threadIdx.x); t < tot; t += (I)(gridDim.x * blockDim.x)) {
    const I pixi = t / hp;
    const int j = (int)(t - pixi * hp);
    const long long pix = (long long)pixi;
    const uint32_t a2 = *reinterpret_cast<const uint32_t*>(x1 + pix * ld1 + 2 * j);
    const uint32_t b2 = *reinterpret_cast<const uint32_t*>(b + pix * ld2 + 2 * j);
    const int l0 = 4 * j, l1 = 4 * j + 2;
    const int p0 = l0 < half ? l0 : half_pad + (l0 - half);
    const int p1 = l1 < half ? l1 : half_pad + (l1 - half);
    T* o = out + pix * ldo;
    *reinterpret_cast<uint32_t*>(o + p0) = __byte_perm(a2, b2, 0x5410);   // (x1[2j], b[2j])
    *reinterpret_cast<uint32_t*>(o + p1) = __byte_perm(a2, b2, 0x7632);   // (x1[2j+1], b[2j+1])
  }
}

// [n][cap][2] per-CTA (lhs, rhs) slots -> [n][2] sums (fp64), for the batch-sharded all-reduce
__global__ void sum_partials_kernel(const double* __restrict__ partials, int cap, int ntasks, double* __restrict__ sums) {
  const int task = blockIdx.x * 4 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (task >= ntasks) return;
  double l = 0.0, r = 0.0;
  for (int i = lane; i < cap; i += 32) {
    l += partials[((long long)task * cap + i) * 2];
    r += partials[((long long)task * cap + i) * 2 + 1];
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    l += __shfl_xor_sync(0xffffffffu, l, o);
    r += __shfl_xor_sync(0xffffffffu, r, o);
  }
  if (lane == 0) {
    sums[2 * task] = l;
    sums[2 * task + 1] = r;
  }
}

int grid_for(long long work) {
  return (int)std::max<long long>(1, std::min<long long>((work + 255) / 256, 16LL * num_sms()));
}

}  // namespace abft

using namespace abft;

extern "C" __attribute__((visibility("default"))) int abft_nhwc_maxpool(const void* x, int32_t n, int32_t h, int32_t w,
                                                                       int32_t c, int64_t ldx, int32_t k, int32_t stride,
                                                                       int32_t pad, int32_t ceil_mode, int32_t dtype,
                                                                       void* out, int64_t ldo, void* stream) {
  if (n < 1 || h < 1 || w < 1 || c < 8 || c % 8 || k < 1 || stride < 1 || pad < 0 || 2 * pad > k)
    return fail(ABFT_E_SHAPE, "maxpool: bad extents (channels a multiple of 8, pad <= k/2)");
  if (ldx < c || ldx % 8 || ldo < c || ldo % 8) return fail(ABFT_E_SHAPE, "maxpool: ldx/ldo must be >= c and a multiple of 8");
  auto osz = [&](int len) {
    const int num = len + 2 * pad - k;
    int o = (ceil_mode ? (num + stride - 1) / stride : num / stride) + 1;
    if (ceil_mode && (o - 1) * stride >= len + pad) --o;   // the last window must start inside the input
    return o;
  };
  const int P = osz(h), Q = osz(w);
  if (P < 1 || Q < 1) return fail(ABFT_E_SHAPE, "maxpool: empty output");
  const long long total = (long long)n * P * Q * (c / 8);
  cudaStream_t st = as_stream(stream);
  const bool small = total < (1LL << 31) - (long long)grid_for(total) * 256;
  if (dtype == ABFT_BF16) {
    if (small)
      maxpool_nhwc_kernel<__nv_bfloat16, uint32_t><<<grid_for(total), 256, 0, st>>>(
          (const __nv_bfloat16*)x, h, w, c, ldx, P, Q, k, stride, pad, (__nv_bfloat16*)out, ldo, total);
    else
      maxpool_nhwc_kernel<__nv_bfloat16, long long><<<grid_for(total), 256, 0, st>>>(
          (const __nv_bfloat16*)x, h, w, c, ldx, P, Q, k, stride, pad, (__nv_bfloat16*)out, ldo, total);
  } else {
    if (small)
      maxpool_nhwc_kernel<__half, uint32_t><<<grid_for(total), 256, 0, st>>>((const __half*)x, h, w, c, ldx, P, Q, k,
                                                                            stride, pad, (__half*)out, ldo, total);
    else
      maxpool_nhwc_kernel<__half, long long><<<grid_for(total), 256, 0, st>>>((const __half*)x, h, w, c, ldx, P, Q, k,
                                                                             stride, pad, (__half*)out, ldo, total);
  }
  return cuda_check(cudaGetLastError(), "maxpool launch");
}

extern "C" __attribute__((visibility("default"))) int abft_nhwc_maxpool_ws(const void* x, int32_t n, int32_t h,
                                                                          int32_t w, int32_t c, int64_t ldx, int32_t k,
                                                                          int32_t stride, int32_t pad, int32_t ceil_mode,
                                                                          int32_t dtype, void* out, int64_t ldo,
                                                                          float* wsum, int32_t ws_ld, int32_t ws_mode,
                                                                          void* stream) {
  if (n < 1 || h < 1 || w < 1 || c < 8 || c % 8 || c > 2048 || k < 1 || stride < 1 || pad < 0 || 2 * pad > k)
    return fail(ABFT_E_SHAPE, "maxpool_ws: bad extents (channels a multiple of 8 up to 2048, pad <= k/2)");
  if (ldx < c || ldx % 8 || ldo < c || ldo % 8) return fail(ABFT_E_SHAPE, "maxpool_ws: ldx/ldo must be >= c and a multiple of 8");
  if (wsum == nullptr || ws_ld < c || (ws_mode != 1 && ws_mode != 2))
    return fail(ABFT_E_VALUE, "maxpool_ws: window sums [1 or 9][ws_ld >= c], ws_mode 1 or 2");
  auto osz = [&](int len) {
    const int num = len + 2 * pad - k;
    int o = (ceil_mode ? (num + stride - 1) / stride : num / stride) + 1;
    if (ceil_mode && (o - 1) * stride >= len + pad) --o;
    return o;
  };
  const int P = osz(h), Q = osz(w);
  if (P < 1 || Q < 1) return fail(ABFT_E_SHAPE, "maxpool_ws: empty output");
  const int cv = c / 8;
  const int threads = cv >= 256 ? cv : (256 / cv) * cv;
  if (threads > 256) return fail(ABFT_E_UNSUPPORTED, "maxpool_ws: more than 256 channel vectors");
  const size_t smem = (size_t)c * sizeof(float);
  (void)ws_ld;
  const long long npix = (long long)n * P * Q;
  if (npix >= (1LL << 30)) return fail(ABFT_E_UNSUPPORTED, "maxpool_ws: more than 2^30 output pixels");
  const int grid = std::max(1, std::min<int>(8 * num_sms(), (int)((npix + 63) / 64)));
  cudaStream_t st = as_stream(stream);
  if (dtype == ABFT_BF16)
    maxpool_ws_kernel<__nv_bfloat16><<<grid, threads, smem, st>>>((const __nv_bfloat16*)x, h, w, c, ldx, P, Q, k, stride,
                                                                   pad, (__nv_bfloat16*)out, ldo, (int)npix, wsum);
  else
    maxpool_ws_kernel<__half><<<grid, threads, smem, st>>>((const __half*)x, h, w, c, ldx, P, Q, k, stride, pad,
                                                            (__half*)out, ldo, (int)npix, wsum);
  return cuda_check(cudaGetLastError(), "maxpool_ws launch");
}

extern "C" __attribute__((visibility("default"))) int abft_nhwc_avgpool(const void* x, int32_t n, int32_t hw, int32_t c,
                                                                       int64_t ldx, int32_t dtype, void* out, int64_t ldo,
                                                                       void* stream) {
  if (n < 1 || hw < 1 || c < 8 || c % 8 || ldx < c || ldx % 8 || ldo < c)
    return fail(ABFT_E_SHAPE, "avgpool: bad extents (channels a multiple of 8)");
  dim3 grid((unsigned)n, (unsigned)((c / 8 + 31) / 32));
  cudaStream_t st = as_stream(stream);
  if (dtype == ABFT_BF16)
    avgpool_nhwc_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>((const __nv_bfloat16*)x, hw, c, ldx, (__nv_bfloat16*)out, ldo);
  else
    avgpool_nhwc_kernel<__half><<<grid, 256, 0, st>>>((const __half*)x, hw, c, ldx, (__half*)out, ldo);
  return cuda_check(cudaGetLastError(), "avgpool launch");
}

extern "C" __attribute__((visibility("default"))) int abft_nhwc_interleave2(const void* x1, int64_t ld1, const void* b,
                                                                           int64_t ld2, int64_t pixels, int32_t half,
                                                                           void* out, int64_t ldo, int32_t half_pad,
                                                                           int32_t dtype, void* stream) {
  if (pixels < 1 || half < 2 || half % 2 || half_pad < half || half_pad % 2 || ldo < half_pad + half || ld1 < half ||
      ld2 < half)
    return fail(ABFT_E_SHAPE, "interleave2: bad extents (half even, half_pad >= half)");
  const long long total = pixels * half;
  cudaStream_t st = as_stream(stream);
  // 16-bit elements either way: the kernel only moves them
  (void)dtype;
  if ((ld1 % 2) || (ld2 % 2) || (ldo % 2) || (reinterpret_cast<uintptr_t>(x1) & 3) ||
      (reinterpret_cast<uintptr_t>(b) & 3) || (reinterpret_cast<uintptr_t>(out) & 3))
    return fail(ABFT_E_VALUE, "interleave2: 4-byte aligned rows (even ld1 / ld2 / ldo)");
  if (total / 2 < (1LL << 31) - (long long)grid_for(total / 2) * 256)
    interleave2_kernel<__half, uint32_t><<<grid_for(total / 2), 256, 0, st>>>(
        (const __half*)x1, ld1, (const __half*)b, ld2, half, (__half*)out, ldo, half_pad, total);
  else
    interleave2_kernel<__half, long long><<<grid_for(total / 2), 256, 0, st>>>(
        (const __half*)x1, ld1, (const __half*)b, ld2, half, (__half*)out, ldo, half_pad, total);
  return cuda_check(cudaGetLastError(), "interleave2 launch");
}

// The border buckets (1..8) of a 3x3 consumer's window sums, from the activation's border pixels
// only.  Each bucket is one pixel segment per image — 1: row 0, 2: row H-1, 3: column 0,
// 4: column W-1 (all of them, corners included), 5..8: the corners (0,0), (0,W-1), (H-1,0),
// (H-1,W-1) — so a CTA = (bucket, group of images) and a thread = (8-channel vector, slice of the
// group's segment pixels) keeps ONE 8-float accumulator, with up to 8 loads in flight.  The CTA's
// slices meet in shared memory and leave as one 16-byte atomic per 4 channels.  Bucket 0 (all
// pixels) comes from the producer's epilogue.
// one CTA of the border pass: bucket `bucket`, images [grp * imgs_per_cta, ...); bsm >= parts * C floats
template <typename T>
__device__ __forceinline__ void border_block(const T* __restrict__ x, int nimg, int imgs_per_cta, int H, int W, int C,
                                             long long ldx, float* __restrict__ ws, int ws_ld, int bucket, int grp,
                                             float* bsm) {
  const int cv = C / 8;
  const int parts = 256 / cv;
  const int c8 = threadIdx.x % cv, part = threadIdx.x / cv;
  const int seg = bucket <= 2 ? W : (bucket <= 4 ? H : 1);      // pixels per image
  const int img0 = grp * imgs_per_cta;
  const int nimg_cta = min(imgs_per_cta, nimg - img0);
  const int items = nimg_cta * seg;
  auto pixel = [&](int it) -> long long {
    const int im = img0 + it / seg, i = it - (it / seg) * seg;
    int hh, ww;
    switch (bucket) {
      case 1: hh = 0; ww = i; break;
      case 2: hh = H - 1; ww = i; break;
      case 3: hh = i; ww = 0; break;
      case 4: hh = i; ww = W - 1; break;
      case 5: hh = 0; ww = 0; break;
      case 6: hh = 0; ww = W - 1; break;
      case 7: hh = H - 1; ww = 0; break;
      default: hh = H - 1; ww = W - 1; break;
    }
    return ((long long)im * H + hh) * W + ww;
  };
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.f;
  auto add = [&](const uint4& u) {
    const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = Unpack2<T>::f(w4[e]);
      acc[2 * e] += f.x;
      acc[2 * e + 1] += f.y;
    }
  };
  if (part < parts) {
    const T* xc = x + c8 * 8;
    int it = part;
    for (; it + 7 * parts < items; it += 8 * parts) {
      uint4 u[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) u[k] = __ldg(reinterpret_cast<const uint4*>(xc + pixel(it + k * parts) * ldx));
#pragma unroll
      for (int k = 0; k < 8; ++k) add(u[k]);
    }
    for (; it < items; it += parts) add(__ldg(reinterpret_cast<const uint4*>(xc + pixel(it) * ldx)));
#pragma unroll
    for (int e = 0; e < 8; ++e) bsm[part * C + c8 * 8 + e] = acc[e];
  }
  __syncthreads();
  float* dst = ws + (long long)bucket * ws_ld;
  for (int c4 = threadIdx.x; c4 < C / 4; c4 += blockDim.x) {
    float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int q = 0; q < parts; ++q) {
      const float4 v = *reinterpret_cast<const float4*>(bsm + q * C + c4 * 4);
      t.x += v.x; t.y += v.y; t.z += v.z; t.w += v.w;
    }
    atomicAdd(reinterpret_cast<float4*>(dst + c4 * 4), t);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) border_sums_kernel(const T* __restrict__ x, int nimg, int imgs_per_cta, int H,
                                                          int W, int C, long long ldx, float* __restrict__ ws,
                                                          int ws_ld) {
  __shared__ __align__(16) float bsm[2048];     // [parts][C]: parts * C = 256 / (C / 8) * C <= 2048
  border_block<T>(x, nimg, imgs_per_cta, H, W, C, ldx, ws, ws_ld, 1 + (int)blockIdx.y, (int)blockIdx.x, bsm);
}

// images per CTA of the border pass: ~16 segment pixels per thread slot of the longest buckets
static int border_imgs_per_cta(int n, int h, int w, int c) {
  const int parts = 256 / (c / 8);
  const int seg = std::max(h, w);
  return std::max(1, std::min(n, (16 * parts + seg - 1) / seg));
}

extern "C" __attribute__((visibility("default"))) int abft_nhwc_border_sums(const void* x, int32_t n, int32_t h,
                                                                           int32_t w, int32_t c, int64_t ldx,
                                                                           int32_t dtype, float* wsum, int32_t ws_ld,
                                                                           void* stream) {
  if (n < 1 || h < 1 || w < 1 || c < 8 || c % 8 || c > 1024 || ldx < c || ldx % 8 || wsum == nullptr || ws_ld < c ||
      ws_ld % 4 || (reinterpret_cast<uintptr_t>(wsum) & 15))
    return fail(ABFT_E_SHAPE, "border_sums: bad extents (channels a multiple of 8 up to 1024, ldx >= c, "
                              "16-byte aligned wsum rows)");
  const int ipc = border_imgs_per_cta(n, h, w, c);
  const dim3 grid((unsigned)((n + ipc - 1) / ipc), 8u);
  cudaStream_t st = as_stream(stream);
  if (dtype == ABFT_BF16)
    border_sums_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>((const __nv_bfloat16*)x, n, ipc, h, w, c, ldx, wsum, ws_ld);
  else
    border_sums_kernel<__half><<<grid, 256, 0, st>>>((const __half*)x, n, ipc, h, w, c, ldx, wsum, ws_ld);
  return cuda_check(cudaGetLastError(), "border_sums launch");
}

// The consumer's global lhs from the producer's window sums (abft_window_lhs): one (tap, channel)
// term per thread over up to 64 CTAs, fp64, one atomic per CTA.
// colck_im2col(r, s, c) of a 3x3 / stride 1 / pad 1 conv over an H x W input = the sum over the
// input rows / columns tap (r, s) reads: all of them minus the row the tap never reaches (r = 0
// misses the last row, r = 2 the first) minus the column likewise, plus their corner (counted
// twice).  Buckets: 0 all, 1 p0, 2 pL, 3 q0, 4 qL, 5 (p0,q0), 6 (p0,qL), 7 (pL,q0), 8 (pL,qL).
__device__ __forceinline__ void window_block(const float* __restrict__ ws, int ld, int C, int R, int S, int ck,
                                             const float* __restrict__ rowck, const float* __restrict__ bias,
                                             int n_out, long long M, double* __restrict__ lhs, int blk, int nblk,
                                             double* red) {
  double acc = 0.0;
  const int taps = R * S;
  for (int i = blk * blockDim.x + threadIdx.x; i < taps * C; i += nblk * blockDim.x) {
    const int tap = i / C, c = i - (i / C) * C;
    double col = ws[c];
    if (R == 3) {
      const int r = tap / 3, sx = tap - (tap / 3) * 3;
      const int rb = r == 0 ? 2 : (r == 2 ? 1 : 0);     // the row bucket the tap misses
      const int cb = sx == 0 ? 4 : (sx == 2 ? 3 : 0);    // the column bucket
      if (rb) col -= ws[(long long)rb * ld + c];
      if (cb) col -= ws[(long long)cb * ld + c];
      if (rb && cb) col += ws[(long long)(5 + (rb == 2 ? 2 : 0) + (cb == 4 ? 1 : 0)) * ld + c];
    }
    acc += col * (double)rowck[(long long)tap * ck + c];
  }
  if (bias != nullptr && blk == 0)
    for (int j = threadIdx.x; j < n_out; j += blockDim.x) acc += (double)M * (double)bias[j];
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    atomicAdd(lhs, t);
  }
}

__global__ void __launch_bounds__(256) window_lhs_kernel(const float* __restrict__ ws, int ld, int C, int R, int S,
                                                         int ck, const float* __restrict__ rowck,
                                                         const float* __restrict__ bias, int n_out, long long M,
                                                         double* __restrict__ lhs) {
  __shared__ double red[8];
  window_block(ws, ld, C, R, S, ck, rowck, bias, n_out, M, lhs, (int)blockIdx.x, (int)gridDim.x, red);
}

// ---- batched fused-checksum work of a whole forward (abft_fused_lhs_batch_*): every producer's
// border buckets in ONE launch, then every fused consumer's window lhs in ONE launch, from a
// device table written once (the activations stay live until the end of the forward)
struct __align__(16) BorderEntry {
  const void* x;
  float* ws;
  long long ldx;
  int n, h, w, c, ws_ld, ipc, groups, begin;
  int pad[3];
};
struct __align__(16) WindowEntry {
  const float* ws;
  const float* rowck;
  const float* bias;
  double* lhs;
  long long M;
  int ld, C, R, S, ck, n_out, begin, nblk;
};
struct __align__(16) FusedBatchHeader {
  int nb, nw, border_blocks, window_blocks;
};

template <typename T>
__global__ void __launch_bounds__(256) border_batch_kernel(const FusedBatchHeader* __restrict__ hdr) {
  __shared__ __align__(16) float bsm[2048];
  const BorderEntry* e = reinterpret_cast<const BorderEntry*>(hdr + 1);
  int i = 0;
  while (i + 1 < hdr->nb && (int)blockIdx.x >= e[i + 1].begin) ++i;
  const BorderEntry& t = e[i];
  const int local = (int)blockIdx.x - t.begin;
  border_block<T>(reinterpret_cast<const T*>(t.x), t.n, t.ipc, t.h, t.w, t.c, t.ldx, t.ws, t.ws_ld,
                  1 + local / t.groups, local % t.groups, bsm);
}

__global__ void __launch_bounds__(256) window_batch_kernel(const FusedBatchHeader* __restrict__ hdr) {
  __shared__ double red[8];
  const WindowEntry* e = reinterpret_cast<const WindowEntry*>(reinterpret_cast<const BorderEntry*>(hdr + 1) + hdr->nb);
  int i = 0;
  while (i + 1 < hdr->nw && (int)blockIdx.x >= e[i + 1].begin) ++i;
  const WindowEntry& t = e[i];
  window_block(t.ws, t.ld, t.C, t.R, t.S, t.ck, t.rowck, t.bias, t.n_out, t.M, t.lhs, (int)blockIdx.x - t.begin,
               t.nblk, red);
}

extern "C" __attribute__((visibility("default"))) int abft_window_lhs(const float* wsum, int32_t ws_ld, int32_t C,
                                                                     int32_t R, int32_t S, int32_t ck,
                                                                     const float* rowck, const float* bias,
                                                                     int32_t n_out, int64_t M, double* lhs,
                                                                     void* stream) {
  if (wsum == nullptr || rowck == nullptr || lhs == nullptr) return fail(ABFT_E_VALUE, "window_lhs: null pointer");
  if (!((R == 1 && S == 1) || (R == 3 && S == 3))) return fail(ABFT_E_UNSUPPORTED, "window_lhs: 1x1 or 3x3 consumers");
  if (C < 1 || ws_ld < C || ck < C || M < 0 || (bias != nullptr && n_out < 1))
    return fail(ABFT_E_SHAPE, "window_lhs: bad extents");
  const int grid = std::max(1, std::min(64, (R * S * C + 255) / 256));
  window_lhs_kernel<<<grid, 256, 0, as_stream(stream)>>>(wsum, ws_ld, C, R, S, ck, rowck, bias, n_out, M, lhs);
  return cuda_check(cudaGetLastError(), "window_lhs launch");
}

extern "C" __attribute__((visibility("default"))) int64_t abft_fused_lhs_batch_bytes(int32_t n_border,
                                                                                     int32_t n_window) {
  return (int64_t)sizeof(FusedBatchHeader) + (int64_t)n_border * (int64_t)sizeof(BorderEntry) +
         (int64_t)n_window * (int64_t)sizeof(WindowEntry);
}

extern "C" __attribute__((visibility("default"))) int abft_fused_lhs_batch_prepare(
    const abft_border_task_t* bt, int32_t nb, const abft_window_task_t* wt, int32_t nw, void* table,
    int64_t table_bytes, int32_t* grids) {
  if (nb < 0 || nw < 0 || (nb > 0 && bt == nullptr) || (nw > 0 && wt == nullptr) || table == nullptr ||
      grids == nullptr || (reinterpret_cast<uintptr_t>(table) & 15))
    return fail(ABFT_E_VALUE, "fused_lhs_batch: bad arguments (16-byte aligned device table)");
  if (table_bytes < abft_fused_lhs_batch_bytes(nb, nw)) return fail(ABFT_E_SHAPE, "fused_lhs_batch: table too small");
  std::vector<uint8_t> host((size_t)abft_fused_lhs_batch_bytes(nb, nw), 0);
  auto* hdr = reinterpret_cast<FusedBatchHeader*>(host.data());
  auto* be = reinterpret_cast<BorderEntry*>(hdr + 1);
  auto* we = reinterpret_cast<WindowEntry*>(be + nb);
  int blocks = 0;
  for (int i = 0; i < nb; ++i) {
    const abft_border_task_t& t = bt[i];
    if (t.n < 1 || t.h < 1 || t.w < 1 || t.c < 8 || t.c % 8 || t.c > 1024 || t.ldx < t.c || t.ldx % 8 ||
        t.wsum == nullptr || t.x == nullptr || t.ws_ld < t.c || t.ws_ld % 4 || (reinterpret_cast<uintptr_t>(t.wsum) & 15))
      return fail(ABFT_E_SHAPE, "fused_lhs_batch: bad border task " + std::to_string(i));
    BorderEntry& e = be[i];
    e.x = t.x; e.ws = t.wsum; e.ldx = t.ldx; e.n = t.n; e.h = t.h; e.w = t.w; e.c = t.c; e.ws_ld = t.ws_ld;
    e.ipc = border_imgs_per_cta(t.n, t.h, t.w, t.c);
    e.groups = (t.n + e.ipc - 1) / e.ipc;
    e.begin = blocks;
    blocks += 8 * e.groups;
  }
  hdr->nb = nb; hdr->border_blocks = blocks;
  int wblocks = 0;
  for (int i = 0; i < nw; ++i) {
    const abft_window_task_t& t = wt[i];
    if (t.wsum == nullptr || t.rowck == nullptr || t.lhs == nullptr || !((t.R == 1 && t.S == 1) || (t.R == 3 && t.S == 3)) ||
        t.C < 1 || t.ws_ld < t.C || t.ck < t.C || t.M < 0 || (t.bias != nullptr && t.n_out < 1))
      return fail(ABFT_E_SHAPE, "fused_lhs_batch: bad window task " + std::to_string(i));
    WindowEntry& e = we[i];
    e.ws = t.wsum; e.rowck = t.rowck; e.bias = t.bias; e.lhs = t.lhs; e.M = t.M; e.ld = t.ws_ld; e.C = t.C;
    e.R = t.R; e.S = t.S; e.ck = t.ck; e.n_out = t.n_out;
    e.nblk = std::max(1, std::min(64, (t.R * t.S * t.C + 255) / 256));
    e.begin = wblocks;
    wblocks += e.nblk;
  }
  hdr->nw = nw; hdr->window_blocks = wblocks;
  grids[0] = blocks; grids[1] = wblocks;
  return cuda_check(cudaMemcpy(table, host.data(), host.size(), cudaMemcpyHostToDevice), "fused_lhs_batch table copy");
}

extern "C" __attribute__((visibility("default"))) int abft_fused_lhs_batch_launch(const void* table,
                                                                                  const int32_t* grids,
                                                                                  int32_t dtype, void* stream) {
  if (table == nullptr || grids == nullptr) return fail(ABFT_E_VALUE, "fused_lhs_batch: null table");
  cudaStream_t st = as_stream(stream);
  const auto* hdr = reinterpret_cast<const FusedBatchHeader*>(table);
  if (grids[0] > 0) {
    if (dtype == ABFT_BF16) border_batch_kernel<__nv_bfloat16><<<grids[0], 256, 0, st>>>(hdr);
    else border_batch_kernel<__half><<<grids[0], 256, 0, st>>>(hdr);
    int rc = cuda_check(cudaGetLastError(), "border batch launch");
    if (rc != ABFT_OK) return rc;
  }
  if (grids[1] > 0) {
    window_batch_kernel<<<grids[1], 256, 0, st>>>(hdr);
    return cuda_check(cudaGetLastError(), "window batch launch");
  }
  return ABFT_OK;
}

extern "C" __attribute__((visibility("default"))) int abft_sum_partials(const double* partials, int32_t cap,
                                                                       int32_t ntasks, double* sums, void* stream) {
  if (ntasks < 1 || cap < 1) return fail(ABFT_E_SHAPE, "sum_partials: ntasks and cap must be >= 1");
  sum_partials_kernel<<<(ntasks + 3) / 4, 128, 0, as_stream(stream)>>>(partials, cap, ntasks, sums);
  return cuda_check(cudaGetLastError(), "sum_partials launch");
}
