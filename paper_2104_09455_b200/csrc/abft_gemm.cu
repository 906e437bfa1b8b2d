// abft_gemm.cu — the protected linear layer on sm_100a.
//
// One persistent, warp-specialised tcgen05 GEMM whose epilogue carries every ABFT
// scheme of the reference (tiled.py:400-503):
//
//   warp 0      TMA producer: A [128 x 64] and B^T [BN x 64] tiles (SW128) -> smem ring
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2-5   epilogue: TMEM -> registers; fault injection; thread-level checks;
//               output summation (global); ReLU / rounding / store; fused next-layer
//               activation checksum
//   warps 6-9   checksum generator (thread-level schemes only): per k-block it sums
//               each group of Nt rows of the B^T tile on CUDA cores and writes the
//               group-checksum rows into the smem ring, so one extra tcgen05.mma
//               N-slice computes At * rowck(Bt) for every (row, column-group) pair
//               (tiled.py:221-242) — no extra HBM traffic.
//
// Fault model: delta added to the fp32 accumulator before any checksum, ReLU or
// store (tiled.py:197-200, :291-293); the checksum / shadow side stays clean.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cfloat>
#include <cstdio>
#include <map>
#include <mutex>
#include <tuple>

#include "abft_common.cuh"
#include "sm100_ptx.cuh"

namespace abft {

constexpr int BM = 128;            // UMMA M (one TMEM lane per output row)
constexpr int BK = 64;             // 64 fp16 = 128 B = one SW128 row
constexpr int NUM_THREADS = 320;   // 10 warps
constexpr int EPI_WARP0 = 2;
constexpr int CK_WARP0 = 6;
constexpr int COLCK_SMEM_MAX = 4096;

struct GemmParams {
  int M, N, K, m_ext, n_ext, tol_k;
  int bm_eff, bn_eff, mt, nt, groups, nck, nck_pad;
  int num_m_blocks, num_n_blocks, num_tiles, nkb;
  int stages, acc_stages, cols_per_acc, shadow_off, tmem_cols;
  int scheme, out_dtype, relu, split;
  double r;
  uint32_t off_b, off_ck, off_rec, off_colck, off_bar;
  uint32_t stage_a_bytes, stage_b_bytes, stage_ck_bytes;
  int rec_stride;
  void* C;
  long long ldc;
  const abft_fault_t* faults;
  int nfaults;
  double* out_sum;
  float* next_colck;
  int colck_in_smem;
  abft_thread_verdict_t* verdicts;
  int n_trows, n_tcols;
  int* fired_count;
  int* fired;
  int fired_cap;
  uint32_t idesc_main, idesc_ck;
};

template <typename T>
struct ElemTraits;
template <>
struct ElemTraits<__half> {
  static __device__ __forceinline__ float to_f(__half x) { return __half2float(x); }
  static __device__ __forceinline__ __half from_f(float x) { return __float2half_rn(x); }
  static __device__ __forceinline__ float2 unpack2(uint32_t u) {
    __half2 h = *reinterpret_cast<__half2*>(&u);
    return __half22float2(h);
  }
  static __device__ __forceinline__ uint32_t pack2(float a, float b) {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
};
template <>
struct ElemTraits<__nv_bfloat16> {
  static __device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
  static __device__ __forceinline__ __nv_bfloat16 from_f(float x) { return __float2bfloat16_rn(x); }
  static __device__ __forceinline__ float2 unpack2(uint32_t u) {
    __nv_bfloat162 h = *reinterpret_cast<__nv_bfloat162*>(&u);
    return __bfloat1622float2(h);
  }
  static __device__ __forceinline__ uint32_t pack2(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
};

__device__ __forceinline__ float round_out(float y, int out_dtype) {
  if (out_dtype == ABFT_OUT_F16) return __half2float(__float2half_rn(y));
  if (out_dtype == ABFT_OUT_BF16) return __bfloat162float(__float2bfloat16_rn(y));
  return y;
}

__device__ __forceinline__ bool scheme_has_ck(int s) { return s == ABFT_ONE_SIDED || s == ABFT_TWO_SIDED; }
__device__ __forceinline__ bool scheme_has_shadow(int s) { return s == ABFT_REPL_FULL || s == ABFT_REPL_SINGLE; }
__device__ __forceinline__ bool scheme_thread_level(int s) { return s >= ABFT_ONE_SIDED; }

// Butterfly transpose-reduction: on return lane l holds sum over the warp of v[l].
__device__ __forceinline__ float warp_column_sums(float (&v)[32], int lane) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
#pragma unroll
    for (int i = 0; i < s; ++i) {
      const bool upper = (lane & s) != 0;
      float send = upper ? v[i] : v[i + s];
      float keep = upper ? v[i + s] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  return v[0];
}

template <typename T, int BN>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    abft_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ GemmParams p) {
  using TR = ElemTraits<T>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = ptx::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);

  uint8_t* sm_a = smem;
  uint8_t* sm_b = smem + p.off_b;
  uint8_t* sm_ck = smem + p.off_ck;
  float2* rec = reinterpret_cast<float2*>(smem + p.off_rec);
  float* colck_s = reinterpret_cast<float*>(smem + p.off_colck);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.off_bar);
  uint64_t* full = bars;
  uint64_t* ckfull = bars + p.stages;
  uint64_t* empty = bars + 2 * p.stages;
  uint64_t* tfull = bars + 3 * p.stages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);
  double* red_d = reinterpret_cast<double*>(tmem_holder + 4);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const bool has_ck = scheme_has_ck(p.scheme);
  const bool has_shadow = scheme_has_shadow(p.scheme);
  const bool thread_level = scheme_thread_level(p.scheme);

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&ckfull[s], 128);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 128);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(&tmA);
    ptx::tma_prefetch(&tmB);
  }
  if (warp == 1) ptx::tmem_alloc(tmem_holder, (uint32_t)p.tmem_cols);
  if (warp >= CK_WARP0 && has_ck) {
    // zero the padding checksum rows [nck, nck_pad) of every stage once
    const int ct = threadIdx.x - CK_WARP0 * 32;
    const int pad_rows = p.nck_pad - p.nck;
    for (int s = 0; s < p.stages; ++s) {
      uint4* base = reinterpret_cast<uint4*>(sm_ck + s * p.stage_ck_bytes + p.nck * 128);
      for (int i = ct; i < pad_rows * 8; i += 128) base[i] = make_uint4(0, 0, 0, 0);
    }
    ptx::fence_proxy_async_smem();
  }
  if (warp >= EPI_WARP0 && warp < CK_WARP0 && p.colck_in_smem) {
    for (int i = threadIdx.x - EPI_WARP0 * 32; i < p.N; i += 128) colck_s[i] = 0.f;
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      const uint32_t tx = p.stage_a_bytes + p.stage_b_bytes;
      for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
        const int m0 = (tile / p.num_n_blocks) * p.bm_eff;
        const int n0 = (tile % p.num_n_blocks) * p.bn_eff;
        for (int kb = 0; kb < p.nkb; ++kb) {
          ptx::mbar_wait(&empty[s], ph ^ 1);
          ptx::mbar_arrive_expect_tx(&full[s], tx);
          ptx::tma_load_2d(sm_a + s * p.stage_a_bytes, &tmA, &full[s], kb * BK, m0);
          ptx::tma_load_2d(sm_b + s * p.stage_b_bytes, &tmB, &full[s], kb * BK, n0);
          if (++s == p.stages) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      int t_local = 0;
      for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x, ++t_local) {
        const int acc = t_local % p.acc_stages;
        const uint32_t aph = (uint32_t)(t_local / p.acc_stages) & 1u;
        ptx::mbar_wait(&tempty[acc], aph ^ 1);
        ptx::tc_fence_after();
        const uint32_t d = tmem_base + (uint32_t)(acc * p.cols_per_acc);
        for (int kb = 0; kb < p.nkb; ++kb) {
          ptx::mbar_wait(&full[s], ph);
          if (has_ck) ptx::mbar_wait(&ckfull[s], ph);
          ptx::tc_fence_after();
          const uint32_t a_addr = ptx::smem_u32(sm_a + s * p.stage_a_bytes);
          const uint32_t b_addr = ptx::smem_u32(sm_b + s * p.stage_b_bytes);
          const uint32_t c_addr = ptx::smem_u32(sm_ck + s * p.stage_ck_bytes);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t adesc = ptx::desc_kmajor_sw128(a_addr + k * 32);
            const uint64_t bdesc = ptx::desc_kmajor_sw128(b_addr + k * 32);
            const uint32_t accum = (kb | k) != 0;
            ptx::mma_f16_ss(d, adesc, bdesc, p.idesc_main, accum);
            if (has_ck) ptx::mma_f16_ss(d + BN, adesc, ptx::desc_kmajor_sw128(c_addr + k * 32), p.idesc_ck, accum);
            if (has_shadow) ptx::mma_f16_ss(d + p.shadow_off, adesc, bdesc, p.idesc_main, accum);
          }
          ptx::mma_commit(&empty[s]);
          if (++s == p.stages) { s = 0; ph ^= 1; }
        }
        ptx::mma_commit(&tfull[acc]);
      }
    }
  } else if (warp >= CK_WARP0) {
    // ----------------------------------------------- checksum-row generator
    if (has_ck) {
      const int ct = threadIdx.x - CK_WARP0 * 32;
      const int items = p.groups * 8;
      int s = 0;
      uint32_t ph = 0;
      for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
        for (int kb = 0; kb < p.nkb; ++kb) {
          ptx::mbar_wait(&full[s], ph);
          const uint8_t* bt = sm_b + s * p.stage_b_bytes;
          uint8_t* ck = sm_ck + s * p.stage_ck_bytes;
          for (int it = ct; it < items; it += 128) {
            const int g = it >> 3, c = it & 7;
            float acc[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[e] = 0.f;
            const int r0 = g * p.nt;
            for (int r = 0; r < p.nt; ++r) {
              const int n = r0 + r;
              const uint4 raw = *reinterpret_cast<const uint4*>(bt + n * 128 + ((c ^ (n & 7)) << 4));
              const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 f = TR::unpack2(w[e]);
                acc[2 * e] += f.x;
                acc[2 * e + 1] += f.y;
              }
            }
            uint32_t hi[4], lo[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              hi[e] = TR::pack2(acc[2 * e], acc[2 * e + 1]);
              const float2 h = TR::unpack2(hi[e]);
              lo[e] = TR::pack2(acc[2 * e] - h.x, acc[2 * e + 1] - h.y);
            }
            *reinterpret_cast<uint4*>(ck + g * 128 + ((c ^ (g & 7)) << 4)) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
            if (p.split) {
              const int g2 = p.groups + g;
              *reinterpret_cast<uint4*>(ck + g2 * 128 + ((c ^ (g2 & 7)) << 4)) =
                  make_uint4(lo[0], lo[1], lo[2], lo[3]);
            }
          }
          ptx::fence_proxy_async_smem();
          ptx::mbar_arrive(&ckfull[s]);
          if (++s == p.stages) { s = 0; ph ^= 1; }
        }
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue
    const int et = threadIdx.x - EPI_WARP0 * 32;   // 0..127 (named-barrier rank)
    const int q = warp & 3;                         // TMEM lane quadrant of this warp
    const int row = q * 32 + lane;                  // tile row == TMEM lane
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    const int rs = p.rec_stride;
    double rhs_acc = 0.0;
    int col_lo = 0x7fffffff, col_hi = -1;
    int t_local = 0;
    for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x, ++t_local) {
      const int acc = t_local % p.acc_stages;
      const uint32_t aph = (uint32_t)(t_local / p.acc_stages) & 1u;
      const int m0 = (tile / p.num_n_blocks) * p.bm_eff;
      const int n0 = (tile % p.num_n_blocks) * p.bn_eff;
      const int gm = m0 + row;
      const bool row_in_tile = row < p.bm_eff;
      const bool row_store = row_in_tile && gm < p.M;
      bool row_fault = false;
      if (row_in_tile)
        for (int f = 0; f < p.nfaults; ++f) row_fault |= (p.faults[f].row == gm);
      col_lo = min(col_lo, n0);
      col_hi = max(col_hi, min(n0 + p.bn_eff, p.N));

      ptx::mbar_wait(&tfull[acc], aph);
      ptx::tc_fence_after();
      const uint32_t tacc = tmem_base + lane_addr + (uint32_t)(acc * p.cols_per_acc);

      if (has_ck) {
        // checksum column per (row, group): hi (+ lo) TMEM columns -> rec[row][g].x
        for (int c0 = 0; c0 < p.groups; c0 += 32) {
          float hi[32], lo[32];
          __syncwarp();
          ptx::tmem_ld32(tacc + BN + c0, hi);
          if (p.split) ptx::tmem_ld32(tacc + BN + p.groups + c0, lo);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            if (c0 + j < p.groups) rec[row * rs + c0 + j].x = p.split ? hi[j] + lo[j] : hi[j];
          }
        }
      }

      float gsum = 0.f, ssum = 0.f, best_c = 0.f, best_s = 0.f;
      double best_key = -DBL_MAX;
      int cnt = 0, g = 0;
      float tsum = 0.f;
      for (int c0 = 0; c0 < p.bn_eff; c0 += 32) {
        float v[32], sh[32];
        __syncwarp();
        ptx::tmem_ld32(tacc + c0, v);
        if (has_shadow) ptx::tmem_ld32(tacc + p.shadow_off + c0, sh);
        ptx::tmem_ld_wait();
        const int gc0 = n0 + c0;
        if (row_fault) {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            for (int f = 0; f < p.nfaults; ++f)
              if (p.faults[f].row == gm && p.faults[f].col == gc0 + j && c0 + j < p.bn_eff) v[j] += p.faults[f].delta;
        }
        if (thread_level) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            if (c0 + j < p.bn_eff) {
              const float x = v[j];
              gsum += x;
              if (p.scheme == ABFT_REPL_FULL) {
                const double dx = x, ds = sh[j];
                const double key = fabs(dx - ds) - tolerance(p.r, p.tol_k, ds, dx);
                if (key > best_key) { best_key = key; best_c = x; best_s = sh[j]; }
              } else if (p.scheme == ABFT_REPL_SINGLE) {
                ssum += sh[j];
              }
              if (++cnt == p.nt) {
                float2& rr = rec[row * rs + g];
                if (p.scheme == ABFT_REPL_FULL) rr = make_float2(best_s, best_c);
                else if (p.scheme == ABFT_REPL_SINGLE) rr = make_float2(ssum, gsum);
                else rr.y = gsum;
                gsum = 0.f; ssum = 0.f; best_key = -DBL_MAX; cnt = 0; ++g;
              }
            }
          }
        }
        if (p.out_sum != nullptr) {
#pragma unroll
          for (int j = 0; j < 32; ++j) tsum += (c0 + j < p.bn_eff) ? v[j] : 0.f;
        }
        if (p.out_dtype != ABFT_OUT_NONE || p.next_colck != nullptr) {
          // ReLU + rounding to the storage grid (checksum.py:235 storage_array(activation(c)))
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            float y = p.relu ? fmaxf(v[j], 0.f) : v[j];
            v[j] = round_out(y, p.out_dtype);
          }
          const bool full_chunk = (c0 + 32 <= p.bn_eff) && (gc0 + 32 <= p.N);
          if (row_store && p.out_dtype != ABFT_OUT_NONE) {
            if (p.out_dtype == ABFT_OUT_F32) {
              float* dst = reinterpret_cast<float*>(p.C) + (long long)gm * p.ldc + gc0;
              if (full_chunk && (p.ldc % 4 == 0) && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
                for (int j = 0; j < 32; j += 4)
                  *reinterpret_cast<float4*>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
              } else {
#pragma unroll
                for (int j = 0; j < 32; ++j)
                  if (c0 + j < p.bn_eff && gc0 + j < p.N) dst[j] = v[j];
              }
            } else {
              T* dst = reinterpret_cast<T*>(p.C) + (long long)gm * p.ldc + gc0;
              if (full_chunk && (p.ldc % 8 == 0) && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
                for (int j = 0; j < 32; j += 8) {
                  uint4 u;
                  u.x = TR::pack2(v[j], v[j + 1]);
                  u.y = TR::pack2(v[j + 2], v[j + 3]);
                  u.z = TR::pack2(v[j + 4], v[j + 5]);
                  u.w = TR::pack2(v[j + 6], v[j + 7]);
                  *reinterpret_cast<uint4*>(dst + j) = u;
                }
              } else {
#pragma unroll
                for (int j = 0; j < 32; ++j)
                  if (c0 + j < p.bn_eff && gc0 + j < p.N) dst[j] = TR::from_f(v[j]);
              }
            }
          }
          if (p.next_colck != nullptr) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = (row_store && c0 + j < p.bn_eff && gc0 + j < p.N) ? v[j] : 0.f;
            const float colsum = warp_column_sums(v, lane);
            if (c0 + lane < p.bn_eff && gc0 + lane < p.N && colsum != 0.f) {
              if (p.colck_in_smem) atomicAdd(&colck_s[gc0 + lane], colsum);
              else atomicAdd(&p.next_colck[gc0 + lane], colsum);
            }
          }
        }
      }
      // TMEM accumulator stage fully read: hand it back to the MMA issuer
      ptx::tc_fence_before();
      ptx::mbar_arrive(&tempty[acc]);
      if (row_in_tile) rhs_acc += (double)tsum;

      if (thread_level) {
        ptx::named_bar_sync(1, 128);
        const int tr_count = p.bm_eff / p.mt;
        const int pairs = tr_count * p.groups;
        const bool vector_rule = (p.scheme == ABFT_ONE_SIDED || p.scheme == ABFT_REPL_FULL);
        for (int pi = et; pi < pairs; pi += 128) {
          const int tr = pi / p.groups, gg = pi % p.groups;
          const int t_row = m0 / p.mt + tr, t_col = n0 / p.nt + gg;
          if (t_row >= p.n_trows || t_col >= p.n_tcols) continue;
          double out_diff, out_tol;
          bool fired = false;
          if (vector_rule) {
            double bk = -DBL_MAX;
            out_diff = 0.0; out_tol = 0.0;
            for (int i = tr * p.mt; i < tr * p.mt + p.mt; ++i) {
              const float2 rr = rec[i * rs + gg];
              const double lhs = rr.x, rhs = rr.y;
              const double diff = fabs(lhs - rhs);
              const double tol = tolerance(p.r, p.tol_k, lhs, rhs);
              fired |= diff > tol;
              if (diff - tol > bk) { bk = diff - tol; out_diff = diff; out_tol = tol; }
            }
          } else {
            double lhs = 0.0, rhs = 0.0;
            for (int i = tr * p.mt; i < tr * p.mt + p.mt; ++i) {
              const float2 rr = rec[i * rs + gg];
              lhs += rr.x; rhs += rr.y;
            }
            out_diff = fabs(lhs - rhs);
            out_tol = tolerance(p.r, p.tol_k, lhs, rhs);
            fired = out_diff > out_tol;
          }
          if (p.verdicts != nullptr) {
            abft_thread_verdict_t vv;
            vv.t_row = t_row; vv.t_col = t_col; vv.detected = fired ? 1 : 0; vv.pad = 0;
            vv.max_abs_diff = out_diff; vv.tol = out_tol;
            p.verdicts[(long long)t_row * p.n_tcols + t_col] = vv;
          }
          if (fired && p.fired_count != nullptr) {
            const int slot = atomicAdd(p.fired_count, 1);
            if (p.fired != nullptr && slot < p.fired_cap) {
              p.fired[2 * slot] = t_row;
              p.fired[2 * slot + 1] = t_col;
            }
          }
        }
        ptx::named_bar_sync(1, 128);
      }
    }
    // -------- per-CTA flush of the global-ABFT output summation and fused colck
    if (p.out_sum != nullptr) {
      double x = rhs_acc;
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (lane == 0) red_d[et >> 5] = x;
      ptx::named_bar_sync(1, 128);
      if (et == 0) atomicAdd(p.out_sum, red_d[0] + red_d[1] + red_d[2] + red_d[3]);
    }
    if (p.next_colck != nullptr && p.colck_in_smem) {
      ptx::named_bar_sync(1, 128);
      for (int i = col_lo + et; i < col_hi; i += 128) {
        const float x = colck_s[i];
        if (x != 0.f) atomicAdd(&p.next_colck[i], x);
      }
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  __syncwarp();
  if (warp == 1) ptx::tmem_dealloc(tmem_base, (uint32_t)p.tmem_cols);
}

// ============================================================== host side
namespace {

PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

// K-major 2-D map: dims {K, rows}, row pitch `ld` elements, box {64, box_rows}, SW128.
int make_map(CUtensorMap* map, const void* base, int dtype, int64_t k, int64_t rows, int64_t ld, int box_rows) {
  auto enc = get_encode_fn();
  if (!enc) return fail(ABFT_E_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
  cuuint64_t dims[2] = {(cuuint64_t)k, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, dtype == ABFT_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2,
                   const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(ABFT_E_CUDA, "cuTensorMapEncodeTiled failed with CUresult " + std::to_string((int)r));
  return ABFT_OK;
}

struct MapKey {
  const void* base;
  int dtype;
  int64_t k, rows, ld;
  int box;
  bool operator<(const MapKey& o) const {
    return std::tie(base, dtype, k, rows, ld, box) < std::tie(o.base, o.dtype, o.k, o.rows, o.ld, o.box);
  }
};

int cached_map(CUtensorMap* out, const void* base, int dtype, int64_t k, int64_t rows, int64_t ld, int box_rows) {
  static std::mutex mu;
  static std::map<MapKey, CUtensorMap> cache;
  MapKey key{base, dtype, k, rows, ld, box_rows};
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) { *out = it->second; return ABFT_OK; }
  }
  int rc = make_map(out, base, dtype, k, rows, ld, box_rows);
  if (rc != ABFT_OK) return rc;
  std::lock_guard<std::mutex> g(mu);
  if (cache.size() > 4096) cache.clear();
  cache[key] = *out;
  return ABFT_OK;
}

template <typename T, int BN>
int launch_bn(const CUtensorMap& ma, const CUtensorMap& mb, const GemmParams& p, size_t smem, int grid,
              cudaStream_t st) {
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(abft_gemm_kernel<T, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    max_smem_optin());
  });
  if (attr_err != cudaSuccess) return cuda_check(attr_err, "cudaFuncSetAttribute(abft_gemm_kernel)");
  abft_gemm_kernel<T, BN><<<grid, NUM_THREADS, smem, st>>>(ma, mb, p);
  return cuda_check(cudaGetLastError(), "abft_gemm_kernel launch");
}

template <typename T>
int launch_typed(int bn, const CUtensorMap& ma, const CUtensorMap& mb, const GemmParams& p, size_t smem, int grid,
                 cudaStream_t st) {
  switch (bn) {
    case 32: return launch_bn<T, 32>(ma, mb, p, smem, grid, st);
    case 64: return launch_bn<T, 64>(ma, mb, p, smem, grid, st);
    case 128: return launch_bn<T, 128>(ma, mb, p, smem, grid, st);
    case 256: return launch_bn<T, 256>(ma, mb, p, smem, grid, st);
  }
  return fail(ABFT_E_VALUE, "unsupported tile_n");
}

int ceil_div(int a, int b) { return (a + b - 1) / b; }
int round_up(int a, int b) { return ceil_div(a, b) * b; }
uint32_t pow2_at_least(uint32_t x) {
  uint32_t r = 32;
  while (r < x) r <<= 1;
  return r;
}

}  // namespace
}  // namespace abft

using namespace abft;

extern "C" __attribute__((visibility("default"))) int abft_gemm(const abft_gemm_args_t* a, void* stream) {
  if (a == nullptr) return fail(ABFT_E_VALUE, "null args");
  if (a->M < 1 || a->N < 1 || a->K < 1) return fail(ABFT_E_SHAPE, "GEMM extents must be >= 1");
  if (a->dtype != ABFT_F16 && a->dtype != ABFT_BF16) return fail(ABFT_E_VALUE, "dtype must be ABFT_F16 or ABFT_BF16");
  if (a->scheme < ABFT_UNPROTECTED || a->scheme > ABFT_REPL_SINGLE) return fail(ABFT_E_VALUE, "unknown scheme");
  if (a->lda < a->K || a->ldbt < a->K || (a->lda % 8) || (a->ldbt % 8))
    return fail(ABFT_E_SHAPE, "lda/ldbt must be >= K and multiples of 8 (16-byte TMA row pitch)");
  if ((reinterpret_cast<uintptr_t>(a->A) & 15) || (reinterpret_cast<uintptr_t>(a->Bt) & 15))
    return fail(ABFT_E_VALUE, "A and Bt must be 16-byte aligned");
  if (a->out_dtype != ABFT_OUT_NONE && (a->C == nullptr || a->ldc < a->N))
    return fail(ABFT_E_SHAPE, "C must be non-null with ldc >= N");
  const bool thread_level = a->scheme >= ABFT_ONE_SIDED;
  const bool has_ck = a->scheme == ABFT_ONE_SIDED || a->scheme == ABFT_TWO_SIDED;
  const bool has_shadow = a->scheme == ABFT_REPL_FULL || a->scheme == ABFT_REPL_SINGLE;
  int mt = thread_level ? a->thread_m : 1, nt = thread_level ? a->thread_n : 1;
  int m_ext = thread_level ? a->m_ext : a->M, n_ext = thread_level ? a->n_ext : a->N;
  if (thread_level) {
    if (mt < 1 || nt < 1 || mt > BM || nt > 256) return fail(ABFT_E_UNSUPPORTED, "thread tile must be <= 128 x 256");
    if (m_ext < a->M || n_ext < a->N || m_ext % mt || n_ext % nt)
      return fail(ABFT_E_SHAPE, "m_ext/n_ext must cover M/N and be multiples of the thread tile");
  }
  if (a->scheme == ABFT_GLOBAL && a->out_sum == nullptr) return fail(ABFT_E_VALUE, "global scheme needs out_sum");

  const int sms = a->num_sms > 0 ? a->num_sms : num_sms();
  // ---- CTA N tile
  int bn = a->tile_n;
  if (bn == 0) {
    // largest tile that still gives >= one tile per SM; otherwise the smallest
    // efficient one (max parallelism for bandwidth-bound layers).  Thread-level
    // schemes keep <= 32 checksum groups per tile (epilogue record budget).
    const int cap = thread_level ? std::min(256, 32 * nt) : 256;
    const int m_blocks = ceil_div(m_ext, (BM / mt) * mt);
    int smallest = 0;
    bn = 0;
    for (int cand : {256, 128, 64, 32}) {
      if (cand > cap || cand < nt) continue;
      if (cand > 32 && cand / 2 >= round_up(n_ext, 32)) continue;     // > 2x wider than needed
      if (cand == 32 && n_ext > 32 && cap >= 64 && nt <= 64) continue;  // 64 is the narrowest efficient tile
      const int eff = (cand / nt) * nt;
      if (bn == 0 && (long long)m_blocks * ceil_div(n_ext, eff) >= sms) bn = cand;
      smallest = cand;
    }
    if (bn == 0) bn = smallest;
    if (bn == 0) return fail(ABFT_E_UNSUPPORTED, "no CTA tile fits this thread tile");
  }
  if (bn != 32 && bn != 64 && bn != 128 && bn != 256) return fail(ABFT_E_VALUE, "tile_n must be 32/64/128/256");
  if (bn < nt) return fail(ABFT_E_UNSUPPORTED, "thread_n larger than the CTA tile");

  GemmParams p{};
  p.M = a->M; p.N = a->N; p.K = a->K; p.m_ext = m_ext; p.n_ext = n_ext; p.tol_k = a->tol_k > 0 ? a->tol_k : a->K;
  p.mt = mt; p.nt = nt;
  p.bm_eff = (BM / mt) * mt;
  p.bn_eff = (bn / nt) * nt;
  p.groups = thread_level ? p.bn_eff / nt : 0;
  if (thread_level && p.groups > 32) return fail(ABFT_E_UNSUPPORTED, "more than 32 checksum groups per CTA tile");
  p.split = (has_ck && a->ck_split) ? 1 : 0;
  p.nck = has_ck ? p.groups * (p.split ? 2 : 1) : 0;
  p.nck_pad = has_ck ? round_up(p.nck, 16) : 0;
  p.num_m_blocks = ceil_div(m_ext, p.bm_eff);
  p.num_n_blocks = ceil_div(n_ext, p.bn_eff);
  p.num_tiles = p.num_m_blocks * p.num_n_blocks;
  p.nkb = ceil_div(a->K, BK);
  p.cols_per_acc = bn + p.nck_pad + (has_shadow ? bn : 0);
  p.shadow_off = bn + p.nck_pad;
  p.acc_stages = (2 * p.cols_per_acc <= 512) ? 2 : 1;
  if (p.cols_per_acc > 512) return fail(ABFT_E_UNSUPPORTED, "TMEM budget exceeded");
  p.tmem_cols = (int)pow2_at_least((uint32_t)(p.acc_stages * p.cols_per_acc));
  p.scheme = a->scheme; p.out_dtype = a->out_dtype; p.relu = a->relu;
  p.r = tol_ratio(a->numeric);
  p.C = a->C; p.ldc = a->ldc;
  p.faults = a->faults; p.nfaults = a->faults ? a->nfaults : 0;
  p.out_sum = a->out_sum;
  p.next_colck = a->next_colck;
  p.colck_in_smem = (a->next_colck != nullptr && a->N <= COLCK_SMEM_MAX) ? 1 : 0;
  p.verdicts = a->verdicts;
  p.n_trows = m_ext / mt; p.n_tcols = n_ext / nt;
  p.fired_count = a->fired_count; p.fired = a->fired; p.fired_cap = a->fired_cap;
  const uint32_t fmt = a->dtype == ABFT_BF16 ? 1u : 0u;
  p.idesc_main = ptx::idesc_f16(fmt, BM, bn);
  p.idesc_ck = has_ck ? ptx::idesc_f16(fmt, BM, p.nck_pad) : 0u;

  // ---- shared memory carve-up (all tile buffers 1024-aligned)
  p.stage_a_bytes = BM * BK * 2;
  p.stage_b_bytes = bn * BK * 2;
  p.stage_ck_bytes = (uint32_t)round_up(p.nck_pad * BK * 2, 1024);
  p.rec_stride = thread_level ? (p.groups | 1) : 0;
  const uint32_t rec_bytes = thread_level ? (uint32_t)round_up(BM * p.rec_stride * 8, 1024) : 0;
  const uint32_t colck_bytes = p.colck_in_smem ? (uint32_t)round_up(a->N * 4, 1024) : 0;
  const uint32_t bar_bytes = 1024;
  const uint32_t stage_bytes = p.stage_a_bytes + p.stage_b_bytes + p.stage_ck_bytes;
  const int budget = max_smem_optin() - 1024 /*alignment slack*/ - (int)(rec_bytes + colck_bytes + bar_bytes);
  int stages = budget / (int)stage_bytes;
  if (stages > 8) stages = 8;
  if (stages < 2) return fail(ABFT_E_UNSUPPORTED, "shared memory budget too small for a 2-stage pipeline");
  p.stages = stages;
  p.off_b = stages * p.stage_a_bytes;
  p.off_ck = p.off_b + stages * p.stage_b_bytes;
  p.off_rec = p.off_ck + stages * p.stage_ck_bytes;
  p.off_colck = p.off_rec + rec_bytes;
  p.off_bar = p.off_colck + colck_bytes;
  const size_t smem = (size_t)p.off_bar + bar_bytes + 1024;

  CUtensorMap ma, mb;
  int rc = cached_map(&ma, a->A, a->dtype, a->K, a->M, a->lda, BM);
  if (rc != ABFT_OK) return rc;
  rc = cached_map(&mb, a->Bt, a->dtype, a->K, a->N, a->ldbt, bn);
  if (rc != ABFT_OK) return rc;

  const int grid = std::min(p.num_tiles, sms);
  cudaStream_t st = as_stream(stream);
  if (a->dtype == ABFT_BF16) return launch_typed<__nv_bfloat16>(bn, ma, mb, p, smem, grid, st);
  return launch_typed<__half>(bn, ma, mb, p, smem, grid, st);
}
