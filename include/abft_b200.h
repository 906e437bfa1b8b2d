/*
 * abft_b200.h — C-ABI of the B200-native ABFT-protected linear-layer path.
 *
 * The reference (abft_guard 0.1.0, pure Python) has no FFI; these entry points
 * are what its hot-path functions become when the arithmetic moves to sm_100a.
 * Each declaration cites the reference interface it replaces.  Plain pointers
 * and sizes only; every data pointer is a DEVICE pointer owned by the caller;
 * the library allocates nothing on the hot path.  All calls are asynchronous
 * on `stream` (a cudaStream_t passed as void*); results are valid after the
 * stream synchronises — the reference's deferred verification
 * (checksum.py:207-211, :237).
 *
 * Return codes map onto the reference exceptions (errors.py:4-28):
 *   ABFT_OK 0, ABFT_E_SHAPE 1 -> ShapeMismatchError, ABFT_E_VALUE 2 -> ValueError,
 *   ABFT_E_OVERFLOW 3 -> ExactOverflowError, ABFT_E_CUDA 4 (launch/driver error),
 *   ABFT_E_UNSUPPORTED 5 (a configuration the tensor-core path does not cover).
 * The message of the last failure on the calling thread: abft_last_error().
 */
#ifndef ABFT_B200_H
#define ABFT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ABFT_OK = 0, ABFT_E_SHAPE = 1, ABFT_E_VALUE = 2, ABFT_E_OVERFLOW = 3, ABFT_E_CUDA = 4,
       ABFT_E_UNSUPPORTED = 5 };

/* storage element type of A / B (shapes.py:22-57: binary16 storage) */
enum { ABFT_F16 = 0, ABFT_BF16 = 1 };
/* output element type */
enum { ABFT_OUT_F32 = 0, ABFT_OUT_F16 = 1, ABFT_OUT_BF16 = 2, ABFT_OUT_NONE = 3 };
/* comparison rule (checksum.py:143-148): tau = r*K*max(|lhs|,|rhs|,1) with
 * r = 0 (exact-int), 2^-10 (binary16), 2^-23 (binary32), 2^-7 (bf16, B200 extension) */
enum { ABFT_NUM_EXACT = 0, ABFT_NUM_BINARY16 = 1, ABFT_NUM_BINARY32 = 2, ABFT_NUM_BF16 = 3 };
/* tiled.py:42-48 (Scheme) — same order as the reference enum */
enum { ABFT_UNPROTECTED = 0, ABFT_GLOBAL = 1, ABFT_ONE_SIDED = 2, ABFT_TWO_SIDED = 3,
       ABFT_REPL_FULL = 4, ABFT_REPL_SINGLE = 5 };

/* OutputFault / ThreadMmaFault after _fault_cell (tiled.py:92-121, :386-397) */
typedef struct { int32_t row, col; float delta; } abft_fault_t;

/* Verdict (checksum.py:35-43) */
typedef struct { double lhs, rhs, tol; int32_t detected, k; } abft_verdict_t;

/* ThreadVerdict (tiled.py:149-157) */
typedef struct { int32_t t_row, t_col, detected, pad; double max_abs_diff, tol; } abft_thread_verdict_t;

/*
 * One protected GEMM C = A * B (tiled.py:400-503 execute; checksum.py:130 accumulate_matmul).
 *   A  [M x K]  row-major (K-major), element `dtype`, leading dim lda (elements, %8 == 0)
 *   Bt [N x K]  row-major = B^T (K-major weights, as prepared by abft_pack), ldbt %8 == 0
 *   C  [M x N]  row-major, `out_dtype`; ReLU applied before the store when relu != 0
 * Faults add delta to the fp32 accumulator before any checksum, ReLU or store
 * (tiled.py:197-200; checksum.py:232-233).  Thread-level verdicts cover the
 * tiling-padded extents m_ext x n_ext (tiled.py:423-431); tol_k is the K the
 * thread-level tolerance uses (k_step-padded K, tiled.py:242).
 * Global scheme: out_sum[0] += sum of the fp32 outputs (output_summation,
 * checksum.py:120-127) — verification is deferred to abft_verify.
 * next_colck (optional, [N]) += column sums of the STORED, ReLU'd, rounded
 * outputs: the next layer's activation checksum fused into this epilogue
 * (checksum.py:229 + :235).
 */
typedef struct {
  const void* A;  int64_t lda;
  const void* Bt; int64_t ldbt;
  void* C;        int64_t ldc;
  int32_t M, N, K;
  int32_t m_ext, n_ext, tol_k;
  int32_t dtype, out_dtype, numeric, scheme;
  int32_t thread_m, thread_n;
  int32_t relu;
  int32_t ck_split;                     /* 1: checksum columns as hi+lo pairs (near-fp32), 0: single */
  const abft_fault_t* faults; int32_t nfaults;
  double* out_sum;                      /* global: [1] accumulated output summation */
  float* next_colck;                    /* optional [N] */
  abft_thread_verdict_t* verdicts;      /* optional [(m_ext/thread_m) x (n_ext/thread_n)] row-major */
  int32_t* fired_count;                 /* optional: number of thread tiles whose check fired */
  int32_t* fired;                       /* optional [fired_cap x 2] (t_row, t_col) of fired tiles */
  int32_t fired_cap;
  int32_t tile_n;                       /* CTA N tile: 0 = auto, else 32/64/128/192/224/256 */
  int32_t num_sms;                      /* persistent grid size cap: 0 = all SMs */
  /* optional checksum rows prepared offline by abft_ck_rows for THIS call's plan; when null the
   * checksum warps generate them on chip from each B^T tile (one-sided / two-sided only) */
  const void* ck_rows; int64_t ldck; int32_t ck_rows_n;
  /* optional [K] fp32, global scheme: += column sums of A as the kernel stages it (the activation
   * checksum of checksum.py:90-96 / :229 computed from the shared-memory A tiles the MMA consumes,
   * so the global scheme needs no extra pass over A; for a conv this is the windowed im2col sum) */
  float* a_colck;
  /* optional [1] fp64, global scheme: += sum over rows of A . rowck(B-tile), i.e. the lhs
   * colck(A) . rowck(B) of checksum.py:108-117 regrouped as 1^T (A (B 1)): one extra MMA
   * N-slice per tile driven by the offline checksum rows (abft_ck_rows with nt = the plan's
   * bn_eff, split hi/lo, nck_pad = 16) and a row sum in the epilogue.  Needs ck_rows. */
  double* out_lhs;
  /* optional fused deferred verification (checksum.py:207-211, :237): when the launch's last
   * CTA finishes, the verdicts of vn layers are formed from vsums [vn][2] (lhs, rhs) with the
   * tau rule for K = vk[i] and this call's numeric mode, written to vout [vn] and counted into
   * *vdetected.  vdone is a zero-initialised counter the kernel resets for the next launch.
   * A chain passes this on its last layer and needs no separate verification launch. */
  const double* vsums; const int32_t* vk; int32_t vn; int32_t* vdone; abft_verdict_t* vout; int32_t* vdetected;
  /* 1: programmatic dependent launch — the kernel's prologue (barrier init, TMEM allocation,
   * descriptor prefetch) overlaps the previous kernel on the stream; its first operand load
   * waits for that kernel's completion (griddepcontrol.wait).  For chained layers. */
  int32_t pdl;
  /* layout of ck_rows: 0 = separate checksum rows (abft_ck_rows, loaded by their own TMA and
   * multiplied by their own MMA N-slice); 1 = augmented weights (abft_aug_weights): per CTA
   * N-tile the tile's weight rows followed by its checksum rows, so one TMA box and ONE MMA
   * instruction (N = tile + checksum columns) per k-step produce outputs and checksums.
   * With layout 1, ck_rows replaces Bt as the B operand (Bt is still used for shapes). */
  int32_t ck_layout;
  /* optional [ceil(K/64)*64] fp32 (zero past K, 16-byte aligned), global scheme with out_lhs:
   * the row checksum of B (sum over N of Bt[n][k], in Bt's K layout; checksum.py:99-105).  The lhs is then accumulated as
   * sum over rows of A . lhs_rowck by the checksum warps, from the shared-memory A tiles the
   * MMA consumes (each A tile once, in its first N block): no checksum rows in the MMA, so the
   * CTA tile stays as wide as the unprotected one.  ck_rows is not used; excludes a_colck.
   * Works in every A-load mode, the halo conv included. */
  const float* lhs_rowck;
  /* optional [partials_cap][2] fp64, global scheme: instead of adding its (lhs, rhs) partial to
   * out_lhs / out_sum with one atomic per CTA, CTA b writes it to out_partials[b] with plain
   * stores (no contended atomics at the kernel's tail); slots past the launch's grid must hold
   * zeros.  abft_verify_partials sums the slots and applies the tau rule.  partials_cap must be
   * >= the plan's grid (abft_gemm_plan out[7]; the SM count always suffices). */
  double* out_partials; int32_t partials_cap;
  /* optional [N] fp32 (16-byte aligned) per-output-column bias — a BN-folded conv / FC bias, which
   * the reference never models (roofline.py:3-4).  Added to the fp32 accumulator after fault
   * injection and before every checksum, sum, ReLU and store, with the exact checksum corrections
   * (SURVEY H3): the global lhs gains sum_{rows < M} sum_j bias_j (= M * sum(bias)) so that
   * lhs = colck(A) . rowck(B) + M * sum(bias) still equals rhs = sum(C + bias); each one-sided
   * group's checksum column gains sum_{j in group} bias_j.  Thread-level: one-sided with
   * thread_n 8 or 16 only (ABFT_E_UNSUPPORTED otherwise). */
  const float* bias;
  /* optional residual [M x N] in the storage dtype (ld_res elements, a multiple of 8, 16-byte
   * aligned base): added after the checks and before the ReLU and the store — the shortcut of a
   * residual block, outside the checked contraction like the reference's activation (checksum.py:235). */
  const void* residual; int64_t ld_res;
  /* plan hints (0 = the planner's choice): bit 0 = no k-block pairs (one k-block per pipeline stage,
   * deeper pipeline); bit 1 = Bt is zero-padded to >= round_up(N, 256) rows, so the weight map covers
   * whole tiles (no out-of-bounds boxes); bit 2 = two output staging buffers per epilogue warp even
   * when one would buy a pipeline stage; bit 3 = direct 16-byte stores of the output from the
   * epilogue registers instead of shared-memory staging + bulk tensor stores.  The profilers time
   * the alternatives and keep the fastest (T_o = min over plans); bit 4 = the chunk-split epilogue
   * (both warp sets on every tile) for narrow tiles, which otherwise alternate whole tiles; bits 6-8
   * = k-blocks of gathered-stem copies in flight (3..7, 0 = 3); bit 9 = 64-byte-row output stores
   * (32-column boxes) instead of 128-byte rows; bit 10 = the global lhs comes from outside the
   * kernel (see wsum below); bit 11 = (abft_conv2d) per-tap im2col boxes instead of the halo
   * windows for a stride-1 conv (full 128-row tiles, no row-shifted A operands); bit 12 = CTA pairs:
   * 2-CTA clusters on the two SMs of a TPC, one M = 256 tcgen05.mma.cta_group::2 per k-step issued
   * by the leader, each CTA staging its own 128 A rows and half of the B rows (plain-class GEMMs /
   * 64-channel im2col convs: unprotected, global with the checksum slice in the weight tile or the
   * external lhs; ABFT_E_UNSUPPORTED otherwise). */
  int32_t plan_flags;
  /* optional window column sums of THIS layer's stored output (after bias / residual / ReLU /
   * rounding) for the next layer's global lhs (the fused activation checksum):
   * wsum [buckets][ws_ld] fp32, accumulated (the caller zeroes it); ws_mode 1 = one bucket, the
   * column sums (a pointwise / FC consumer); 2 = nine buckets for a 3x3 / stride 1 / pad 1
   * consumer: all rows, output row p == 0, p == P-1, column q == 0, q == Q-1, and the four corners
   * (0,0), (0,Q-1), (P-1,0), (P-1,Q-1), where a row is the output pixel (n*P + p)*Q + q.
   * plan_flags bit 10: the global scheme takes its lhs from outside the kernel (abft_window_lhs
   * adds it to the partial slots), so no checksum slice / dot runs and the bias correction is the
   * caller's. */
  float* wsum; int32_t ws_ld, ws_mode, ws_P, ws_Q;
} abft_gemm_args_t;

int abft_gemm(const abft_gemm_args_t* args, void* stream);

/* Grouped launch: many independent protected GEMMs (same dtype, scheme, thread tile, output type,
 * ReLU and tile_n — one kernel configuration) as ONE persistent launch over all their tiles, e.g.
 * one layer depth of a group of DLRM chains (the ~5 us launch latency, not the math, bounds such
 * small GEMMs).  Per problem: A / B (or augmented weights) / C, M, N, K, out_partials (global) —
 * no faults, bias, residual or fused verification.  prepare() writes the problem table (tensor
 * maps, extents, outputs; count * abft_group_problem_bytes(), 64-byte aligned device memory) once,
 * synchronously; launch() is stream-ordered and graph-capturable.  Outputs, (lhs, rhs) slots and
 * fired-tile counts equal those of launching each problem alone (the slots are added atomically
 * per problem and CTA: the caller zeroes them, as for abft_verify_partials). */
int abft_gemm_group_prepare(const abft_gemm_args_t* args, int32_t count, void* table, int64_t table_bytes);
int abft_gemm_group_launch(const abft_gemm_args_t* args, int32_t count, const void* table, void* stream);
int abft_group_problem_bytes(void);

/* The global lhs of a layer whose activation checksum came from the producer's window sums
 * (abft_gemm_args_t.wsum): lhs += sum_{r,s,c<C} colck_im2col(r,s,c) * rowck[(r*S + s)*ck + c]
 * + M * sum_{j<n_out} bias[j] (bias optional), where colck_im2col is the im2col column sum of the
 * consumer's (R x S, stride 1, "same" padding) input rebuilt from the nine buckets (R = S = 3) or
 * the plain column sums (R = S = 1) — the reference's checksum_dot(colck(A), rowck(B))
 * (checksum.py:108-117) on the lowered GEMM.  fp64 dot, one atomic add into *lhs. */
/* Buckets 1..8 of the window sums (rows on the first / last row and column of each image and the
 * four corners) of an NHWC activation [n][h][w][c] (ldx elements per pixel), from its border
 * pixels; bucket 0 comes from the producer (abft_gemm_args_t.wsum, ws_mode 1). Accumulates. */
int abft_nhwc_border_sums(const void* x, int32_t n, int32_t h, int32_t w, int32_t c, int64_t ldx, int32_t dtype,
                          float* wsum, int32_t ws_ld, void* stream);
int abft_window_lhs(const float* wsum, int32_t ws_ld, int32_t C, int32_t R, int32_t S, int32_t ck,
                    const float* rowck, const float* bias, int32_t n_out, int64_t M, double* lhs, void* stream);

/* The two calls above for a whole forward in two launches: every producer's border buckets, then
 * every fused consumer's window lhs (tasks = the calls' arguments).  _prepare validates the tasks
 * and writes the device table (16-byte aligned, abft_fused_lhs_batch_bytes) synchronously, once;
 * grids[2] (out) = the two launches' CTA counts; _launch is stream-ordered and graph-capturable.
 * The activations must still hold the producers' outputs when the batch runs. */
typedef struct {
  const void* x; float* wsum; int64_t ldx; int32_t n, h, w, c, ws_ld;
} abft_border_task_t;
typedef struct {
  const float* wsum; const float* rowck; const float* bias; double* lhs; int64_t M;
  int32_t ws_ld, C, R, S, ck, n_out;
} abft_window_task_t;
int64_t abft_fused_lhs_batch_bytes(int32_t n_border, int32_t n_window);
int abft_fused_lhs_batch_prepare(const abft_border_task_t* border, int32_t n_border, const abft_window_task_t* window,
                                 int32_t n_window, void* table, int64_t table_bytes, int32_t* grids);
int abft_fused_lhs_batch_launch(const void* table, const int32_t* grids, int32_t dtype, void* stream);

/* The kernel configuration abft_gemm would use for `args` (no launch):
 * out[0] tile_n, [1] bn_eff, [2] checksum groups per tile, [3] nck_pad, [4] pipeline stages,
 * [5] 1 if offline checksum rows are recommended (B tiles re-read by > 2 M-blocks),
 * [6] number of N blocks, [7] persistent grid size, [8] rows per N-block of augmented weights
 * (tile_n + real checksum rows), [9] reserved.  Augmented weights with tile_n = 256 keep their
 * layout; the kernel then reads the checksum rows by a second box into their own MMA N-slice. */
int abft_gemm_plan(const abft_gemm_args_t* args, int32_t* out /*[10]*/);

/* Offline checksum rows for a plan: out [(n_blocks*nck_pad) x ldo] (n_blocks = plan out[6], rows of
 * blocks past N are zero), row nb*nck_pad + j holds
 * the fp16/bf16 hi (j < G) / lo (G <= j < 2G, split) part of sum_{r<nt} Bt[nb*bn_eff + j*nt + r][:]
 * (the weight-tile checksum of tiled.py:240, prepared once per weight like checksum.py:175). */
int abft_ck_rows(const void* Bt, int32_t N, int32_t K, int64_t ldbt, int32_t dtype, int32_t bn_eff, int32_t nt,
                 int32_t split, int32_t nck_pad, int32_t n_blocks, void* out, int64_t ldo, void* stream);

/* Augmented weights for a plan (ck_layout 1): out [(n_blocks * rows) x ldo], rows = plan out[8]
 * = tile_n + G*(split ? 2 : 1) with G = bn_eff / nt; block nb holds Bt rows nb*bn_eff .. +bn_eff
 * (zero past N and past bn_eff), then that block's G hi (and G lo) checksum rows.  The MMA
 * reads nck_pad checksum rows; the padding rows are never stored and their products are ignored. */
int abft_aug_weights(const void* Bt, int32_t N, int32_t K, int64_t ldbt, int32_t dtype, int32_t tile_n, int32_t bn_eff,
                     int32_t nt, int32_t split, int32_t nck_pad, int32_t n_blocks, void* out, int64_t ldo, void* stream);

/*
 * Column sums of a row-major [rows x cols] matrix into out[cols] (fp32).
 *   column_checksum(A)  (checksum.py:90-96):  X = A,   rows = M, cols = K
 *   row_checksum(B)     (checksum.py:99-105):  X = B^T, rows = N, cols = K
 *   offline_weight_checksum (checksum.py:175-187) = the latter, once per weight.
 * accumulate != 0 adds into out (for batch shards / K4a+K4b mixes).
 */
int abft_colsum(const void* X, int32_t rows, int32_t cols, int64_t ldx, int32_t dtype,
                float* out, int32_t accumulate, void* stream);

/*
 * Layout/padding pack (the zero-padded copies of tiled.py:428-431 and the
 * K-major weight layout the tensor-core path consumes):
 *   transpose == 0: dst[r][c] = src[r][c] for r<rows, c<cols; zero for c in [cols, dst_cols)
 *   transpose != 0: dst[c][r] = src[r][c]  (dst is [cols x dst_cols], zero for r in [rows, dst_cols))
 * Element size is 2 bytes (fp16/bf16).
 */
int abft_pack(const void* src, int32_t rows, int32_t cols, int64_t lds,
              void* dst, int32_t dst_cols, int64_t ldd, int32_t transpose, void* stream);

/* Element-type conversion helpers for host adapters: int64 (exact-int mode,
 * values must be exactly representable) or fp32 -> fp16/bf16 storage. */
int abft_convert_i64(const int64_t* src, int64_t n, int32_t dtype, void* dst, void* stream);

/* Sum of all entries of a row-major matrix (output_summation, checksum.py:120-127):
 * *out += sum in fp64; elem 0 = fp16, 1 = bf16, 2 = fp32. */
int abft_matrix_sum(const void* X, int32_t rows, int32_t cols, int64_t ldx, int32_t elem, double* out,
                    void* stream);

/*
 * Batched global-ABFT verification (checksum.py:108-117 checksum_dot, :151-169):
 * for layer i, lhs_i = dot(colck_i, rowck_i) over k_i terms (fp64), rhs_i =
 * *rhs_i, tau = r*k_i*max(|lhs|,|rhs|,1), detected = |lhs-rhs| > tau.
 * `sums` receives [lhs_i, rhs_i] (so multi-GPU callers can all-reduce partials
 * and call abft_verify_sums); `out` receives one Verdict per layer;
 * `detected_count` (optional) += number of flagged layers.
 */
/* k = checksum length; tol_k = the K of the tau rule when it differs (0 = k): the unpadded
 * K of the reference GEMM (tiled.py:471-473), e.g. C*R*S of a conv whose channels were padded */
typedef struct { const float* colck; const float* rowck; const double* rhs; int32_t k, tol_k; } abft_global_task_t;

int abft_global_lhs(const abft_global_task_t* tasks /*device*/, int32_t ntasks, double* sums /*[n][2]*/,
                    void* stream);
int abft_verify_sums(const double* sums /*[n][2]*/, const int32_t* k /*device [n]*/, int32_t ntasks,
                     int32_t numeric, abft_verdict_t* out, int32_t* detected_count, void* stream);
/* The tau rule over per-CTA partial slots: task i's (lhs, rhs) = the sum of its cap slots
 * partials[i][0..cap) (written by abft_gemm with out_partials). */
int abft_verify_partials(const double* partials /*[n][cap][2]*/, int32_t cap, const int32_t* k /*device [n]*/,
                         int32_t ntasks, int32_t numeric, abft_verdict_t* out, int32_t* detected_count, void* stream);
/* Single-GPU fast path: abft_global_lhs + abft_verify_sums fused into one launch. */
int abft_global_verify(const abft_global_task_t* tasks, int32_t ntasks, int32_t numeric, double* sums,
                       abft_verdict_t* out, int32_t* detected_count, void* stream);

/*
 * Implicit-GEMM convolution with the same ABFT epilogues (the reference lowers
 * convs to GEMMs by im2col, shapes.py:156-180 layer_to_gemm: M = n*P*Q, N = OC, K = C*R*S).
 *   gemm.A    the NHWC input [n][h][w][c] (c = physical channels, a multiple of 8; channels
 *             past the model's real C are zero), read through a TMA im2col map — the im2col
 *             matrix is never materialised.  gemm.lda is ignored.
 *   gemm.Bt   packed weights [OC x K], K = r*s*c ordered (r, s, c) (abft_conv_pack_weight)
 *   gemm.M/K  derived (M = n*P*Q, K = r*s*c); pass 0 or the same values
 *   gemm.C    output [M x OC] = NHWC [n][P][Q][OC]
 * All scheme / fault / verdict / fused-checksum fields keep their GEMM meaning with
 * row = output pixel index (n*P + p)*Q + q and col = output channel.
 * 1x1 / stride-1 / pad-0 convs run as the plain GEMM of the NHWC matrix.
 */
typedef struct {
  abft_gemm_args_t gemm;
  int32_t n, h, w, c;
  int32_t r, s, stride_h, stride_w, pad_h, pad_w;
  int32_t c_real;          /* the model's input channels (<= c; 0 = c) */
  void* workspace;         /* explicit-im2col mode only: >= plan out[6] bytes, 16-byte aligned */
  int64_t ws_bytes;
} abft_conv_args_t;

int abft_conv2d(const abft_conv_args_t* args, void* stream);
/* The kernel plan of a conv (no launch):
 *   out[0] A-load mode: 0 = plain GEMM of the NHWC matrix (1x1, stride 1, pad 0);
 *          1 = TMA im2col, 64-channel columns (channels zero-padded to a multiple of 64);
 *          2 = TMA im2col, 8-channel columns;
 *          3 = explicit im2col into the workspace, then the plain GEMM (few input channels,
 *              e.g. network stems, where K = r*s*c_real is packed densely)
 *   out[1] packed-weight channel stride ck, out[2] P, out[3] Q,
 *   out[4] K of the GEMM (r*s*ck, or round8(r*s*c_real) in mode 3), out[5] M = n*P*Q,
 *          5 = gathered A tiles (the checksum warps copy (tap, channel) chunks with cp.async:
 *              <= 4 real channels, or C < 48 a multiple of 8), weights resident in shared memory;
 *   out[6] workspace bytes (mode 3; for mode 5 the size of the explicit im2col the call falls back
 *          to when the gather cannot take it, e.g. weights + window sums past shared memory) */
int abft_conv_plan(const abft_conv_args_t* args, int32_t* out /*[8]*/);
/* The kernel plan abft_conv2d would use for `args` (no launch), laid out as abft_gemm_plan's
 * out[0..8]; out[9] = the A-load mode actually used.  Augmented weights / checksum rows for a
 * conv call are prepared from THIS plan (the conv's A-load mode enters the tile choice). */
int abft_conv_gemm_plan(const abft_conv_args_t* args, int32_t* out /*[10]*/);
/* torch-layout weight [OC][cin][r][s] -> K-major [OC][ldo] with element (r, s, c) at
 * (r*s_ + s)*ck + c, channels >= cin and columns >= r*s*ck zero (ldo >= r*s*ck) */
int abft_conv_pack_weight(const void* w, int32_t oc, int32_t cin, int32_t r, int32_t s, int32_t ck, void* out,
                          int64_t ldo, void* stream);
/* windowed activation checksum of the conv's im2col matrix, out[(ri*s + si)*c + ch]
 * (column_checksum of the lowered A, checksum.py:90-96), fp32; accumulate != 0 adds */
int abft_conv_colck(const void* X, int32_t n, int32_t h, int32_t w, int32_t c, int32_t r, int32_t s,
                    int32_t stride_h, int32_t stride_w, int32_t pad_h, int32_t pad_w, int32_t dtype, float* out,
                    int32_t accumulate, void* stream);

/*
 * Glue of a protected CNN forward (config C5).  The reference protects linear layers only and
 * models a network by its linear-layer list (shapes.py:198-212 model_to_gemm_sequence; the
 * overhead is taken over the linear layers), so these have no reference
 * counterpart and carry no checks.  16-bit NHWC tensors, channels a multiple of 8, pixel
 * strides ldx / ldo in elements (>= c, multiples of 8: a channel slice of a wider buffer works).
 */
/* max pooling, window k, stride, symmetric pad (<= k/2), PyTorch ceil_mode rule; out [n][P][Q] */
int abft_nhwc_maxpool(const void* x, int32_t n, int32_t h, int32_t w, int32_t c, int64_t ldx, int32_t k,
                      int32_t stride, int32_t pad, int32_t ceil_mode, int32_t dtype, void* out, int64_t ldo,
                      void* stream);
/* the same max pooling, also accumulating the column sums of its output (bucket 0 of the window
 * sums, abft_gemm_args_t.wsum) for the next layer's fused global lhs; a 3x3 consumer's border
 * buckets come from abft_nhwc_border_sums.  ws_mode: 1 or 2 (the consumer's), the caller zeroes wsum. */
int abft_nhwc_maxpool_ws(const void* x, int32_t n, int32_t h, int32_t w, int32_t c, int64_t ldx, int32_t k,
                         int32_t stride, int32_t pad, int32_t ceil_mode, int32_t dtype, void* out, int64_t ldo,
                         float* wsum, int32_t ws_ld, int32_t ws_mode, void* stream);
/* global average pooling: out[n][c] = mean over the hw pixels of image n (fp32 sum) */
int abft_nhwc_avgpool(const void* x, int32_t n, int32_t hw, int32_t c, int64_t ldx, int32_t dtype, void* out,
                      int64_t ldo, void* stream);
/* ShuffleNet v2: out = channel_shuffle(cat(x1, b), 2) for 2*half channels, stored in the "halves"
 * layout: logical channels [0, half) at physical [0, half), [half, 2*half) at [half_pad, half_pad + half) */
int abft_nhwc_interleave2(const void* x1, int64_t ld1, const void* b, int64_t ld2, int64_t pixels, int32_t half,
                          void* out, int64_t ldo, int32_t half_pad, int32_t dtype, void* stream);
/* per-CTA (lhs, rhs) slots [n][cap][2] (abft_gemm out_partials) -> sums [n][2]: a shard's per-layer
 * partials, all-reduced across ranks before abft_verify_sums (batch sharding, checksum.py:237) */
int abft_sum_partials(const double* partials, int32_t cap, int32_t ntasks, double* sums, void* stream);

/* Clear a per-forward accumulator block (one graph memset node instead of a kernel). */
int abft_zero(void* p, int64_t bytes, void* stream);

/* Library introspection */
const char* abft_last_error(void);
int abft_version(void);                 /* 10000*major + 100*minor + patch */
int abft_struct_size(int32_t which);    /* sizeof: 0 gemm args, 1 conv args, 2 global task, 3 verdict,
                                          4 thread verdict, 5 fault (ABI check for FFI mirrors) */
int abft_device_sms(void);              /* SM count of the current device (0 if none) */

#ifdef __cplusplus
}
#endif
#endif /* ABFT_B200_H */
