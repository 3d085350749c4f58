/*
 * dpkfac.h -- C ABI of libdpkfac.so, the B200 (sm_100a) DP-KFAC second-order update.
 *
 * Every entry point replaces one function of the reference's hot path
 * (kfaclab 0.1.0, /root/reference/pkg/src/kfaclab); the citation is given
 * beside each declaration.  The reference is Python-over-numpy, so its "FFI"
 * is the Python call itself: INTEGRATION.md shows the ctypes binding a
 * kfaclab maintainer would add to route kfac.py / distsim.py through here.
 *
 * Conventions
 *   - All matrix / tensor pointers are DEVICE pointers owned by the caller
 *     (torch owns every byte; the library never allocates persistent memory).
 *     Scratch space is passed in explicitly as (workspace, bytes); its size
 *     comes from the matching *_workspace_bytes query and its content need not
 *     be initialised (the GEMM engine's tile-scheduler counters at its start are
 *     cleared on the stream by each call).
 *   - Matrices are row-major float32.  Factors are d x d and exactly symmetric.
 *   - Calls are asynchronous on the given stream and stateless, hence
 *     reentrant across streams.  No C++ exception crosses this boundary.
 *   - Return value: DPK_OK or a synchronous error (bad argument, shape, CUDA
 *     launch failure).  Numeric failures (non-SPD pivot, non-positive trace or
 *     eigen denominator, non-finite values) are reported asynchronously through
 *     caller-provided device int32 "info" words: 0 = fine, >0 = failure code.
 *   - Precision: DPK_PREC_TF32 runs one tcgen05 kind::tf32 pass on
 *     round-to-nearest TF32 operands; DPK_PREC_TF32_TRUNC feeds the raw fp32
 *     bits (the tensor core truncates to TF32, no conversion pass);
 *     DPK_PREC_3XTF32 splits every operand into hi + lo TF32 parts and
 *     accumulates hi*hi + hi*lo + lo*hi (fp32-grade).  DPK_PREC_3XF16 (SPD inverse and
 *     preconditioning entry points) is the same 3-product split with fp16 hi / lo
 *     parts (11-bit significands: hi + lo carry 22 bits like 3xTF32) on kind::f16
 *     MMAs at twice the tf32 rate; each operand is first scaled by an exact power of
 *     two from its measured amax (largest magnitude in [2^14, 2^15)) and the epilogue
 *     undoes both scales exactly.
 */
#ifndef DPKFAC_H_
#define DPKFAC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* dpk_stream_t; /* a cudaStream_t (torch.cuda.current_stream().cuda_stream) */

enum {
  DPK_OK = 0,
  DPK_EARG = 1,     /* invalid argument (reference ArgumentError, errors.py:17) */
  DPK_ESHAPE = 2,   /* incompatible shapes (reference ShapeError, errors.py:13) */
  DPK_ECUDA = 3,    /* CUDA launch / runtime failure */
  DPK_ENOSPACE = 4  /* workspace too small */
};

enum { DPK_PREC_TF32 = 1, DPK_PREC_TF32_TRUNC = 2, DPK_PREC_3XTF32 = 3, DPK_PREC_3XF16 = 4 };

/* info codes written to device info words */
enum {
  DPK_INFO_OK = 0,
  DPK_INFO_TRACE = 1,      /* Tr(A) <= 0 or Tr(G) <= 0 (kfac.py:133-136) */
  DPK_INFO_NOT_SPD_A = 2,  /* damped A not positive definite (kfac.py:149-150) */
  DPK_INFO_NOT_SPD_G = 3,  /* damped G not positive definite (kfac.py:153-154) */
  DPK_INFO_EIG_DENOM = 4,  /* eigen damping denominator <= 0 (kfac.py:185-189) */
  DPK_INFO_NONFINITE = 5   /* non-finite decomposition (numerics.py:87-96) */
};

/* ------------------------------------------------------------------------
 * Operand views: how to read element (row r, column k) of a column-per-sample
 * capture X (reference convention, model.py:14-16: d x B, columns = samples).
 * ------------------------------------------------------------------------ */
enum {
  DPK_OPND_ROWS_K = 0,  /* X[r,k] = data[r*ld + k]            (rows contiguous in k)   */
  DPK_OPND_ROWS_MN = 1, /* X[r,k] = data[k*ld + r]            (e.g. nn.Linear input B x d) */
  DPK_OPND_IM2COL = 2,  /* X[(c,i,j),(n,oh,ow)] = x[n, c, oh*sh-ph+i*dh, ow*sw-pw+j*dw] or 0:
                           the implicit-im2col linear form of a Conv2d input (F.unfold order) */
  DPK_OPND_IM2COL_TAPMAJOR = 3, /* same values, rows ordered (i, j, c) -- the channels-last
                           weight order.  With an NHWC input (c contiguous, C % 32 == 0) a
                           SYRK fetches it with tiled TMA tap boxes (5-D map over the input,
                           tap-shifted coordinates, zero fill outside the image; a GEMM
                           operand uses TMA im2col loads); the factor is then a
                           symmetric permutation of the (c,i,j) one and the gradient must
                           be packed with dpk_segment.perm_khw. */
  DPK_OPND_ROWS_K_F16 = 4 /* X[r,k] = ((const __half*)data)[r*ld + k]: a feature-major fp16
                           patch matrix (dpk_im2col_materialize_f16), ld % 8 == 0.  SYRKs on
                           it run tcgen05 kind::f16 (fp32 accumulate): the same 11-bit
                           significand as the TF32 path at half the operand bytes and twice
                           the MMA rate; values beyond the fp16 range become inf and surface
                           as a non-SPD factor (NumericError). */,
  DPK_OPND_IM2COL_TAPMAJOR_F16 = 5 /* the DPK_OPND_IM2COL_TAPMAJOR view over an fp16 NHWC copy of
                           the input (dpk_im2col_convert_f16; strides in halves): SYRK only,
                           TMA-only -- rows (i, j, c) fetched by TMA im2col loads of 64 output
                           pixels x 64 channels straight into the kind::f16 MN-major operand
                           layout, so the patch matrix never exists in memory.  Requires
                           C % 64 == 0, c contiguous, 16-byte aligned strides, no bias row. */
};

typedef struct dpk_operand {
  const float* data;
  int32_t kind;
  int32_t rows;      /* feature rows, excluding the bias row */
  int32_t bias_row;  /* 1: a constant-ones row is appended LAST (model.py:140-143) */
  int32_t _pad0;
  int64_t cols;      /* number of sample columns M (B, or B*OH*OW for convs) */
  int64_t ld;        /* ROWS_K / ROWS_MN leading dimension in elements */
  /* IM2COL geometry: input tensor N x C x H x W addressed with element strides */
  int32_t C, H, W, OH, OW;
  int32_t kh, kw, sh, sw, ph, pw, dh, dw;
  int32_t _pad1;
  int64_t sn, sc, shs, sws;
} dpk_operand;

/* ------------------------------------------------------------------------
 * K1 / K2: Kronecker-factor construction with the running average fused.
 *   F <- alpha * X X^T + beta * F      (F d x d, d = rows + bias_row)
 * replaces kfac.compute_factors (kfac.py:85-104) + update_running_average
 * (kfac.py:107-125): first update alpha = s^2/M, beta = 0 (F not read);
 * later alpha = xi*s^2/M, beta = 1 - xi, where s scales the capture
 * (s = B_local for torch grad_output, model.py:9-12).  Lower-triangle tiles
 * are computed on tcgen05 tensor cores and mirrored, so F is exactly
 * symmetric like the reference's (F + F^T)/2.
 * ------------------------------------------------------------------------ */
typedef struct dpk_factor_job {
  dpk_operand x;
  float* factor;
  float alpha;
  float beta;
  /* Optional (may be NULL): device int32 holding the float bits of amax|X| when the
   * operand stores the power-of-two prescaled values X * 2^-e (the fp16 patches of
   * dpk_im2col_materialize_f16 with dpk_im2col_job.amax set); the epilogue then
   * applies alpha * 2^(2e), exactly.  e = dpk_prescale_exponent(amax). */
  const int32_t* x_amax;
} dpk_factor_job;

size_t dpk_factor_workspace_bytes(const dpk_factor_job* jobs, int n_jobs);
int dpk_syrk_ema(const dpk_factor_job* jobs, int n_jobs, void* workspace, size_t ws_bytes, int precision,
                 dpk_stream_t stream);
/* K2 entry point: identical contract; every job's operand must be DPK_OPND_IM2COL or
 * DPK_OPND_IM2COL_TAPMAJOR (implicit im2col: patches are never written; see the
 * operand kinds above).  Measured on B200 the TMA-only implicit forms are TMA-issue
 * bound, so DPKFAC materializes patches by default (dpk_im2col_materialize). */
int dpk_conv_im2col_syrk_ema(const dpk_factor_job* jobs, int n_jobs, void* workspace, size_t ws_bytes,
                             int precision, dpk_stream_t stream);

/* ------------------------------------------------------------------------
 * Patch matrix for the conv A factor, sample-major:  out[k*ld + r] = X[r, k]
 * (X = the operand's implicit-im2col view, bias ones row included), so the
 * SYRK can stream it with 2-D TMA (MN-major) at full tensor-core rate.  With a
 * channels-last input and DPK_OPND_IM2COL_TAPMAJOR rows every (pixel, tap) is
 * one contiguous C-float copy.  ld >= rows + bias_row.
 * ------------------------------------------------------------------------ */
typedef struct dpk_im2col_job {
  dpk_operand x; /* DPK_OPND_IM2COL or DPK_OPND_IM2COL_TAPMAJOR */
  float* out;
  int64_t ld;
  /* fp16 patches only, optional (NULL = no scaling): device int32 written by
   * dpk_im2col_amax (the float bits of amax|X|, the bias ones row included).  The
   * fp16 kernel then stores half(X * 2^-e) with e = floor(log2 amax) - 14, so the
   * largest patch value lands in [2^14, 2^15): nothing can overflow the fp16 range
   * (65504) and small values sit as far above the subnormals as possible; pass the
   * same pointer as dpk_factor_job.x_amax so the SYRK undoes the scale exactly. */
  int32_t* amax;
} dpk_im2col_job;

int dpk_im2col_materialize(const dpk_im2col_job* jobs, int n_jobs, dpk_stream_t stream);
/* The same patch values as fp16, FEATURE-major: out[r*ld + k] = half(X[r, k])
 * (round to nearest), ld >= cols and ld % 8 == 0; read back as DPK_OPND_ROWS_K_F16. */
int dpk_im2col_materialize_f16(const dpk_im2col_job* jobs, int n_jobs, dpk_stream_t stream);
/* The implicit-SYRK input: out = half(x * 2^-e), the dense channels-last conv input copied
 * element for element (N*H*W*C halves, 16-byte aligned; e from jobs[i].amax as above, or
 * 0 without it).  The job's x must be the dense NHWC DPK_OPND_IM2COL_TAPMAJOR view with
 * C % 8 == 0; read back through DPK_OPND_IM2COL_TAPMAJOR_F16 (same geometry, data = out).
 * One launch. */
int dpk_im2col_convert_f16(const dpk_im2col_job* jobs, int n_jobs, dpk_stream_t stream);
/* amax|X| of every job's implicit-im2col view (= amax over the conv input, or 1 with
 * a bias row, whichever is larger) into *jobs[i].amax as float bits (non-finite
 * inputs propagate: the factor then fails as non-SPD, never silently).  One launch;
 * jobs without an amax pointer are skipped. */
int dpk_im2col_amax(const dpk_im2col_job* jobs, int n_jobs, dpk_stream_t stream);

/* ------------------------------------------------------------------------
 * Grouped tensor-core GEMM used by preconditioning (and exposed for tests):
 *   out[m,n] = alpha * sum_k A[m,k] B[n,k] + beta * cin[m,n]
 * with A = a (rows M) and B = b (rows N) read through operand views.
 * symmetric=1 computes lower tiles only and mirrors (requires M == N).
 * ------------------------------------------------------------------------ */
typedef struct dpk_gemm_job {
  dpk_operand a;
  dpk_operand b;
  float* out;
  int64_t ldo;
  const float* cin; /* may alias out; not read when beta == 0 */
  int64_t ldc;
  float alpha;
  float beta;
  int32_t symmetric;
  int32_t _pad0;
} dpk_gemm_job;

size_t dpk_gemm_workspace_bytes(const dpk_gemm_job* jobs, int n_jobs);
int dpk_gemm(const dpk_gemm_job* jobs, int n_jobs, void* workspace, size_t ws_bytes, int precision,
             dpk_stream_t stream);

/* ------------------------------------------------------------------------
 * A6: trace-balancing scalar and damping shifts on device (kfac.py:128-155).
 *   pi = sqrt((tr A / d_A) / (tr G / d_G)); shift_a = pi*sqrt(gamma); shift_g = sqrt(gamma)/pi
 * shifts[2*i] = shift_a, shifts[2*i+1] = shift_g, pis[i] = pi; info[i] = DPK_INFO_TRACE on tr <= 0.
 * ------------------------------------------------------------------------ */
typedef struct dpk_pi_job {
  const float* a;
  const float* g;
  int32_t da;
  int32_t dg;
  float* shifts; /* 2 floats */
  float* pi;     /* 1 float (may be NULL) */
  int32_t* info;
} dpk_pi_job;

int dpk_trace_pi(const dpk_pi_job* jobs, int n_jobs, float gamma, dpk_stream_t stream);

/* ------------------------------------------------------------------------
 * K3: batched damped SPD inverse  dst = (src + shift*I)^-1, symmetrized
 * (numerics.sym_inverse numerics.py:100-114 via kfac.damped_inverses
 * kfac.py:140-155).  Same method as the reference (Cholesky factor, inverse from
 * the factor): n <= 128 runs one shared-memory CTA per matrix (potrf, trtri,
 * L^-T L^-1); larger n recurse on 2x2 blocks whose off-diagonal work (TRSM via
 * the triangular inverse, Schur update, inverse assembly) runs as tcgen05
 * 3xTF32 GEMMs.  On a non-positive pivot *info is set to fail_code and dst is
 * left undefined.  src and dst may not alias.
 * ------------------------------------------------------------------------ */
typedef struct dpk_spd_job {
  const float* src;
  float* dst;
  int32_t n;
  int32_t fail_code;   /* DPK_INFO_NOT_SPD_A or DPK_INFO_NOT_SPD_G */
  const float* shift;  /* device scalar added to the diagonal; NULL = 0 */
  int32_t* info;
} dpk_spd_job;

size_t dpk_chol_inv_workspace_bytes(const dpk_spd_job* jobs, int n_jobs);
int dpk_chol_inv_damped_batched(const dpk_spd_job* jobs, int n_jobs, void* workspace, size_t ws_bytes,
                                dpk_stream_t stream);

/* K3, factored form (same method, one product fewer): dst = X = L^-1 where
 * L L^T = src + shift I, lower triangular with zeros above the diagonal, row
 * stride ldd = round_up(n, 4), dst 16-byte aligned.  The damped inverse of
 * kfac.damped_inverses (kfac.py:140-155) is X^T X; the DP-KFAC optimizer keeps
 * X and applies it with dpk_precond_factored, so the final X^T X product of
 * potri (a third of the inversion's flops) is never formed on the hot path. */
typedef struct dpk_spd_factor_job {
  const float* src;
  float* dst;
  int64_t ldd;
  int32_t n;
  int32_t fail_code;
  const float* shift;
  int32_t* info;
} dpk_spd_factor_job;

size_t dpk_chol_factor_inv_workspace_bytes(const dpk_spd_factor_job* jobs, int n_jobs);
int dpk_chol_factor_inv_batched(const dpk_spd_factor_job* jobs, int n_jobs, void* workspace, size_t ws_bytes,
                                dpk_stream_t stream);

/* ------------------------------------------------------------------------
 * K5: inverse-mode preconditioning out = G_inv @ grad @ A_inv (kfac.py:251-254).
 * tmp is a d_out x d_in scratch matrix per job.
 * ------------------------------------------------------------------------ */
typedef struct dpk_precond_job {
  const float* grad;   /* d_out x d_in */
  const float* a_mat;  /* d_in x d_in  (A_inv, or Q_A for eigen) */
  const float* g_mat;  /* d_out x d_out (G_inv, or Q_G for eigen) */
  const float* a_vals; /* eigen mode: d_in eigenvalues (descending) */
  const float* g_vals; /* eigen mode: d_out eigenvalues */
  float* out;          /* d_out x d_in */
  float* tmp;          /* d_out x d_in scratch */
  int32_t d_out;
  int32_t d_in;
  int32_t* info;       /* eigen mode: DPK_INFO_EIG_DENOM if min denominator <= 0 */
} dpk_precond_job;

size_t dpk_precond_workspace_bytes(const dpk_precond_job* jobs, int n_jobs);
int dpk_precond_inverse(const dpk_precond_job* jobs, int n_jobs, void* workspace, size_t ws_bytes,
                        int precision, dpk_stream_t stream);
/* K5, factored inverses (apply_preconditioner kfac.py:244-254 with
 * G_inv = X_G^T X_G, A_inv = X_A^T X_A from dpk_chol_factor_inv_batched):
 *   out = X_G^T (X_G (grad X_A^T) X_A)   -- four triangular-clipped GEMM phases,
 * the same flops as G_inv @ grad @ A_inv.  tmp: d_out x d_in scratch. */
typedef struct dpk_precond_factor_job {
  const float* grad;  /* d_out x d_in */
  const float* xa;    /* d_in x d_in lower triangular, row stride ldxa */
  const float* xg;    /* d_out x d_out lower triangular, row stride ldxg */
  float* out;         /* d_out x d_in */
  float* tmp;         /* d_out x d_in scratch */
  int64_t ldxa;
  int64_t ldxg;
  int32_t d_out;
  int32_t d_in;
} dpk_precond_factor_job;

size_t dpk_precond_factor_workspace_bytes(const dpk_precond_factor_job* jobs, int n_jobs);
int dpk_precond_factored(const dpk_precond_factor_job* jobs, int n_jobs, void* workspace, size_t ws_bytes,
                         int precision, dpk_stream_t stream);

/* K6: eigen-mode preconditioning (kfac.py:174-191):
 *   out = Q_G ((Q_G^T grad Q_A) / (max(v_G,0) max(v_A,0)^T + gamma)) Q_A^T */
int dpk_precond_eigen(const dpk_precond_job* jobs, int n_jobs, float gamma, void* workspace, size_t ws_bytes,
                      int precision, dpk_stream_t stream);

/* ------------------------------------------------------------------------
 * K4: batched symmetric eigendecomposition (numerics.sym_eig numerics.py:75-97):
 * symmetrize, decompose, eigenvalues DESCENDING, eigenvectors as columns of q.
 * On-chip cyclic Jacobi, one CTA per matrix, n <= 128 (DPK_EARG above that).  The
 * Python layer routes larger factors to cuSOLVER syevd (torch.linalg.eigh) --
 * a library call, the open K4 gap.
 * ------------------------------------------------------------------------ */
typedef struct dpk_eig_job {
  const float* src; /* n x n */
  float* q;         /* n x n, columns = eigenvectors */
  float* w;         /* n eigenvalues, descending */
  int32_t n;
  int32_t _pad0;
  int32_t* info;    /* DPK_INFO_NONFINITE on failure */
} dpk_eig_job;

size_t dpk_syevd_workspace_bytes(const dpk_eig_job* jobs, int n_jobs);
int dpk_syevd_batched(const dpk_eig_job* jobs, int n_jobs, void* workspace, size_t ws_bytes,
                      dpk_stream_t stream);

/* ------------------------------------------------------------------------
 * K7: owner-major gradient pack / unpack for the NCCL reduce-scatter and
 * all-gather that replace distsim._aggregate_grads (distsim.py:259-265) and
 * the per-layer broadcast loop (distsim.py:333-336).  A segment moves the
 * layer gradient [W | b] (rows x (cols_w + has_bias), bias column LAST,
 * model.py:250) between a weight tensor (+ optional bias vector) and a flat
 * buffer at elem offset.  pack: flat = scale * [W | b]; unpack: W, b = scale * flat.
 * ------------------------------------------------------------------------ */
typedef struct dpk_segment {
  float* weight;     /* rows x cols_w, row stride ldw */
  float* bias;       /* rows, or NULL */
  int64_t offset;    /* element offset in the flat buffer */
  int32_t rows;
  int32_t cols_w;
  int64_t ldw;
  int32_t perm_khw;  /* 0: plain.  KH*KW: weight is rows x C x KH x KW (Conv2d) and the
                        flat row is in (kh, kw, c) order, matching DPK_OPND_IM2COL_TAPMAJOR */
  int32_t _pad0;
} dpk_segment;

int dpk_pack_owner_major(const dpk_segment* segs, int n_segs, float* flat, float scale, dpk_stream_t stream);
int dpk_unpack_owner_major(const dpk_segment* segs, int n_segs, const float* flat, float scale,
                           dpk_stream_t stream);

/* ------------------------------------------------------------------------
 * KL-clip of the preconditioned update (north_star; opt-in -- the reference has
 * none, so DPKFAC defaults it off).  With vg = lr^2 * sum over every
 * preconditioned layer of <preconditioned grad, grad>, all preconditioned grads are
 * scaled by nu = min(1, sqrt(kl_clip / |vg|)) (Ba et al. 2017; KAISA).
 *   dpk_kl_dot: out = <pre, grad> over n floats (fp64 accumulation, deterministic),
 *     one launch; workspace of dpk_kl_dot_workspace_bytes(), zeroed once (the
 *     kernel leaves its counter at zero).  Each owner writes its partial into a
 *     slot of its owner-major chunk, so the all-gather that already carries the
 *     preconditioned gradients also carries every rank's partial.
 *   dpk_unpack_owner_major_klclip: the unpack with nu applied in the same pass
 *     (nu computed on the device from the n_slots partials slot_stride apart).
 * ------------------------------------------------------------------------ */
size_t dpk_kl_dot_workspace_bytes(void);
int dpk_kl_dot(const float* pre, const float* grad, int64_t n, float* out, void* workspace, size_t ws_bytes,
               dpk_stream_t stream);
int dpk_unpack_owner_major_klclip(const dpk_segment* segs, int n_segs, const float* flat, float scale,
                                  const float* kl_slots, int n_slots, int64_t slot_stride, float kl_clip, float lr,
                                  dpk_stream_t stream);

/* ------------------------------------------------------------------------
 * Peer all-gather over NVLink (single node; DPKFAC(peer_gather=True)) -- replaces the
 * closing all-gather of the owner-major exchange (distsim.py:333-336 broadcast of the
 * owners' preconditioned gradients; NCCL all_gather_into_tensor otherwise):
 *   dpk_ipc_export: the cudaIpcMemHandle_t (64 bytes) of the allocation holding ptr
 *     and ptr's byte offset in it (caching allocators sub-allocate);
 *   dpk_ipc_open: map another process's exported allocation into `device`'s context;
 *   dpk_peer_gather: dst[i*count .. (i+1)*count) = srcs[i][0 .. count) for every
 *     source (own chunk local, the others peer pointers), one launch; count % 4 == 0,
 *     16-byte aligned.  The caller orders it after every rank's chunk is written.
 * ------------------------------------------------------------------------ */
int dpk_ipc_export(const void* ptr, int device, void* handle, int64_t* offset);
int dpk_ipc_open(const void* handle, int device, void** base);
int dpk_ipc_close(void* base);
int dpk_peer_gather(float* dst, const float* const* srcs, int n_src, int64_t count, dpk_stream_t stream);

/* Library / device introspection. */
const char* dpk_version(void);
const char* dpk_last_error(void);
/* Host-thread setting: tensor-core launches made from this thread use at most `sms`
 * SMs (0 = all).  DPKFAC caps the throughput-bound size classes so the latency-bound
 * inversion chain of the largest factors keeps SMs free while they run. */
int dpk_set_launch_cap(int sms);
/* number of kernels this library has launched in the process (bench evidence) */
unsigned long long dpk_launch_count(void);
/* debug: %globaltimer checkpoints (ns) of CTA 0 of the last GEMM launched with DPK_DEBUG_TS=1 */
int dpk_debug_timestamps(unsigned long long* host16);
/* debug: per work unit of CTA 0 of that launch (first 64 units), 5 checkpoints each: MMA
 * start, first chunk ready, last MMA issued, epilogue start, epilogue end */
int dpk_debug_unit_timestamps(unsigned long long* host320);

#ifdef __cplusplus
}
#endif
#endif /* DPKFAC_H_ */
