/*
 * ldbp.h — C ABI of libldbp, the B200 (sm_100a) hot path of learned digital backpropagation.
 *
 * Method: C. Häger, H. D. Pfister, "Physics-Based Deep Learning for Fiber-Optic
 * Communication Systems", arXiv:2010.14258.  Citations "P:n" are lines of that paper's
 * source; "S:n" lines of SPEC.md; "§8(x)" sections of SURVEY.md.
 *
 * The model (Eq. (7)) maps each independent circular block x in C^n through
 * M steps,   a = h^(i) (*) u   (circular, centred FIR, reading G1 of DESIGN.md:
 *            a_t = sum_{j=-Kh}^{Kh} h_j u_{(t-j) mod n}, frequency response
 *            sum_k h_k e^{-jk omega} as in P:895-896),
 *            u <- a * exp(j gamma'_i |a|^2)  (Kerr step, P:384-388 with the per-step scalar of
 *            Remark 2; gamma' is signed and carries gamma*L_eff*xi).
 *
 * CONVENTIONS (every entry point)
 *  - All data pointers are DEVICE pointers owned by the caller.  The library never allocates
 *    in a call, keeps no mutable global state, is thread-safe, and enqueues its work
 *    asynchronously on `cuda_stream` (a cudaStream_t; NULL = legacy default stream).  No call
 *    synchronises the host, so every call is CUDA-graph capturable.  Results are valid once
 *    the stream has completed the enqueued work.
 *  - Complex arrays are complex64: interleaved (re, im) float32 pairs, row-major, 8-byte
 *    aligned.  Blocks: [B][n].  Taps: [M][T], tap j in [-Kh, Kh] stored at index j + Kh.
 *    gamma: float32 [M] (phase = gamma[i] * |a|^2, radians, |a|^2 in the units of x^2).
 *  - Gradient convention for a complex z and real loss L: dL/dRe z + i dL/dIm z.
 *    Real-valued gradient outputs are float64; complex ones are stored as [..][2] float64.
 *  - Every call returns an ldbp_status.  Validation failures return before anything is
 *    enqueued; a CUDA launch failure returns LDBP_ECUDA.  ldbp_last_error() then returns a
 *    thread-local human-readable detail string.
 *  - Results are deterministic: fixed reduction order, no floating-point atomics.
 */
#ifndef LDBP_H_
#define LDBP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LDBP_ABI_VERSION 2

/* Problem dimensions. */
typedef struct ldbp_dims {
  int64_t batch;   /* B >= 0 independent circular blocks (B = 0: every call is a no-op)   */
  int64_t n;       /* samples per block, n >= 1                                             */
  int32_t steps;   /* M >= 1 model steps (layers)                                */
  int32_t taps;    /* T = 2*Kh + 1, odd, 1 <= T <= LDBP_MAX_TAPS and T <= n                 */
  uint32_t flags;  /* bitwise OR of ldbp_flags                                              */
  int32_t reserved;/* must be 0                                                             */
} ldbp_dims;

/* Compiled specialisations per Kh = 0..15 (T <= 31).  T <= 15 covers every
   BASELINE config and model of the paper; 17..31 are correct but register-heavy (the per-thread
   tap and halo windows spill), and the ESSM entry points keep T <= 15. */
#define LDBP_MAX_TAPS 31

enum ldbp_flags {
  /* Symmetric filters h_{-j} = h_j.  The kernels read only taps[Kh..T-1] of each
     step (the caller promises symmetry), use the folded FIR of fig:filter, and
     return tied-parameter gradients: dtaps[j] = dtaps[-j] = g_j + g_{-j}. */
  LDBP_SYMMETRIC = 1u,
  /* Use IEEE-accurate sincosf for the Kerr rotation instead of the MUFU approximation. */
  LDBP_PRECISE = 2u,
  /* Check every step's activations for non-finite values (SPEC "NaN in activations -> error with
     layer index"): the forward kernels flag the first step whose output holds a NaN/Inf;
     the call then synchronises its stream once and returns LDBP_ENONFINITE with the 1-based step
     in ldbp_last_error().  Applies to ldbp_forward/backward/loss_grad/train_step/rx_train_grad
     (the training calls then use the store-all schedule, so every step is checked); it adds
     256 workspace bytes. */
  LDBP_CHECK_FINITE = 4u,
  /* ldbp_forward only (ignored by the other calls; the forward ignores it when it needs more than
     one launch or LDBP_CHECK_FINITE is set): a serving pipeline of independent batches (BJ config 2,
     one forward per batch of received blocks).  The caller guarantees that no kernel enqueued earlier
     on the stream that may still be running writes x / taps / gamma or reads or writes y — e.g.
     consecutive forwards over a rotation of at least 3 distinct input/output buffers.  The forward is
     then launched as a programmatic dependent launch (no griddepcontrol.wait): its CTAs start loading
     their windows while the previous forward's last wave drains, instead of after it completes. */
  LDBP_STREAM_PIPELINE = 8u
};

typedef enum ldbp_status {
  LDBP_OK = 0,
  LDBP_EINVAL = -1,      /* null/aliased pointer, reserved != 0, unknown flag, bad hyper-parameter */
  LDBP_ESHAPE = -2,      /* T even, T > LDBP_MAX_TAPS, T > n, M < 1, n < 1, B < 0          */
  LDBP_EALIGN = -3,      /* a complex pointer is not 8-byte aligned, a double one not 8-byte */
  LDBP_EWORKSPACE = -4,  /* ws_bytes < ldbp_workspace_bytes(...) or ws == NULL when needed  */
  LDBP_ECUDA = -5,       /* a CUDA runtime error (detail in ldbp_last_error())               */
  LDBP_ENONFINITE = -6   /* LDBP_CHECK_FINITE: a step produced NaN/Inf (step in ldbp_last_error()) */
} ldbp_status;

typedef enum ldbp_op {
  LDBP_OP_FORWARD = 0,
  LDBP_OP_BACKWARD = 1,
  LDBP_OP_LOSS_GRAD = 2,
  LDBP_OP_TRAIN_STEP = 3
} ldbp_op;

int ldbp_abi_version(void);
const char* ldbp_status_string(int status);
/* Thread-local detail of the last failing call on this thread ("" if none). */
const char* ldbp_last_error(void);

/* Device workspace (bytes) the given op needs for these dims; 0 means ws may be NULL.
   Returns a status; *bytes is written on LDBP_OK.
   Backward / loss_grad / train_step choose between two schedules for row a7 (activations):
   "store-all" (default while B*n >= 2^20 and M*B*n*8 bytes <= LDBP_ACT_BUDGET_GB, env, default 96; forced by
   env LDBP_BWD_MODE=1): the forward stores every step's activation in the workspace
   (M*B*n*8 bytes + O(grid*M*T)) and one fused reverse kernel needs no recompute; otherwise (or
   LDBP_BWD_MODE=0) checkpoint + recompute segments with ~M/6 checkpoints.  The choice depends
   only on dims and the environment, so this query and the call agree. */
int ldbp_workspace_bytes(const ldbp_dims* d, int op, size_t* bytes);

/* Number of CUDA kernel launches the op enqueues for these dims (for accounting). */
int ldbp_launch_count(const ldbp_dims* d, int op, int* launches);

/*
 * ldbp_forward — y = f_theta(x), Eq. (7) for every block.
 *   x      [B][n] complex64 in;  y [B][n] complex64 out (must not alias x or ws)
 *   taps   [M][T] complex64;     gamma [M] float32
 *   ws     workspace of ldbp_workspace_bytes(d, LDBP_OP_FORWARD) bytes (may be 0 -> NULL ok)
 */
int ldbp_forward(const ldbp_dims* d, const void* x, void* y, const void* taps, const float* gamma,
                 void* ws, size_t ws_bytes, void* cuda_stream);

/*
 * ldbp_backward — reverse-mode sweep of Eq. (7) for an incoming gradient gy = dL/dy
 * (per step: c = Im(gv conj v), ga = gv e^{-j phi} + 2 gamma' c a,
 * dgamma' = sum c|a|^2, dh_j = sum ga_t conj(u_{t-j}), gu_s = sum_j conj(h_j) ga_{s+j}).
 *   x      [B][n] complex64 (the forward input; the call re-runs the forward into ws)
 *   gy     [B][n] complex64
 *   dtaps  [M][T][2] float64 out: sum over all blocks (tied-parameter form with LDBP_SYMMETRIC)
 *   dgamma [M] float64 out
 *   gx     [B][n] complex64 out, or NULL to skip dL/dx
 */
int ldbp_backward(const ldbp_dims* d, const void* x, const void* gy, const void* taps,
                  const float* gamma, double* dtaps, double* dgamma, void* gx_or_null,
                  void* ws, size_t ws_bytes, void* cuda_stream);

/*
 * ldbp_loss_grad — waveform-MSE training gradient (reading G7; Eq. (2) P:280-285 with the
 * 1/N applied later): with e = f_theta(x) - target,
 *   buf[0]                    = sum_{blocks,t} |e|^2                       (UNscaled)
 *   buf[1 .. M]               = d buf[0] / d gamma'_i
 *   buf[1+M .. 1+M+2MT)       = d buf[0] / d taps as [M][T][2]
 * Taps are multiplied by tap_mask (uint8 [M][T], 1 keep / 0 prune) when non-NULL;
 * masked taps get gradient 0.  buf is this device's UNREDUCED contribution (data parallel:
 * all-reduce SUM it across ranks, then call ldbp_adam_update with n_global = sum B*n).
 */
int ldbp_loss_grad(const ldbp_dims* d, const void* x, const void* target, const void* taps,
                   const float* gamma, const uint8_t* tap_mask_or_null, double* buf,
                   void* ws, size_t ws_bytes, void* cuda_stream);

/*
 * ldbp_adam_update — bias-corrected Adam (mu per Table I) on the real
 * parameter vector master = [taps as [M][T][2] | gamma[M]] (float64, length 2MT+M), with
 * gradient g = reorder(buf_reduced)/n_global.  m, v: float64 moments (same layout), t >= 1 the
 * 1-based step.  Masked taps are forced to 0 with m = v = 0; gamma entries with
 * gamma_learnable[i] == 0 are left unchanged.  Writes the float32 working copies taps_out
 * ([M][T] complex64) and gamma_out ([M]).  Requires lr > 0, 0 <= b1,b2 < 1, eps > 0, n_global > 0.
 */
int ldbp_adam_update(const ldbp_dims* d, const double* buf_reduced, double n_global,
                     double* master, double* m, double* v, int64_t t,
                     double lr, double b1, double b2, double eps,
                     const uint8_t* tap_mask_or_null, const uint8_t* gamma_learnable_or_null,
                     void* taps_out, float* gamma_out, void* cuda_stream);

/*
 * ldbp_train_step — single-process training step: ldbp_loss_grad on the working copies
 * (taps_work, gamma_work) then ldbp_adam_update with n_global = B*n.  buf receives the
 * gradient buffer of this step (buf[0] = sum |e|^2 before the update).
 */
int ldbp_train_step(const ldbp_dims* d, const void* x, const void* target,
                    void* taps_work, float* gamma_work, double* master, double* m, double* v,
                    int64_t t, double lr, double b1, double b2, double eps,
                    const uint8_t* tap_mask_or_null, const uint8_t* gamma_learnable_or_null,
                    double* buf, void* ws, size_t ws_bytes, void* cuda_stream);

/*
 * Receiver-chain symbol loss (the paper's training objective and figure
 * of merit).  Per block b of n samples at sps samples/symbol (K = n/sps symbols):
 *   s_tilde = M y / sqrt(P_b)      M: decimating circular FIR, real even taps h_mf[m + L],
 *                                  m in [-L, L]  (s_tilde_k = sum_m h[m] y_{(k sps - m) mod n};
 *                                  Eq. (12), reading G19: the periodic RRC impulse
 *                                  response truncated to +-L samples)
 *   phi_b = arg(s^H s_tilde)        genie phase
 *   errs_b = sum_k |e^{-j phi_b} s_tilde_k - s_k|^2   (symbol MSE x K; Eq. (13))
 * and gy = dL/dy of L = sum_b errs_b (full chain rule incl. the phase).
 *   y, gy    [B][n] complex64;  symbols [B][K] complex64 (unit power);  power_w [B] float32 (W)
 *   h_mf     [2L+1] float32, 0 <= L <= 256, 2L+1 <= n;  sps in [1, 4], n % sps == 0
 *   errs     [B] float64 out;  gy may be NULL (loss only)
 * Deterministic (fixed-order fp64 block reductions).  Workspace: ldbp_rx_workspace_bytes.
 */
int ldbp_rx_workspace_bytes(int64_t batch, int64_t n, int32_t sps, size_t* bytes);
int ldbp_rx_loss_grad(int64_t batch, int64_t n, int32_t sps, int32_t mf_half, const void* y,
                      const void* symbols, const float* power_w, const float* h_mf, double* errs,
                      void* gy_or_null, void* ws, size_t ws_bytes, void* cuda_stream);

/*
 * ldbp_rx_train_grad — training gradient of the receiver-chain loss through LDBP:
 *   buf = [sum_b errs_b | d/d gamma' [M] | d/d taps [M][T][2]]   (UNscaled, this device's blocks;
 *   with tap_mask as in ldbp_loss_grad), y = f_theta(x) (Eq. 7).  One storing forward, the two
 *   receiver kernels, one reverse sweep seeded with dL/dy (store-all schedule; the segment
 *   schedule re-runs the forward for its checkpoints).  Data parallel: all-reduce buf, then
 *   ldbp_adam_update with n_global = total symbols.  Workspace: ldbp_rx_train_workspace_bytes.
 */
int ldbp_rx_train_workspace_bytes(const ldbp_dims* d, int32_t sps, size_t* bytes);
int ldbp_rx_train_grad(const ldbp_dims* d, const void* x, const void* symbols, const float* power_w,
                       int32_t sps, int32_t mf_half, const float* h_mf, const void* taps,
                       const float* gamma, const uint8_t* tap_mask_or_null, double* buf,
                       void* ws, size_t ws_bytes, void* cuda_stream);

/*
 * Receiver-chain loss with the EXACT circulant matched filter (Eq. (12),
 * M is "a circulant matrix that represents the matched filter"; Eq. (13)).
 * Per block b of n samples (power of two, n <= 65536) at sps in [1, 4] samples/symbol:
 *   z = F^-1 diag(RRC_rolloff) F y   (root-raised-cosine response of the periodic frame)
 *   s_tilde_k = z[k sps],  phi_b = arg(s^H s_tilde),  a = e^{-j phi_b} / sqrt(power_w[b])
 *   errs_b = sum_k |a s_tilde_k - s_k|^2,   L = sum_b w_b errs_b   (w = weights, or all 1)
 *   gy = dL/dy (full chain rule incl. the genie phase; M^T = F^-1 diag(RRC) F U, U = upsampling)
 * y, gy [B][n] complex64; symbols [B][n/sps] complex64; power_w, weights [B] float32; errs [B]
 * float64 out (unweighted); gy may be NULL.  No workspace.  One CTA per block up to 2^14 samples,
 * a 2-/4-CTA cluster beyond (fp32 shared-memory FFTs, fp64 fixed-order reductions: deterministic).
 *   ldbp_rx_exact_train_grad: buf = [sum_b w_b errs_b | d/dgamma' [M] | d/dtaps [M][T][2]] through
 *   LDBP (UNscaled, this device's blocks; tap_mask as in ldbp_loss_grad), y = f_theta(x).
 */
int ldbp_rx_exact_loss_grad(int64_t batch, int64_t n, int32_t sps, float rolloff, const void* y,
                            const void* symbols, const float* power_w, const float* weights_or_null,
                            double* errs, void* gy_or_null, void* cuda_stream);
int ldbp_rx_exact_train_workspace_bytes(const ldbp_dims* d, int32_t sps, size_t* bytes);
int ldbp_rx_exact_train_grad(const ldbp_dims* d, const void* x, const void* symbols,
                             const float* power_w, const float* weights_or_null, int32_t sps,
                             float rolloff, const void* taps, const float* gamma,
                             const uint8_t* tap_mask_or_null, double* buf, void* ws, size_t ws_bytes,
                             void* cuda_stream);

/*
 * Transmitted waveform (the target of the waveform-MSE loss; BASELINE C3 "MSE loss vs
 * transmitted waveform") from transmitted symbols, on the device: Eq. (11) on the periodic frame
 * (P:737-743), RRC roll-off `rolloff` applied as its exact frequency response:
 *   w_b = sqrt(power_w[b]) * sps * e^{j phase[b]} * F^-1 diag(RRC) F U s_b,
 *   out[b][t] = w_b[(t - shift[b]) mod n]          (U: upsampling by sps with zeros)
 * codes: uint8 [batch][n / sps] indices into constellation (complex64 [q], 1 <= q <= 256; codes >= q
 * read entry 0); shift (int32 [batch]) and phase (float32 [batch], rad) may be NULL (0); out:
 * complex64 [batch][n].  n a power of two <= 2^16, sps in [1, 4] dividing n.  Device pointers, the
 * caller's stream, no workspace, no host sync.  Lets a training step's targets cross PCIe as 1 byte
 * per symbol (bench.py e2e).
 */
int ldbp_tx_waveform(int64_t batch, int64_t n, int32_t sps, float rolloff, const uint8_t* codes,
                     const void* constellation, int32_t q, const float* power_w, const int32_t* shift_or_null,
                     const float* phase_or_null, void* out, void* cuda_stream);

/*
 * Learned ESSM (paper §III-D, Eq. nl_filtered): the nonlinear
 * step of Eq. (7) becomes  v_t = a_t exp(j gamma'_i sum_{k=-kappa}^{kappa} eta^(i)_k |a_{(t-k) mod n}|^2)
 * with real per-step filters eta [M][2 kappa + 1] (tap k at index k + kappa), 0 <= kappa <= 32,
 * 2 kappa + 1 <= n.  All pointers are device pointers as above; one launch per step (shared-
 * memory tiles with circular halos: the filter's cone grows by Kh + kappa per step).
 *   ldbp_essm_forward:   y = f_theta(x)
 *   ldbp_essm_loss_grad: buf = [sum |y - target|^2 | dgamma' [M] | dtaps [M][T][2] | deta [M][2kappa+1]]
 *                        (UNscaled, tied taps with LDBP_SYMMETRIC as in ldbp_loss_grad; no mask)
 * Workspace: ldbp_essm_workspace_bytes(d, kappa, LDBP_OP_FORWARD | LDBP_OP_LOSS_GRAD).
 */
int ldbp_essm_workspace_bytes(const ldbp_dims* d, int32_t kappa, int op, size_t* bytes);
int ldbp_essm_forward(const ldbp_dims* d, int32_t kappa, const void* x, void* y, const void* taps,
                      const float* gamma, const float* eta, void* ws, size_t ws_bytes,
                      void* cuda_stream);
int ldbp_essm_loss_grad(const ldbp_dims* d, int32_t kappa, const void* x, const void* target,
                        const void* taps, const float* gamma, const float* eta, double* buf,
                        void* ws, size_t ws_bytes, void* cuda_stream);

/*
 * GPU split-step Fourier channel generator (§IV-A): the link
 * the oracle simulates, per block of n samples (power of two, 2 <= n <= 65536), in one launch:
 *   for each of `spans` spans: for each step delta_s (s < steps_per_span <= 64, deltas_km_host[s]):
 *     u <- u e^{j gamma L_eff(delta_s) |u|^2}                     (Kerr at the segment start, G5)
 *     U_k <- U_k e^{-alpha delta_s / 2} e^{j beta2/2 omega_k^2 delta_s}   (Eqs. (4)-(6))
 *   then the EDFA: u <- e^{alpha span_km / 2} u + ase_sigma * z[span]
 *   omega_k = 2 pi fftfreq(n) fs_hz;  beta2 in s^2/km, alpha in 1/km (nepers), gamma in 1/(W km)
 * ASE draws z (CN(0,1)): noise_or_null != NULL: the given [spans][B][n] complex64 array;
 *   otherwise, if ase_sigma != 0, drawn in the kernel by Philox4x32-10 keyed by
 *   (ase_seed, global block ase_block0 + b, span, sample) — ldbp_inputs.ase_cn_philox is the same
 *   generator in numpy, so a batch sharded over ranks draws the same noise for any rank count;
 *   ase_sigma == 0 and noise NULL: noiseless.
 * decim == 0: u is overwritten with the channel output;  decim > 0: r [B][n/decim] receives the
 * brick-wall low-pass (|fftfreq| <= cutoff) output sampled every decim samples (G8).
 * deltas_km_host is a HOST array read during the call (the values travel in kernel parameters:
 * no copy, no host synchronisation; the call is asynchronous like every other entry point).
 * fp32 in shared memory: one CTA per block up to n = 16384, a 2- or 4-CTA cluster (distributed
 * shared memory, four-step split of the DFT) for 32768 / 65536; dispersion factors and twiddles
 * are fp64-accurate.  Workspace: ldbp_ssfm_workspace_bytes (S x n complex64 dispersion table).
 */
int ldbp_ssfm_workspace_bytes(int64_t n, int32_t steps_per_span, size_t* bytes);
int ldbp_ssfm_link(int64_t batch, int64_t n, int32_t spans, int32_t steps_per_span,
                   const double* deltas_km_host, double span_km, double alpha_np, double beta2,
                   double gamma, double fs_hz, double ase_sigma, const void* noise_or_null,
                   uint64_t ase_seed, int64_t ase_block0, void* u, void* r_or_null, int32_t decim,
                   double cutoff, void* ws, size_t ws_bytes, void* cuda_stream);

/*
 * Launch tracing (profiling aid; off by default; per calling thread).
 * ldbp_trace_begin(capacity) makes every kernel launch of later calls on this thread be
 * bracketed by two CUDA events recorded on the call's stream (events are created here, not
 * in the hot calls' non-traced path).  ldbp_trace_end() waits for those events, writes up to
 * `capacity` records in launch order and stops tracing.  `kind` is an ldbp_kernel_kind;
 * `steps` the model steps the launch covers; `samples` the real (owned) samples B*n it
 * produces; `ms` the event-timed duration.  Recording more launches than the capacity given
 * to ldbp_trace_begin drops the excess (count reports all launches seen).
 */
typedef enum ldbp_kernel_kind {
  LDBP_K_FORWARD = 1,   /* fused forward tile kernel (rows a1-a4)                 */
  LDBP_K_BACKWARD = 2,  /* backward segment kernel (rows a5-a8, recompute + adjoint) */
  LDBP_K_REDUCE = 3,    /* fp64 partial reduction (row a8)                         */
  LDBP_K_ADAM = 4,      /* Adam + mask (row a10)                                   */
  LDBP_K_REVERSE = 5,   /* store-all reverse tile kernel (rows a5, a6, a8)         */
  LDBP_K_RX = 6,        /* receiver-chain loss kernels (NEXT-1)                    */
  LDBP_K_ESSM = 7,      /* ESSM step kernels (NEXT-4)                              */
  LDBP_K_SSFM = 8,      /* SSFM channel generator kernels (NEXT-2)                 */
  LDBP_K_TINY = 9       /* one-CTA fused training step of tiny problems (C1)      */
} ldbp_kernel_kind;

typedef struct ldbp_trace_record {
  int32_t kind;
  int32_t steps;
  int64_t samples;
  float ms;
  int32_t reserved;
} ldbp_trace_record;

int ldbp_trace_begin(int capacity);
int ldbp_trace_end(ldbp_trace_record* out, int capacity, int* count);

#ifdef __cplusplus
}
#endif

#endif /* LDBP_H_ */
