/*
 * lrnr_gpu.h -- C ABI of the B200-native LRNR / FastLRNR residual+gradient path.
 *
 * Drop-in boundary for the hot path of arXiv 2410.04001's reference
 * (/root/reference/proj).  The reference's own "plugin" surface for this path is
 *     lrnr::training::run_batch_gradient(Trainables, ParamSelector, SetupFn, EmitFn,
 *                                        n_terms, ParallelConfig)   (training.hpp:200-202)
 * driven by the PinnTermEmitter (training.cpp:270-329) or the fast-phase emitter
 * (training.cpp:521-563), plus the plain losses loss_tune / loss_fast /
 * loss_meta (training.hpp:90-100) and the per-point jet_forward / residual
 * (model.hpp:118-119, pde.hpp:56).  run_batch_gradient interprets arbitrary
 * caller closures and cannot be offloaded as such; this ABI replaces the
 * (emitter + run_batch_gradient) PAIRS that the training loops call, with the
 * same semantics:
 *   - result = BatchGradResult{value, comps[4], grad} (training.hpp:189-195),
 *   - grad in ParamPacker order (autodiff.cpp:926-946): CoefficientsOnly ->
 *     s_1..s_L concatenated; BasesBiasesAndHyper -> per layer U_l, V_l, b_l,
 *     then hypernetwork W_k, b_k,
 *   - NonFiniteError(layer_tag) (autodiff.hpp:28-34) -> LRNR_ENONFINITE plus
 *     lrnr_gpu_last_layer_tag(),
 *   - std::invalid_argument from require() (linalg.hpp:74-76) -> LRNR_EINVAL.
 * See INTEGRATION.md for the C++ adapter a reference maintainer would add.
 *
 * Plain pointers and sizes only; host arrays are row-major double (the
 * reference's DenseMatrix/DenseVector storage, linalg.hpp:15-46).
 *
 * Flat parameter layouts:
 *   LRNR  (LrnrParams, model.hpp:38-49): per layer l = 0..L-1:
 *           U_l (widths[l+1] x ranks[l]), V_l (widths[l] x ranks[l]), b_l (widths[l+1]).
 *   Fast  (FastParams, model.hpp:65-78): v_in (m_in x r_0); per inner l = 0..L-2:
 *           u_hat (red[l] x r_l), b_hat (red[l]), v_hat (red[l] x r_{l+1});
 *           u_out (m_out x r_{L-1}); b_out (m_out).
 *   Hyper (HyperParams, model.hpp:83-95): per layer k: W_k (hw[k+1] x hw[k]), b_k (hw[k+1]).
 *
 * Threading: one context = one device + one stream; a context is not
 * thread-safe (use one per host thread / GPU).  Results are bitwise
 * run-to-run deterministic for a fixed device (fixed-order reductions, no
 * floating-point atomics), mirroring run_batch_gradient's thread-count
 * invariance (training.cpp:197-199).
 */
#ifndef LRNR_GPU_H
#define LRNR_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define LRNR_OK 0
#define LRNR_EINVAL 1      /* shape / argument error  (std::invalid_argument)            */
#define LRNR_ENONFINITE 2  /* non-finite loss term    (NonFiniteError, see last_layer_tag) */
#define LRNR_ECUDA 3       /* CUDA runtime failure                                        */
#define LRNR_ENOMEM 4      /* device allocation failure                                   */
#define LRNR_ESTATE 5      /* call order error (e.g. no model / points set)               */
#define LRNR_ENCCL 6       /* NCCL failure (communicator init / all-reduce)               */

/* activation (ActivationKind, model.hpp:18; sin is this build's extension) */
#define LRNR_ACT_TANH 0
#define LRNR_ACT_SIN 1

/* arithmetic type of the device path */
#define LRNR_F64 0
#define LRNR_F32 1

/* model slots */
#define LRNR_MODEL_LRNR 0
#define LRNR_MODEL_FAST 1

typedef struct lrnr_gpu_ctx lrnr_gpu_ctx;

/* ---- context ---- */
/* One context = one device + one stream + resident parameters: the role of the
 * reference's per-thread Tape and its bindings (autodiff.hpp:36-170, TapeBindings
 * autodiff.hpp:244, make_bindings autodiff.cpp:979-1018). */
int lrnr_gpu_create(int device, lrnr_gpu_ctx** out);
int lrnr_gpu_destroy(lrnr_gpu_ctx* ctx);
const char* lrnr_gpu_last_error(const lrnr_gpu_ctx* ctx);
/* layer tag of the last LRNR_ENONFINITE (NonFiniteError::layer_tag semantics:
 * l+1 for LRNR layer l, 0 for the FastLRNR input factor, -1 otherwise). */
/* NonFiniteError::layer_tag of the last LRNR_ENONFINITE (autodiff.hpp:28-34). */
int lrnr_gpu_last_layer_tag(const lrnr_gpu_ctx* ctx);
/* Use a caller-owned cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream);
 * NULL restores the context's own stream. */
/* Stream for all work of the context (no reference counterpart: the reference is synchronous). */
int lrnr_gpu_set_stream(lrnr_gpu_ctx* ctx, void* cuda_stream);
/* Options.  LRNR_OPT_FAST_SINCOS (FP32 sin networks): 1 = sin/cos from the SFU
 * approximations after a Cody-Waite reduction (~4e-7 absolute), 0 = polynomial
 * sin/cos after a 3-term reduction (~1.5 ulp, default).  LRNR_OPT_KERNEL:
 * 0 = auto (default): every FP32 model with ranks <= 32 (the LRNR and the
 * FastLRNR) on the tcgen05 tensor-core tile kernel (FP16 two-term split
 * operands, FP32 accumulation), other FP32/FP64 shapes with ranks <= 64 on
 * the FMA tile-GEMM kernel, the rest on the per-point streaming kernel;
 * batches below ~16 points per SM on the small-batch latency kernel (one CTA
 * per point, threads across neurons / ranks);
 * 1 = force the streaming kernel, 2 = tensor-core kernel wherever it applies
 * (also FastLRNR), 3 = FMA tile kernel (no tensor cores), 4 = small-batch
 * kernel at any size, 5 = narrow-network kernel wherever it applies. */
#define LRNR_OPT_FAST_SINCOS 1
#define LRNR_OPT_KERNEL 2
#define LRNR_OPT_TILE_P 3   /* FP32 wide-layer tile: 64 points x 512 threads (default) or 32 x 256 (2 CTAs/SM) */
/* LRNR_OPT_SOLVE (lrnr_gpu_fast_solve): 0 = auto: the persistent solver (one
 * thread-block cluster, one warp per loss term, the whole loop in one launch,
 * per-epoch reduction over distributed shared memory) when every width and
 * rank is <= 32 and the terms fit 8 CTAs x 16 warps; 1 = the graph path (one
 * captured epoch replayed per epoch). */
#define LRNR_OPT_SOLVE 4
/* LRNR_OPT_META_PREC (meta step, lrnr_gpu_meta_loss_grad / lrnr_gpu_meta_terms_grad,
 * FP32 LRNR): 0 = FP32 throughout on the FMA tile kernel (default); 1 = BF16
 * tensor-core operands with FP32 accumulation and FP32 activation / residual /
 * reduction math (tcgen05 meta kernel; BASELINE config 4's "BF16/TF32 inputs
 * with FP32 accumulate"); widths (2, ..., 1), ranks <= 64. */
#define LRNR_OPT_META_PREC 5
int lrnr_gpu_set_option(lrnr_gpu_ctx* ctx, int opt, int value);
/* Number of kernels this context has launched so far (instrumentation). */
/* Kernels launched so far (instrumentation; no reference counterpart). */
int64_t lrnr_gpu_launch_count(const lrnr_gpu_ctx* ctx);

/* ---- model upload (replaces the Tape bindings, autodiff.cpp:826-868) ---- */
/* LrnrParams; widths[L] must be 1 (scalar PDE output), widths[0] must be 2. */
int lrnr_gpu_set_lrnr(lrnr_gpu_ctx* ctx, int depth, const int64_t* widths, const int64_t* ranks,
                      const double* params, int act, int dtype);
/* FastParams (EIM-reduced surrogate); m_in = 2, m_out = 1. */
int lrnr_gpu_set_fast(lrnr_gpu_ctx* ctx, int depth, const int64_t* ranks, const int64_t* red_ranks,
                      int64_t m_in, int64_t m_out, const double* fparams, int act, int dtype);
/* HyperParams: n_layers affine layers, hw[0] = 3, hw[n_layers] = r_total of the
 * model it feeds; tanh hidden, ReLU output, mu normalized by the box
 * (model.cpp:74-81,294-318). */
int lrnr_gpu_set_hyper(lrnr_gpu_ctx* ctx, int n_layers, const int64_t* hw, const double* hparams,
                       const double* box_lo, const double* box_hi);

/* ---- collocation points (CollocationBatch::interior, pde.hpp:33-40) ----
 * n_inst groups of n_per_inst consecutive (x, t) pairs; group i belongs to
 * PDE-parameter instance i.  Host pointer (copied) or device pointer to the
 * same double (x, t) pairs (borrowed; must stay valid while used). */
int lrnr_gpu_set_points(lrnr_gpu_ctx* ctx, const double* xt, int64_t n_inst, int64_t n_per_inst);
int lrnr_gpu_set_points_device(lrnr_gpu_ctx* ctx, const void* xt_dev, int64_t n_inst,
                               int64_t n_per_inst);
/* Double-buffered host points for a training loop: lrnr_gpu_stage_points copies
 * the NEXT batch (host pointer, best pinned) into a staging buffer on an internal
 * copy stream and returns at once, so the copy overlaps the gradient calls of the
 * current batch; the host buffer must stay valid and unmodified until the
 * following lrnr_gpu_use_staged_points returns.  lrnr_gpu_use_staged_points makes
 * the staged batch current (later work on the context's stream waits for the
 * copy).  Same point layout and counts as lrnr_gpu_set_points. */
int lrnr_gpu_stage_points(lrnr_gpu_ctx* ctx, const double* xt, int64_t n_inst, int64_t n_per_inst);
int lrnr_gpu_use_staged_points(lrnr_gpu_ctx* ctx);

/* ---- per-step gradient calls (host buffers; synchronous) ----
 *
 * lrnr_gpu_loss_grad_s: PinnTermEmitter, fine-tune mode, interior terms
 * (training.cpp:286-293): term_i = w * N[u](x_i,t_i; mu)^2 with
 * N = u_t + mu1 u_x - mu2 u_xx - mu3 u(1-u) (pde.cpp:9-13), CoefficientsOnly.
 * Requires n_inst == 1.  w <= 0 selects the reference weight 1/n
 * (training.cpp:364-366).  Outputs: value, comps[4] = {residual, boundary,
 * sparse, local}, grad_s (r_total).  model = LRNR_MODEL_LRNR or _FAST (the
 * squared-residual objective on the FastLRNR, BASELINE config 1). */
int lrnr_gpu_loss_grad_s(lrnr_gpu_ctx* ctx, int model, const double* s, const double* mu, double w,
                         double* out_value, double* out_comps4, double* out_grad_s);

/* Per-instance variant: s (n_inst x r_total), mu (n_inst x 3).  w <= 0 ->
 * 1/(n_inst*n_per_inst).  out_value = total; out_grad_s (n_inst x r_total). */
int lrnr_gpu_loss_grad_s_multi(lrnr_gpu_ctx* ctx, int model, const double* s, const double* mu,
                               double w, double* out_value, double* out_grad_s);

/* ---- full solve-step term set ----
 * lrnr_gpu_set_boundary: the boundary points of the following
 * lrnr_gpu_terms_grad calls, as in CollocationBatch::initial_x / periodic_t
 * (pde.hpp:29-40) or the classified points of the fast phase's sampling set X
 * (reduction.cpp:27-31: t == 0 -> initial x; x == 0 or 2pi -> periodic t).
 *
 * lrnr_gpu_terms_grad: one solve step's loss and dL/ds over every term kind, in
 * BatchGradResult form (training.hpp:189-195):
 *   interior   (points of lrnr_gpu_set_points, single instance): w_int N^2 | w_int |N|
 *   initial    w_ic (u(x,0) - sin x)^2        | w_ic |u(x,0) - sin x|
 *   periodic   w_bc (u(0,t) - u(2pi,t))^2      | w_bc |u(0,t) - u(2pi,t)|
 *   locality   lambda_local * sum ||s - s_init||_1   (when s_init != NULL)
 * objective LRNR_OBJ_SQUARED = the fine-tune PinnTermEmitter (training.cpp:286-327),
 * LRNR_OBJ_ABS = the fast-phase emitter (training.cpp:521-559; there the
 * reference weights are 1.0).  Weights <= 0 -> 1/n of that kind (safe_inv,
 * training.cpp:364-366).  out_comps = {residual, boundary, sparse (0), local}.
 * Boundary terms run a forward pass over the boundary points, then a seeded
 * reverse pass; |N| interior terms use the streaming kernel. */
#define LRNR_OBJ_SQUARED 0
#define LRNR_OBJ_ABS 1
int lrnr_gpu_set_boundary(lrnr_gpu_ctx* ctx, const double* initial_x, int64_t n_ic, const double* periodic_t,
                          int64_t n_bc);
int lrnr_gpu_terms_grad(lrnr_gpu_ctx* ctx, int model, const double* s, const double* mu, int objective, double w_int,
                        double w_ic, double w_bc, const double* s_init, double lambda_local, double* out_value,
                        double* out_comps, double* out_grad_s);

/* ---- solve loops on the device ----
 * lrnr_gpu_fine_tune: fine_tune (training.cpp:428-496) for the bound LRNR:
 * from s_init (= hyper_forward(mu, theta) in the reference), `epochs` epochs of
 * the PinnTermEmitter terms over a batch re-sampled every epoch exactly as
 * pde::sample_collocation(epoch_seed(seed, e), n_int, n_ic, n_bc) (bit-identical
 * host generator, double-buffered pinned upload overlapped with the device),
 * adam_step (autodiff.cpp:1062-1075, lr, beta 0.9/0.999, eps 1e-8),
 * project_nonnegative_coeffs and the best iterate, all on the device.
 * lrnr_gpu_fast_solve: fast_solve (training.cpp:498-607) for the bound
 * FastLRNR on the sampling set X (n_x points, classified as classify_point
 * does): the l1 terms + lambda_local ||s - s_init||_1, the divergence stop
 * (loss > 1e3 x the first loss), Adam + projection + best iterate; one epoch
 * is captured as a CUDA graph and replayed with no host synchronization.
 * Outputs: out_s = best coefficients (r_total), out_losses[e] = the epoch's
 * loss for the recorded epochs (capacity `epochs`), out_n_records, out_flags
 * (1 = aborted on a non-finite value, 2 = diverged), best loss / epoch.
 * Both overwrite the context's resident coefficients and keep its points. */
int lrnr_gpu_fine_tune(lrnr_gpu_ctx* ctx, const double* s_init, const double* mu, double lr, int64_t epochs,
                       int64_t n_int, int64_t n_ic, int64_t n_bc, uint64_t seed, double* out_s, double* out_best_loss,
                       int64_t* out_best_epoch, double* out_losses, int64_t* out_n_records, int* out_flags);
int lrnr_gpu_fast_solve(lrnr_gpu_ctx* ctx, const double* s_init, const double* mu, const double* X, int64_t n_x,
                        double lambda_local, double lr, int64_t epochs, double* out_s, double* out_best_loss,
                        int64_t* out_best_epoch, double* out_losses, int64_t* out_n_records, int* out_flags);

/* ---- evaluation: l1_relative_error (pde.cpp:166-178) on the device ----
 * u of `model` with coefficients s on the GridField grid x_i = 2 pi i / n_x,
 * t_j = j / n_t (j = 0..n_t; t = 0 when n_t = 0), against ref_values
 * ((n_t + 1) x n_x, row j = time): sum |u - ref| / sum |ref|. */
int lrnr_gpu_l1_error(lrnr_gpu_ctx* ctx, int model, const double* s, const double* ref_values, int64_t n_x,
                      int64_t n_t, double* out_l1);

/* ---- checkpoint interop (proj/src/checkpoint.cpp) ----
 * The reference's "LRNR" v1 file (named FP64 tensors + JSON meta), read and
 * written by host C++ (no JSON library). Getters take NULL arrays to query the
 * sizes first; flat layouts are those of lrnr_gpu_set_lrnr / _set_hyper /
 * _set_fast. Files written here load with the reference's checkpoint_load and
 * vice versa (tests/test_host.py). */
typedef struct lrnr_ckpt lrnr_ckpt;
const char* lrnr_ckpt_last_error(void);
/* An empty Checkpoint (checkpoint.hpp). */
int lrnr_ckpt_create(lrnr_ckpt** out);
/* checkpoint_load (checkpoint.cpp:127-161). */
int lrnr_ckpt_load(const char* path, lrnr_ckpt** out);
/* checkpoint_save (checkpoint.cpp:103-125). */
int lrnr_ckpt_save(const lrnr_ckpt* c, const char* path);
void lrnr_ckpt_free(lrnr_ckpt* c);
/* get_lrnr (checkpoint.cpp:174-186). */
int lrnr_ckpt_get_lrnr(const lrnr_ckpt* c, int* L, int64_t* widths, int64_t* ranks, int64_t* n_params, double* params);
/* put_lrnr (checkpoint.cpp:163-172). */
int lrnr_ckpt_put_lrnr(lrnr_ckpt* c, int L, const int64_t* widths, const int64_t* ranks, const double* params);
/* get_hyper (checkpoint.cpp:201-215). */
int lrnr_ckpt_get_hyper(const lrnr_ckpt* c, int* K, int64_t* hw, int64_t* n_params, double* params, double* lo3,
                        double* hi3);
/* put_hyper (checkpoint.cpp:188-199). */
int lrnr_ckpt_put_hyper(lrnr_ckpt* c, int K, const int64_t* hw, const double* params, int L_split,
                        const int64_t* split, const double* lo3, const double* hi3);
/* has_fast (checkpoint.cpp:231). */
int lrnr_ckpt_has_fast(const lrnr_ckpt* c);
/* get_fast (checkpoint.cpp:233-248). */
int lrnr_ckpt_get_fast(const lrnr_ckpt* c, int* L, int64_t* ranks, int64_t* red_ranks, int64_t* n_params,
                       double* params);
/* put_fast (checkpoint.cpp:217-229). */
int lrnr_ckpt_put_fast(lrnr_ckpt* c, int L, const int64_t* ranks, const int64_t* red_ranks, int64_t m_in,
                       int64_t m_out, const double* params);
/* get_sampling (checkpoint.cpp:282-288). */
int lrnr_ckpt_get_sampling(const lrnr_ckpt* c, int64_t* n, double* xt);
/* put_sampling (checkpoint.cpp:276-280). */
int lrnr_ckpt_put_sampling(lrnr_ckpt* c, int64_t n, const double* xt);

/* Hypernetwork-coupled step (BASELINE config 3; the emit_hyper + emit_fast_jet
 * composition of autodiff.cpp:883-922): s_i = hyper(mu_i) on device, the model
 * gradient per instance, then the hypernetwork VJP summed over instances.
 * mus (n_inst x 3).  Outputs: value, per-instance grad_s (n_inst x r_total, may
 * be NULL), grad_theta (hyper flat layout). */
int lrnr_gpu_hyper_loss_grad(lrnr_gpu_ctx* ctx, int model, const double* mus, double w,
                             double* out_value, double* out_grad_s, double* out_grad_theta);

/* Meta step (BASELINE config 4; PinnTermEmitter meta_mode interior terms,
 * training.cpp:283-293 with lambda_sparse = 0): gradient w.r.t. the LRNR bases
 * and biases AND the hypernetwork, in ParamPacker(BasesBiasesAndHyper) order.
 * mus (n_inst x 3).  Requires the LRNR model and the hypernetwork. */
int lrnr_gpu_meta_loss_grad(lrnr_gpu_ctx* ctx, const double* mus, double w, double* out_value,
                            double* out_grad);

/* meta_train's step with its regularizers (training.cpp:283-305, 368-389), on
 * the same resident points / mus as lrnr_gpu_meta_loss_grad:
 *   + lambda_sparse * w * sum_l banded_decay(s_l(mu), gamma) per interior term
 *     (Tape::banded_decay_penalty, autodiff.cpp:346-360) -> out_comps[2];
 *   + lambda_ortho * sum_l (||U_l^T U_l - I||_F^2 + ||V_l^T V_l - I||_F^2)
 *     (gram_ortho_penalty, autodiff.cpp:322-342; meta_train's grad() term)
 *     -> out_ortho.
 * plus the meta boundary terms when lrnr_gpu_set_meta_boundary set any -> out_comps[1].
 * out_value = interior + boundary + sparse + ortho (meta_train's `loss`), out_grad =
 * bg.grad + ro.grad in ParamPacker (BasesBiasesAndHyper) order. */
/* Meta-mode boundary points (PinnTermEmitter meta branch, training.cpp:307-327):
 * per instance i, n_ic initial x's (initial_x[i * n_ic + k]) and n_bc periodic
 * t's (periodic_t[i * n_bc + k]), evaluated with that instance's s = hyper(mu_i)
 * by the following lrnr_gpu_meta_terms_grad calls (n_inst must match the
 * interior points' instance count). Weights 1/(n_inst n_ic), 1/(n_inst n_bc)
 * (safe_inv over the batch, training.cpp:364-366). Pass 0 counts to clear. */
int lrnr_gpu_set_meta_boundary(lrnr_gpu_ctx* ctx, int64_t n_inst, const double* initial_x, int64_t n_ic,
                               const double* periodic_t, int64_t n_bc);
int lrnr_gpu_meta_terms_grad(lrnr_gpu_ctx* ctx, const double* mus, double w, double lambda_sparse, double gamma,
                             double lambda_ortho, double* out_value, double* out_comps, double* out_ortho,
                             double* out_grad);

/* ---- forward only ---- */
/* Output jets (u, u_x, u_t, u_xx) per point (jet_forward, model.cpp:357-405);
 * s (n_inst x r_total); out (n_points x 4). */
int lrnr_gpu_jets(lrnr_gpu_ctx* ctx, int model, const double* s, double* out_jets);
/* Interior loss only (loss_tune / loss_fast interior part, training.cpp:76-105). */
int lrnr_gpu_loss(lrnr_gpu_ctx* ctx, int model, const double* s, const double* mu, double w,
                  double* out_value);

/* ---- device-resident step (no host sync; for benchmarks and multi-GPU) ----
 * lrnr_gpu_upload_coeffs: s (n_inst x r_total) and mu (n_inst x 3) to device.
 * lrnr_gpu_run: launch the residual+gradient of `model` over the resident
 * points with the resident coefficients; writes n_inst rows of
 * [value, grad_s(r_total)] as double into dev_out (device pointer; NULL = the
 * context's own buffer).  Asynchronous on the context stream.
 * lrnr_gpu_check: synchronize and map a recorded non-finite term to
 * LRNR_ENONFINITE (+ layer tag). */
int lrnr_gpu_upload_coeffs(lrnr_gpu_ctx* ctx, const double* s, const double* mu, int64_t n_inst);
/* lrnr_gpu_run / _check / _download: run_batch_gradient (training.cpp:191-263) over resident
 * points and coefficients without host synchronization (multi-GPU steps, benchmarks). */
int lrnr_gpu_run(lrnr_gpu_ctx* ctx, int model, double w, double* dev_out);
int lrnr_gpu_check(lrnr_gpu_ctx* ctx);
/* Copy the context's result buffer (n_inst x (1 + r_total) doubles) to host. */
int lrnr_gpu_download(lrnr_gpu_ctx* ctx, double* host_out, int64_t n_doubles);

/* Achievable FMA-pipe rate of this device (dtype LRNR_F32 / LRNR_F64), TFLOP/s,
 * from a full-chip independent-chain FMA kernel; the roofline denominator. */
/* FP32 / FP64 FMA-chain microbenchmark: the roofline denominator (measurement aid; no reference
 * counterpart). */
int lrnr_gpu_fma_peak(lrnr_gpu_ctx* ctx, int dtype, double* out_tflops);

/* ---- multi-GPU: an NCCL communicator per context ----
 * The reference's only parallelism is run_batch_gradient's thread pool with a
 * fixed-order chunk combine (training.cpp:243-259). Here one process drives
 * one GPU through one context, each rank holds a shard of the points (or of
 * the PDE-parameter instances), and a context with a communicator attached
 * sums its results over the ranks with ncclAllReduce on the context stream,
 * after its own fixed-order reduction:
 *   lrnr_gpu_run / _loss_grad_s / _loss_grad_s_multi / _terms_grad / _loss /
 *   _loss_tune / _loss_fast / _loss_meta: value, comps and dL/ds rows summed
 *     (points sharded; the instance list is the same on every rank);
 *   lrnr_gpu_hyper_loss_grad: value and dL/dtheta summed, per-instance dL/ds
 *     rows stay local (instances sharded);
 *   lrnr_gpu_meta_loss_grad / _meta_terms_grad: value, comps and the packed
 *     bases + hypernetwork gradient summed (the Gram penalty, which depends on
 *     the bases only, is added once).
 * Default weights (w <= 0) become 1/n over every rank's terms. Every rank must
 * make the same sequence of calls (each may involve a collective). The solve
 * loops, jets, values and l1_error stay per-rank.
 * libnccl is loaded at run time (dlopen "libnccl.so.2"), so inside a process
 * that already mapped NCCL (PyTorch) that library is shared. */
/* ncclGetUniqueId into out_id (id_bytes >= 128). */
int lrnr_gpu_comm_unique_id(void* out_id, size_t id_bytes);
/* ncclCommInitRank(nranks, id, rank) on the context's device; the context owns it. */
int lrnr_gpu_comm_init(lrnr_gpu_ctx* ctx, int nranks, int rank, const void* id, size_t id_bytes);
/* Attach a caller-owned ncclComm_t (NULL detaches; the caller destroys it). */
int lrnr_gpu_set_comm(lrnr_gpu_ctx* ctx, void* nccl_comm);
/* Size and rank of the attached communicator (1, 0 without one). */
int lrnr_gpu_comm_info(const lrnr_gpu_ctx* ctx, int* nranks, int* rank);
/* In-place sum over the ranks of n device doubles on the context stream (e.g. a
 * caller's own lrnr_gpu_run output buffers). */
int lrnr_gpu_allreduce(lrnr_gpu_ctx* ctx, double* dev, int64_t n);

/* ---- plain losses and values, forward only (training.cpp:76-189, model.cpp:260-292) ----
 * out3 = LossBreakdown {total, residual, boundary} (training.hpp:82-86). Boundary
 * terms need u only and run the value-only (1-slot) forward; interior terms the
 * 4-slot jets. A non-finite total -> LRNR_ENONFINITE with layer tag -1, as the
 * reference's NonFiniteError(-1).
 * lrnr_gpu_values: lrnr_forward / fast_forward (u only) of `model` at n host
 *   (x, t) pairs with coefficients s (r_total) -> out_u (n).
 * lrnr_gpu_loss_tune: loss_tune (training.cpp:139-163): mean N^2 over the
 *   resident points (single instance) + mean (u(x,0) - sin x)^2 over the
 *   initial x + mean (u(0,t) - u(2pi,t))^2 over the periodic t of
 *   lrnr_gpu_set_boundary. model = LRNR_MODEL_FAST evaluates the same terms on
 *   the FastLRNR.
 * lrnr_gpu_loss_fast: loss_fast (training.cpp:165-189): SUMS of |N| at the
 *   interior points of the sampling set X (n_x (x, t) pairs, classified as
 *   classify_point, reduction.cpp:27-31), |u(x,0) - sin x| at its initial and
 *   |u(0,t) - u(2pi,t)| at its periodic points.
 * lrnr_gpu_loss_meta: loss_meta (training.cpp:109-137): per-instance mu
 *   (mus n_inst x 3) through the hypernetwork, s_i = hyper_forward(mu_i): mean
 *   N^2 over the resident points (n_inst groups) + the means over the meta
 *   boundary points of lrnr_gpu_set_meta_boundary. */
int lrnr_gpu_values(lrnr_gpu_ctx* ctx, int model, const double* s, const double* xt, int64_t n, double* out_u);
int lrnr_gpu_loss_tune(lrnr_gpu_ctx* ctx, int model, const double* s, const double* mu, double* out3);
int lrnr_gpu_loss_fast(lrnr_gpu_ctx* ctx, int model, const double* s, const double* mu, const double* X, int64_t n_x,
                       double* out3);
int lrnr_gpu_loss_meta(lrnr_gpu_ctx* ctx, const double* mus, double* out3);

/* ---- host-side setup (no GPU needed; reference reduction.cpp / model.cpp) ---- */
/* BASELINE config generator: make_lrnr_params(orthonormal,
 * bias 0) from Rng(seed), then b <- 0.1*normal(), s <- U[0,1] sorted descending. */
/* make_lrnr_params (model.cpp:454-504) + the BASELINE init recipe (b = 0.1 normal, s = U[0,1]
 * sorted descending), bit-identical streams (rng.hpp:13-44). */
int lrnr_host_make_baseline_model(int depth, const int64_t* widths, const int64_t* ranks,
                                  uint64_t seed, double* out_params, double* out_s);
/* make_hyper_params (model.cpp:480-504) from a fresh Rng(seed). */
int lrnr_host_make_hyper_params(int depth_split, const int64_t* split, int hidden_depth,
                                int hidden_width, uint64_t seed, double out_w_scale,
                                double out_bias, double* out_params);
/* sample_collocation interior points (pde.cpp:20-49), optional per-point mu. */
int lrnr_host_sample_collocation(uint64_t seed, int64_t n_interior, const double* mu_lo,
                                 const double* mu_hi, int with_mu, double* out_xt,
                                 double* out_mu);
/* training.cpp:20-26 and pde.cpp:20-49 (no mu): the fine_tune epoch batch. */
uint64_t lrnr_host_epoch_seed(uint64_t base, int64_t epoch);
int lrnr_host_sample_batch(uint64_t seed, int64_t n_int, int64_t n_ic, int64_t n_bc, double* out_xt,
                           double* out_ic_x, double* out_per_t);
/* FastLRNR construction: harvest_snapshots at SamplingSetX::uniform_grid(nx, nt)
 * with n_perturb Gaussian perturbations (sigma * extent), greedy EIM with budget
 * r_hat per inner layer, build_fastparams (reduction.cpp:10-31,111-283), for
 * n_mu coefficient vectors s (n_mu x r_total; the hyper_forward outputs).
 * out_indices ((L-1) x r_hat, -1 padded), out_red ((L-1)), out_fparams. */
int lrnr_host_build_fast(int depth, const int64_t* widths, const int64_t* ranks,
                         const double* params, int act, const double* s, int64_t n_mu,
                         int64_t nx, int64_t nt, int64_t n_perturb, double sigma, uint64_t seed,
                         int64_t r_hat, int64_t* out_red, int64_t* out_indices,
                         double* out_fparams, int* out_exhausted);

/* hyper_forward (model.cpp:294-318) for n_mu parameter vectors mus (n_mu x 3) -> out_s
 * (n_mu x hw[K]); bit-identical to the reference build (the mu-grid snapshot recipe of
 * harvest_snapshots evaluates it, reduction.cpp:111-148). */
int lrnr_host_hyper_forward(int n_layers, const int64_t* hw, const double* hparams, const double* box_lo,
                            const double* box_hi, int64_t n_mu, const double* mus, double* out_s);

/* SamplingSetX::uniform_grid (reduction.cpp:10-25): nx * nt (x, t) pairs, x fastest. */
int lrnr_host_uniform_grid(int64_t nx, int64_t nt, double* out_xt);
/* The columns harvest_snapshots evaluates (reduction.cpp:111-148): for each of
 * n_mu coefficient vectors and each of the n_sampling points, the point then
 * n_perturb Gaussian perturbations (sigma * extent, clamped), from the
 * reference's Rng stream bit-identically: n_mu * n_sampling * (1+n_perturb) pairs. */
int lrnr_host_harvest_points(const double* sampling_xt, int64_t n_sampling, int64_t n_mu, int64_t n_perturb,
                             double sigma, uint64_t seed, double* out_xt);
/* reduction::eim_greedy (reduction.cpp:150-238) on one m x n_cols row-major
 * snapshot matrix: out_idx (r_hat, -1 padded), out_xi (m x r_hat row-major,
 * zero padded), out_count = the basis size, out_exhausted. */
int lrnr_host_eim_greedy(int64_t m, int64_t n_cols, const double* snapshots, int64_t r_hat, int64_t* out_idx,
                         double* out_xi, int64_t* out_count, int* out_exhausted);
/* reduction::build_fastparams (reduction.cpp:240-283) from given EIM bases:
 * red (L-1), indices ((L-1) x r_hat), xi (per inner layer M_l x r_hat
 * row-major, concatenated) -> out_fparams (the lrnr_host_build_fast layout). */
int lrnr_host_build_fastparams(int depth, const int64_t* widths, const int64_t* ranks, const double* params,
                               int act, int64_t r_hat, const int64_t* red, const int64_t* indices,
                               const double* xi, double* out_fparams);

/* Q-DEIM index selection (BASELINE.json configs[1]: "indices from pivoted QR of U^l";
 * SURVEY.md Appendix A.3).  The reference selects by greedy EIM on harvested snapshots
 * (reduction.cpp:176-232) and has no pivoted-QR mode, so only the selection is new:
 * lrnr_host_qdeim returns the rows a column-pivoted QR of xi^T picks (xi m x r row-major;
 * largest residual norm first, lowest index on ties; out_idx r entries, -1 padded,
 * out_count = rank found).  lrnr_host_build_fast_qdeim builds, per inner layer,
 * EimBasis{xi = U^l, indices = qdeim(U^l)} with r_hat_l = r_l and runs the reference's
 * build_fastparams (reduction.cpp:240-283) on it; r_hat >= max r_l sizes out_indices
 * ((L-1) x r_hat, -1 padded).  Outputs as lrnr_host_build_fast. */
int lrnr_host_qdeim(int64_t m, int64_t r, const double* xi, int64_t* out_idx, int64_t* out_count);
int lrnr_host_build_fast_qdeim(int depth, const int64_t* widths, const int64_t* ranks, const double* params,
                               int act, int64_t r_hat, int64_t* out_red, int64_t* out_indices,
                               double* out_fparams);

/* ---- FastLRNR construction on the device ---------
 * lrnr_gpu_eim_greedy replaces reduction::eim_greedy (reduction.cpp:150-238):
 * the residual sweep over all snapshot columns runs on the device, one thread
 * per column, in the reference's FP64 operation order (the x86-64-v3 build
 * contracts a*b+c to FMA; so does this), so indices and basis columns are
 * bit-identical to lrnr_host_eim_greedy on the same snapshots. Same outputs.
 * lrnr_gpu_build_fast replaces harvest_snapshots + eim_greedy +
 * build_fastparams (reduction.cpp:111-283; lrnr_host_build_fast's signature
 * plus ctx): the hidden-state harvest is a device forward pass (activation
 * values may differ from libm in the last ulp), every inner layer's greedy
 * sweep runs concurrently on the device, and the O(r_hat^2 r) assembly of the
 * reduced matrices runs on the host.
 * lrnr_gpu_harvest_snapshots is reduction::harvest_snapshots alone, for any
 * SamplingSetX (sampling_xt, n_sampling points): the inner layers' M_l x n_cols
 * snapshot blocks (row-major, concatenated) to the host. */
int lrnr_gpu_harvest_snapshots(lrnr_gpu_ctx* ctx, int depth, const int64_t* widths, const int64_t* ranks,
                               const double* params, int act, const double* s, int64_t n_mu,
                               const double* sampling_xt, int64_t n_sampling, int64_t n_perturb, double sigma,
                               uint64_t seed, double* out_snapshots);
int lrnr_gpu_eim_greedy(lrnr_gpu_ctx* ctx, int64_t m, int64_t n_cols, const double* snapshots, int64_t r_hat,
                        int64_t* out_idx, double* out_xi, int64_t* out_count, int* out_exhausted);
int lrnr_gpu_build_fast(lrnr_gpu_ctx* ctx, int depth, const int64_t* widths, const int64_t* ranks,
                        const double* params, int act, const double* s, int64_t n_mu, int64_t nx, int64_t nt,
                        int64_t n_perturb, double sigma, uint64_t seed, int64_t r_hat, int64_t* out_red,
                        int64_t* out_indices, double* out_fparams, int* out_exhausted);

#ifdef __cplusplus
}
#endif

#endif /* LRNR_GPU_H */
