/*
 * afg.h - C ABI of the B200 (sm_100a) operator kernels behind the AffineForge
 * graph/operator API.
 *
 * The reference executes every operator nest in its CPU interpreter
 * (af::interpret, /root/reference/proj/include/af/interp.h:97-100, hot loop
 * proj/src/interp.cpp:440-561). Each entry point below replaces the
 * interpretation of one operator (or one fused operator chain) of a lowered
 * graph (proj/src/frontend.cpp:975 lowerGraphToAffine):
 *
 *   afg_gemm              <- lowerMatmul            frontend.cpp:679-733
 *                            + broadcast_in_dim/add/max epilogue nests
 *                              (frontend.cpp:447-500), fused before the store
 *   afg_gemm_batched      <- batch_matmul lowering  frontend.cpp:679-733
 *   afg_conv2d_nhwc       <- lowerConv              frontend.cpp:752-970 as the
 *                            implicit GEMM of SPEC.md:388-452 (conv_gemm.cpp
 *                            is a stub in the reference)
 *   afg_conv2d_nchw       <- lowerConv, direct (general stride/dilation/
 *                            padding/transposed, frontend.cpp:764-904)
 *   afg_attention_fwd     <- transpose->batch_matmul->add->softmax->batch_matmul
 *                            (test_frontend.cpp:275-305; SPEC.md:454-529,
 *                            attention.cpp is a stub in the reference)
 *   afg_softmax_lastdim   <- lowerSoftmax           frontend.cpp:564-625
 *   afg_layernorm_residual<- (no reference op; additive extension)
 *   afg_elementwise       <- lowerElementwiseBinary frontend.cpp:447-459, exp
 *   afg_reduce_lastdim    <- lowerReduceShaped      frontend.cpp:628-675
 *   afg_gemm_i8           <- quant repositioning    SPEC.md:531-572 (quant.cpp
 *                            is a stub): i8 x i8 -> i32 matmul + requant
 *   afg_conv2d_nhwc_i8    <- quant repositioning of lowerConv (frontend.cpp:
 *                            752-970) as an i8 implicit GEMM + requant
 *
 * Conventions
 *  - All tensor pointers are caller-owned DEVICE pointers, dense row-major
 *    unless a leading dimension is given. No entry point allocates device
 *    memory, except the tensor-map cache which is host-side only.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream). Every call is
 *    stream-ordered and asynchronous; errors in argument validation are
 *    reported synchronously, kernel faults surface at the next sync.
 *  - No C++ exception crosses this boundary. Failures return a status and set
 *    a thread-local message readable with afg_last_error() (the reference
 *    reports GraphError / InterpError, frontend.h:26-28, interp.h:29-31).
 *  - There is no CPU fallback: without a usable sm_100 device every compute
 *    entry point returns AFG_ERR_CUDA.
 */
#ifndef AFG_H
#define AFG_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define AFG_API __attribute__((visibility("default")))
#else
#define AFG_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum afg_status {
  AFG_OK = 0,
  AFG_ERR_INVALID_ARG = 1, /* shape / pointer / alignment contract violated */
  AFG_ERR_UNSUPPORTED = 2, /* valid request this build has no kernel for      */
  AFG_ERR_CUDA = 3,        /* CUDA runtime / driver error, or no sm_100 device */
  AFG_ERR_NCCL = 4,
  AFG_ERR_INTERNAL = 5
} afg_status;

/* Element types. F32/F16 mirror af::ElementType (ir.h:29); BF16 is the
 * additive extension the BASELINE configs need (the reference carries bf16
 * values in f32 tensors). */
typedef enum afg_dtype { AFG_F32 = 0, AFG_F16 = 1, AFG_BF16 = 2 } afg_dtype;

/* y = act(acc + bias[n]); NONE ignores bias. */
typedef enum afg_epilogue {
  AFG_EPI_NONE = 0,
  AFG_EPI_BIAS = 1,
  AFG_EPI_BIAS_RELU = 2,      /* max(acc + bias, 0): the graph's max(x, zeros) */
  AFG_EPI_BIAS_GELU_TANH = 3, /* x * sigmoid(2u), u = sqrt(2/pi)(x + .044715x^3) */
  AFG_EPI_BIAS_GELU_ERF = 4   /* 0.5 x (1 + erf(x / sqrt 2)) (BERT)              */
} afg_epilogue;

/* Storage of the B operand of a GEMM. The reference matmul is A[M,K] x B[K,N]
 * (frontend.cpp:679-733), i.e. AFG_B_KN. AFG_B_NK stores B transposed
 * ([N,K] row-major, e.g. packed conv filters / linear weights). */
typedef enum afg_layout { AFG_B_KN = 0, AFG_B_NK = 1 } afg_layout;

typedef enum afg_binop {
  AFG_OP_ADD = 0,
  AFG_OP_SUB = 1,
  AFG_OP_MUL = 2,
  AFG_OP_MAX = 3,
  AFG_OP_EXP = 4 /* unary: b ignored */
} afg_binop;

typedef enum afg_reduce_kind {
  AFG_REDUCE_SUM = 0,
  AFG_REDUCE_MAX = 1,
  AFG_REDUCE_MAXABS = 2 /* max |x| (NaN-propagating) */
} afg_reduce_kind;

/* ------------------------------------------------------------ runtime --- */

AFG_API const char* afg_last_error(void);
AFG_API const char* afg_version(void);
/* Number of visible devices with compute capability 10.x (0 if none). */
AFG_API int afg_device_count(void);
/* Number of afg kernel launches issued by this process so far (all entry
 * points, all devices); bench.py uses it to report gpu_launches. */
AFG_API uint64_t afg_launch_count(void);

/* ------------------------------------------------------------ GEMM (K1) --- */

/* C[M,N] = epi(A[M,K] . B + bias) (+ residual[M,N]).
 *  - ab_dtype BF16/F16: tcgen05 tensor-core kernel, fp32 accumulation in TMEM.
 *    Requires lda, ldb multiples of 8 elements and 16-byte aligned A, B;
 *    other shapes run the SIMT kernel.
 *  - ab_dtype F32: fp32 SIMT kernel (FFMA, fp32 accumulation).
 *  - c_dtype may differ from ab_dtype; bias is fp32 [N] (may be NULL only if
 *    epi == AFG_EPI_NONE); residual has c_dtype and leading dimension ldc.
 * Leading dimensions are in elements. */
AFG_API afg_status afg_gemm(const void* A, int64_t lda, const void* B, int64_t ldb,
                    const float* bias, const void* residual, void* C, int64_t ldc,
                    int64_t M, int64_t N, int64_t K, afg_dtype ab_dtype, afg_dtype c_dtype,
                    afg_layout b_layout, afg_epilogue epi, void* stream);

/* Strided-batched C_b = A_b . B_b (batch_matmul, frontend.cpp:679-733 with
 * batch dims): all operands dense row-major [batch, rows, cols], B is
 * [batch, K, N]. No epilogue. */
AFG_API afg_status afg_gemm_batched(const void* A, const void* B, void* C, int64_t batch,
                            int64_t M, int64_t N, int64_t K, afg_dtype ab_dtype,
                            afg_dtype c_dtype, void* stream);

/* ------------------------------------------------------------ conv (K2) --- */

/* Implicit-GEMM convolution, NHWC activations:
 *   x [B,H,W,C], w [OC,KH,KW,C] (K-major filter), y [B,OH,OW,OC]
 *   y = epi(conv(x, w) + bias)
 * GEMM view: M = B*OH*OW, N = OC, K = KH*KW*C. Explicit
 * asymmetric-capable padding: input row iy = oy*stride_h + ky*dil_h - pad_top.
 * dtype BF16/F16 (tensor cores; C % 64 == 0 for the TMA path) or F32. */
AFG_API afg_status afg_conv2d_nhwc(const void* x, const void* w, const float* bias, void* y,
                           int64_t B, int64_t H, int64_t W, int64_t C, int64_t OC,
                           int64_t KH, int64_t KW, int64_t stride_h, int64_t stride_w,
                           int64_t pad_top, int64_t pad_left, int64_t dil_h,
                           int64_t dil_w, int64_t OH, int64_t OW, afg_dtype dtype,
                           afg_epilogue epi, void* stream);

/* afg_conv2d_nhwc with an explicit output type: x / w in `dtype`, y in
 * `y_dtype` (F32 keeps the fp32 accumulator unrounded; the graph executor's
 * f32-declared NHWC conv chains use it). */
AFG_API afg_status afg_conv2d_nhwc_ex(const void* x, const void* w, const float* bias, void* y,
                              int64_t B, int64_t H, int64_t W, int64_t C, int64_t OC,
                              int64_t KH, int64_t KW, int64_t stride_h, int64_t stride_w,
                              int64_t pad_top, int64_t pad_left, int64_t dil_h,
                              int64_t dil_w, int64_t OH, int64_t OW, afg_dtype dtype,
                              afg_dtype y_dtype, afg_epilogue epi, void* stream);

/* Direct convolution in the reference's own NCHW/OIHW layout (and IOHW for
 * transposed), exactly the semantics of frontend.cpp:752-970 / the oracle
 * convReference (oracles.cpp:78-120), fp32 accumulate. pad_* are the begin
 * pads of convGeometry (frontend.cpp:115-149). */
AFG_API afg_status afg_conv2d_nchw(const void* x, const void* w, void* y, int64_t B, int64_t C,
                           int64_t H, int64_t W, int64_t OC, int64_t KH, int64_t KW,
                           int64_t stride_h, int64_t stride_w, int64_t dil_h,
                           int64_t dil_w, int64_t pad_top, int64_t pad_left,
                           int transposed, int64_t OH, int64_t OW, afg_dtype x_dtype,
                           afg_dtype y_dtype, void* stream);

/* OIHW -> OHWI filter repack for afg_conv2d_nhwc. */
AFG_API afg_status afg_conv_pack_filter(const void* w_oihw, void* w_ohwi, int64_t OC, int64_t C,
                                int64_t KH, int64_t KW, afg_dtype dtype, void* stream);

/* ------------------------------------------------------- attention (K3) --- */

/* o = softmax(scale * q k^T + bias [+ causal mask]) v, per (b, h):
 *   q [B,H,Nq,D], k/v [B,H,Nk,D], o [B,H,Nq,D], bias [B,H,Nq,Nk] fp32 or NULL.
 * causal: key j is masked for j > i (the -inf additive bias of SURVEY.md §8a8).
 * The reference has no scale (scale = 1 reproduces it). dtype F16/BF16 runs
 * the tcgen05 flash kernel (D in {64,128}); F32 runs the SIMT kernel.
 * Output dtype o_dtype (F32 keeps the reference's unrounded output). */
AFG_API afg_status afg_attention_fwd(const void* q, const void* k, const void* v,
                             const float* bias, void* o, int64_t B, int64_t H,
                             int64_t Nq, int64_t Nk, int64_t D, float scale, int causal,
                             afg_dtype dtype, afg_dtype o_dtype, void* stream);

/* Same with explicit element strides {seq, head, batch} for q, k, v and o
 * (head_dim contiguous), e.g. reading Q/K/V straight out of a fused
 * [B, S, 3, H, D] QKV projection and writing O as [B, S, H, D] (BERT).
 * Tensor-core path only (f16/bf16, D in {64,128}, strides multiples of 8). */
AFG_API afg_status afg_attention_fwd_strided(const void* q, const void* k, const void* v,
                                     const float* bias, void* o, int64_t B, int64_t H,
                                     int64_t Nq, int64_t Nk, int64_t D, float scale, int causal,
                                     afg_dtype dtype, afg_dtype o_dtype, const int64_t* q_strides,
                                     const int64_t* k_strides, const int64_t* v_strides,
                                     const int64_t* o_strides, void* stream);

/* ------------------------------------------------- memory-bound chains --- */

/* Row softmax over the last axis (frontend.cpp:564-625 / oracles.cpp:175-190). */
AFG_API afg_status afg_softmax_lastdim(const void* x, void* y, int64_t rows, int64_t cols,
                               afg_dtype x_dtype, afg_dtype y_dtype, void* stream);

/* y = layernorm(x + residual) * gamma + beta over the last axis, biased
 * variance, fp32 statistics. residual may be NULL. Also writes the sum
 * x + residual to `sum_out` when non-NULL. */
AFG_API afg_status afg_layernorm_residual(const void* x, const void* residual, const float* gamma,
                                  const float* beta, void* y, void* sum_out, int64_t rows,
                                  int64_t cols, float eps, afg_dtype dtype, void* stream);

/* out = op(a, b) elementwise over n elements; b may be broadcast along the
 * last axis when b_period > 0 (b[i % b_period]). */
AFG_API afg_status afg_elementwise(const void* a, const void* b, void* out, int64_t n,
                           int64_t b_period, afg_binop op, afg_dtype a_dtype,
                           afg_dtype b_dtype, afg_dtype out_dtype, void* stream);

/* out[r] = reduce(x[r, 0:cols]) */
AFG_API afg_status afg_reduce_lastdim(const void* x, void* out, int64_t rows, int64_t cols,
                              afg_reduce_kind kind, afg_dtype x_dtype, afg_dtype out_dtype,
                              void* stream);

/* y = x broadcast into `out_shape`: input dim d maps to output dim dims[d]
 * (broadcast_in_dim, frontend.cpp:489-500). */
AFG_API afg_status afg_broadcast_in_dim(const void* x, void* y, int in_rank, const int64_t* in_shape,
                                int out_rank, const int64_t* out_shape, const int64_t* dims,
                                afg_dtype x_dtype, afg_dtype y_dtype, void* stream);

/* int8 GEMM (quant module: the repositioned
 * dequant(Qa) . dequant(Qb) -> quant pattern; K1c, tcgen05 kind::i8).
 * A: i8 [M,K] row-major (pitch lda bytes); B: i8 [N,K] row-major (K-major,
 * pitch ldb bytes; the reference's [K,N] operand transposed once, e.g. with
 * afg_transpose); exact i32 accumulation (K < 131072). out_mode:
 *  0: C i32 [M,N] = A . B^T                     (bit-exact integer matmul)
 *  1: C i8  = clamp(round_half_away(acc * scale), -128, 127)   (requantise)
 *  2: C f32 = (float)(acc * scale)                            (dequantise)
 * with scale = s_a * s_b (/ s_out for mode 1), applied in double. ldc in
 * elements of C. A / B need 16-byte aligned bases and pitches. */
AFG_API afg_status afg_gemm_i8(const void* A, int64_t lda, const void* B, int64_t ldb, void* C,
                               int64_t ldc, int64_t M, int64_t N, int64_t K, int out_mode,
                               float scale, void* stream);

/* int8 implicit-GEMM convolution (the conv half of the quant path; K1c on
 * TMA im2col): x i8 NHWC [B,H,W,C], w i8 OHWI [OC,KH,KW,C], output NHWC
 * [B*OH*OW, OC] as afg_gemm_i8's out_mode / scale (i32 exact, requantised i8,
 * dequantised f32). C % 16 == 0; explicit pad_top / pad_left (the far-side
 * padding follows from OH / OW), stride / dilation as afg_conv2d_nhwc. */
AFG_API afg_status afg_conv2d_nhwc_i8(const void* x, const void* w, void* y, int64_t B, int64_t H,
                                      int64_t W, int64_t C, int64_t OC, int64_t KH, int64_t KW,
                                      int64_t stride_h, int64_t stride_w, int64_t pad_top,
                                      int64_t pad_left, int64_t dil_h, int64_t dil_w, int64_t OH,
                                      int64_t OW, int out_mode, float scale, void* stream);

/* Quantisation chain (interp.cpp quant/dequant; oracles.cpp:387-398):
 *  mode 0 quantize  : y = clamp(round_half_away(x / scale), -128, 127)
 *  mode 1 dequantize: y = x * scale
 *  mode 2 / 3       : y = saturate(nearbyint(x)) to i8 / i32 (roundToType)
 * Integer-typed tensors are carried exactly in f32 storage. */
AFG_API afg_status afg_quantize(const void* x, void* y, int64_t n, float scale, int mode,
                        afg_dtype x_dtype, afg_dtype y_dtype, void* stream);

/* The GEMM epilogue as a standalone pass over an accumulator tile:
 * out[r, c] = act(acc[r, c] + bias[c]) (+ residual[r, c]), rows x cols,
 * row pitch ld for acc / residual / out. Used after a split-K reduction
 * (the fp32 partial sums are reduced across GPUs, then finished here). */
AFG_API afg_status afg_epilogue_apply(const void* acc, const float* bias, const void* residual,
                              void* out, int64_t rows, int64_t cols, int64_t ld,
                              afg_epilogue epi, afg_dtype acc_dtype, afg_dtype out_dtype,
                              void* stream);

/* Dtype conversion (RNE), used by the graph executor's host staging. */
AFG_API afg_status afg_convert(const void* x, void* y, int64_t n, afg_dtype x_dtype,
                       afg_dtype y_dtype, void* stream);

/* General permutation of a dense tensor (rank <= 6): y = transpose(x, perm). */
AFG_API afg_status afg_transpose(const void* x, void* y, int rank, const int64_t* shape,
                         const int64_t* perm, afg_dtype dtype, void* stream);

/* Deterministic synthetic inputs on device: x[i] = lo + u_i (hi - lo),
 * u_i from splitmix64(seed, i), rounded (RNE) to `dtype`. */
AFG_API afg_status afg_fill_uniform(void* x, int64_t n, uint64_t seed, float lo, float hi,
                            afg_dtype dtype, void* stream);

/* ------------------------------------------------ multi-GPU (NVLink) --- */

/* NCCL communicators (libnccl.so.2 resolved at first use). One per rank via
 * a unique id (128 bytes) shared out of band, or all of a process's devices
 * at once (ncclCommInitAll). `comm` values are ncclComm_t. */
AFG_API afg_status afg_comm_unique_id(void* id_out /* 128 bytes */);
AFG_API afg_status afg_comm_init_rank(void** comm, int world, const void* id, int rank);
AFG_API afg_status afg_comm_init_all(void** comms, int ndev, const int* devices);
AFG_API afg_status afg_comm_destroy(void* comm);

/* Split-K / tensor-parallel (row-parallel) GEMM, the one BASELINE config with
 * an exchange step: every rank holds A[:, K_r] ([M, K_local])
 * and B[K_r, :], computes its fp32 partial product on the tensor cores, the
 * partials are summed across ranks over NVLink by NCCL, and the epilogue
 * (bias / ReLU / GELU) runs on the sum:
 *   AFG_SPLITK_REDUCE_SCATTER: C = rows [rank*M/P, (rank+1)*M/P) of the
 *                              result ([M/P, N], M % P == 0);
 *   AFG_SPLITK_ALL_REDUCE    : C = the full [M, N] result on every rank.
 * workspace: device memory of afg_gemm_splitk_workspace(M, N, P, mode) bytes. */
#define AFG_SPLITK_REDUCE_SCATTER 0
#define AFG_SPLITK_ALL_REDUCE 1
AFG_API size_t afg_gemm_splitk_workspace(int64_t M, int64_t N, int world, int mode);
AFG_API afg_status afg_gemm_splitk(const void* A, int64_t lda, const void* B, int64_t ldb,
                                   const float* bias, void* C, int64_t ldc, int64_t M, int64_t N,
                                   int64_t K_local, afg_dtype ab_dtype, afg_dtype c_dtype,
                                   afg_layout b_layout, afg_epilogue epi, void* comm, int mode,
                                   void* workspace, size_t workspace_bytes, void* stream);

/* Thread-per-device group (include/afg_multi.h): one host thread per device,
 * each with its own stream and (for > 1 device) NCCL communicator.
 * afg_group_run calls fn(user, rank, device, stream, comm) on every device's
 * thread concurrently, then waits for all streams; the first failing status
 * is returned. */
typedef struct afg_group afg_group;
typedef afg_status (*afg_group_fn)(void* user, int rank, int device, void* stream, void* comm);
AFG_API afg_status afg_group_create(int ndev, const int* devices, afg_group** out);
AFG_API void afg_group_destroy(afg_group* g);
AFG_API int afg_group_size(const afg_group* g);
AFG_API afg_status afg_group_run(afg_group* g, afg_group_fn fn, void* user);

/* --------------------------------------------------- encoder layer (BERT) --- */

/* One post-LN transformer encoder layer (BERT-base: hidden 768, 12 heads,
 * ffn 3072), x/y [batch*seq, hidden]; weights in the reference matmul layout
 * W[K,N] (afg_gemm AFG_B_KN); biases / LN params fp32. Seven stream-ordered
 * launches (see csrc/encoder.cpp); no allocation: `workspace` must hold
 * afg_encoder_layer_workspace(...) bytes. */
AFG_API size_t afg_encoder_layer_workspace(int64_t batch, int64_t seq, int64_t hidden,
                                           int64_t ffn, afg_dtype dtype);
AFG_API afg_status afg_encoder_layer_fwd(
    const void* x, void* y, int64_t batch, int64_t seq, int64_t hidden, int64_t heads,
    int64_t ffn, const void* w_qkv, const float* b_qkv, const void* w_o, const float* b_o,
    const float* ln1_g, const float* ln1_b, const void* w_1, const float* b_1, const void* w_2,
    const float* b_2, const float* ln2_g, const float* ln2_b, float eps, afg_dtype dtype,
    void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------ graph executor --- */

/* The drop-in for the reference's parseGraphJson -> lowerGraphToAffine ->
 * interpret path (frontend.cpp:57-113, :975; interp.cpp:690-696) for callers
 * that cannot use the C++ API of afg_graph.h: executes the graph JSON on the
 * current device with the given host inputs (values as doubles, keyed by
 * tensor id with or without '%'; rounded to the declared element type on
 * upload like the interpreter, interp.cpp:212-213) and returns the outputs
 * keyed "%id" as doubles. flags: AFG_GRAPH_FUSE enables the kernel patterns
 * and fused regions; AFG_GRAPH_EXACT keeps f32 tensors off the tensor cores
 * (bit-exact paths only).
 * GraphError -> AFG_ERR_INVALID_ARG, InterpError -> AFG_ERR_CUDA. */
#define AFG_GRAPH_FUSE 1
#define AFG_GRAPH_EXACT 2
typedef struct afg_graph_result afg_graph_result;
AFG_API afg_status afg_graph_run(const char* graph_json, int n_inputs, const char* const* names,
                         const double* const* data, const int64_t* numel, int flags,
                         void* stream, afg_graph_result** out);
/* The same, sharded over devices[0..ndev) (entries may repeat a device): one
 * host thread per shard, the leading extent shard_extent (0: the first
 * input's) split into contiguous blocks and propagated through the graph;
 * GraphError if the graph mixes rows across shards (afg_graph.h GpuOptions). */
AFG_API afg_status afg_graph_run_sharded(const char* graph_json, int n_inputs,
                                         const char* const* names, const double* const* data,
                                         const int64_t* numel, int flags, int ndev,
                                         const int* devices, int64_t shard_extent,
                                         afg_graph_result** out);
AFG_API int afg_graph_result_count(const afg_graph_result* r);
AFG_API const char* afg_graph_result_name(const afg_graph_result* r, int i);
AFG_API int afg_graph_result_rank(const afg_graph_result* r, int i);
AFG_API int64_t afg_graph_result_dim(const afg_graph_result* r, int i, int d);
AFG_API int64_t afg_graph_result_numel(const afg_graph_result* r, int i);
AFG_API const double* afg_graph_result_data(const afg_graph_result* r, int i);
/* One line per launched kernel (group): what the planner fused. */
AFG_API const char* afg_graph_result_plan(const afg_graph_result* r);
AFG_API void afg_graph_result_free(afg_graph_result* r);
/* Graph JSON read + validation only (GraphError -> AFG_ERR_INVALID_ARG). */
AFG_API afg_status afg_graph_check_json(const char* graph_json);

#ifdef __cplusplus
}
#endif

#endif /* AFG_H */
