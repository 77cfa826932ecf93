/*
 * pp200.h -- C-ABI of libpp200.so, the B200 (sm_100a) compute and transport
 * library behind the pipeline runtime in paper_2412_14374_b200.
 *
 * The reference (pipecraft, /root/reference/pkg) has no native code: its
 * "kernels" are numpy expressions inside the op interpreter
 *   eval_op        pkg/src/pipecraft/executor.py:59-96
 * and its transport is the in-process FIFO
 *   Channel        pkg/src/pipecraft/executor.py:201-254
 * driven by the per-actor interpreter
 *   _worker/_run_task  pkg/src/pipecraft/executor.py:316-384.
 * Every entry point below replaces one of those numpy expressions or Channel
 * methods; the comment on each cites the reference line it stands in for.
 *
 * Conventions
 *  - All pointers are device pointers owned by the caller (e.g. torch tensors'
 *    data_ptr()).  `stream` is a cudaStream_t passed as void*.
 *  - Every call is stream-ordered, allocates nothing, never synchronises the
 *    host, and returns PC_OK (0) or an error code; the message is available
 *    from pc_last_error() on the calling thread.
 *  - Matrices are row-major.  transA/transB follow numpy: C = op(A) @ op(B)
 *    with op(X) = X.T when trans is 1 (the reference's explicit `transpose`
 *    ops, executor.py:78-79, become operand majors, never copies).
 */
#ifndef PP200_H
#define PP200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum pc_status {
  PC_OK = 0,
  PC_ERR_ARG = 1,
  PC_ERR_CUDA = 2,
  PC_ERR_NCCL = 3,
  PC_ERR_UNSUPPORTED = 4
};

enum pc_dtype { PC_F32 = 0, PC_F64 = 1, PC_BF16 = 2, PC_I32 = 3 };

/* GEMM epilogue flags (combinable where meaningful). */
#define PC_EPI_BIAS 1       /* acc += bias[n] (fp32 vector)                       */
#define PC_EPI_GELU 2       /* aux_out = acc; C = gelu_tanh(acc)                  */
#define PC_EPI_RESIDUAL 4   /* C = acc + aux[m,n]                                 */
#define PC_EPI_GELU_GRAD 8  /* C = acc * gelu_tanh'(aux[m,n])                     */
#define PC_EPI_ACCUM 16     /* C += acc (fp32 C; in-place gradient accumulation)  */
#define PC_EPI_RELU 32      /* aux_out = acc; C = max(acc, 0)  (executor.py:70-71) */
#define PC_EPI_RELU_GRAD 64 /* C = acc * (aux[m,n] > 0)        (executor.py:89-90) */
#define PC_EPI_SPLITK_ZERO_C 128 /* caller guarantees an fp32 C filled with zeros: the
                                    kernel may split K in two halves reduce-added into C
                                    (deterministic: two terms onto 0 commute) */
#define PC_EPI_SPLITK_ORDERED 256 /* with PC_EPI_ACCUM: the kernel may split K in 2 or 4
                                    parts added onto C in a fixed order, ((C + h0) + h1)..,
                                    sequenced per tile by flags: aux = zeroed uint32 flag
                                    array, ldaux = its length (>= tiles x 16) */

const char* pc_last_error(void);
int pc_version(void);
int pc_device_sm_count(void);

/* C[M,N] = op(A)[M,K] @ op(B)[K,N] with epilogue.  Replaces `a @ b`
 * (executor.py:66-67).  dtype_in: PC_BF16 (tcgen05/TMEM/TMA path, fp32
 * accumulate), PC_F32 (FFMA), PC_F64 (DFMA).  dtype_out: same as input, or
 * PC_F32 for bf16 inputs.  aux/aux_out have C's dtype. */
int pc_gemm(int dtype_in, int dtype_out, int transA, int transB, int64_t M, int64_t N, int64_t K,
            const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
            int epilogue, const void* bias, const void* aux, int64_t ldaux, void* aux_out,
            int64_t ldaux_out, void* stream);

/* The tcgen05 tile choice pc_gemm makes for a bf16 problem (transB as pc_gemm; split_ok:
 * 0 = no split allowed, 1 = PC_EPI_SPLITK_ZERO_C with fp32 C (K split 1 or 2),
 * 2 = PC_EPI_ACCUM | PC_EPI_SPLITK_ORDERED (1 or 2)): tile width, CTA pair (1 or 2),
 * K split. */
/* Two weight gradients in one launch (the attention-output and qkv weights of a
 * block share N = d_model and K = tokens): C1 (+)= A1^T B1 [M1 x N] and
 * C2 (+)= A2^T B2 [M2 x N], A / B stored [K, M] / [K, N] bf16 (MN-major), C fp32,
 * epilogue PC_EPI_ACCUM | PC_EPI_SPLITK_ORDERED (aux = zeroed flag array) or
 * PC_EPI_SPLITK_ZERO_C.  M1 must fill whole tiles (a multiple of 256).  Replaces two
 * `matmul`s of the accumulation chain (executor.py:66-67) with the same sums. */
int pc_gemm_wgrad_pair(int64_t M1, int64_t M2, int64_t N, int64_t K, const void* A1, int64_t lda1,
                       const void* B1, int64_t ldb1, float* C1, int64_t ldc1, const void* A2,
                       int64_t lda2, const void* B2, int64_t ldb2, float* C2, int64_t ldc2,
                       int epilogue, void* aux, int64_t ldaux, void* stream);
int pc_gemm_tile_choice(int transB, int64_t M, int64_t N, int64_t K, int split_ok, int* bn,
                        int* cta_pair, int* ksplit);
/* Force the tcgen05 GEMM tile width (0 = heuristic, else 64/128/192/256). Test hook. */
int pc_gemm_set_tile_n(int bn);
/* CTA-pair (cta_group::2, 256-row tiles over two SMs) selection: 0 = heuristic,
 * 1 = never, 2 = whenever the tile allows it (128/256; 192 with a K-major B).  Test hook. */
/* Largest K split the tile chooser may pick (1, 2, 4, 8; default 4).  Tuning hook. */
int pc_gemm_set_max_split(int ks);
int pc_gemm_set_cta_pair(int mode);
/* Profiling ablation of the tcgen05 GEMM (outputs are garbage while set):
 * bit0 = skip the epilogue work, bit1 = skip the operand TMA loads, bit2 = skip the
 * epilogue's aux-input TMA loads. */
int pc_gemm_set_ablation(int bits);
/* 1 (default) = write C through smem + TMA bulk store when legal; 0 = direct stores. Test hook. */
int pc_gemm_set_tma_store(int on);

/* ---- elementwise / reductions (executor.py:59-96 numpy expressions) ---- */
enum pc_ewise_op {
  PC_EW_ADD = 1,      /* out = a + b      ("add", executor.py:68-69; grad-merge add :335-336) */
  PC_EW_MUL = 2,      /* out = a * b      ("scale"/"mul", :76-77, :86-87); b_n==1 broadcasts */
  PC_EW_RELU = 3,     /* out = max(a, 0)  (:70-71)                                         */
  PC_EW_RELU_GRAD = 4 /* out = a * (b>0)  (:88-90)                                         */
};
int pc_fill(int dtype, int64_t n, double value, void* out, void* stream);
int pc_ewise(int op, int dtype, int64_t n, const void* a, const void* b, int64_t b_n, void* out,
             void* stream);
/* *out = 0.5 * sum(x*x): "sub-sample-loss" (executor.py:72-75); deterministic. */
int pc_sumsq_half(int dtype, int64_t n, const void* x, void* out, void* stream);
int pc_sum_f32(int64_t n, const float* x, float* out, void* stream);
/* out[c] (+)= sum_r x[r,c]: "sum-to" (executor.py:50-56) and bias gradients. */
int pc_col_sum(int dtype_in, int dtype_out, int64_t rows, int64_t cols, const void* x,
               int64_t ldx, void* out, int accumulate, void* ws, int64_t ws_bytes, void* stream);
/* A/B hook: 1 (default) bf16 column sums (bias / LayerNorm / RMSNorm parameter
 * gradients) as one-pass cluster reductions (no workspace), 0 the two-stage
 * workspace kernel below. */
int pc_colsum_set_cluster(int on);
/* Scratch for the two-stage (many-CTA, fixed-order) column reductions used by
 * pc_col_sum and pc_layernorm_bwd; with ws == NULL they fall back to one stage. */
int pc_reduce_workspace_bytes(int64_t rows, int64_t cols, int64_t* bytes);
/* dst = src or src^T (slice / concat / broadcast materialisation, :78-95); lds = 0 with
 * trans = 0 repeats one source row (or one element, cols = 1) into every dst row. */
int pc_copy2d(int dtype, int64_t rows, int64_t cols, const void* src, int64_t lds, int trans,
              void* dst, int64_t ldd, void* stream);
/* acc += part in place: the fused fp32 gradient accumulator replacing the
 * grad-merge chain (taskgraph.py:369-433, executor.py:335-336). */
int pc_accumulate(int dtype_acc, int dtype_part, int64_t n, void* acc, const void* part,
                  void* stream);
/* w_out = w - lr*g (executor.py:340-344); optional bf16 shadow copy of w_out. */
int pc_sgd_update(int dtype, int64_t n, const void* w, const void* g, double lr, void* w_out,
                  void* shadow_bf16, void* stream);
int pc_cast(int dtype_in, int dtype_out, int64_t n, const void* in, void* out, void* stream);
/* *slot = %globaltimer (ns), stream-ordered; the measured task timeline (bubble). */
int pc_timestamp(void* slot, void* stream);

/* ---- GPT vocabulary (oracle/gpt.py semantics; no reference counterpart) ---- */
int pc_layernorm_fwd(int dtype, int64_t rows, int64_t d, const void* x, const float* gamma,
                     const float* beta, void* y, float* mean, float* rstd, float eps,
                     void* stream);
/* dx = dres + LN_bwd(dy); dgamma, dbeta written (fp32). dres may be NULL. */
int pc_layernorm_bwd(int dtype, int64_t rows, int64_t d, const void* dy, const void* x,
                     const float* gamma, const float* mean, const float* rstd, const void* dres,
                     void* dx, float* dgamma, float* dbeta, void* ws, int64_t ws_bytes,
                     void* stream);
/* As pc_layernorm_bwd; accumulate = 1 adds dgamma / dbeta onto the fp32 gradient
 * accumulators (acc + partial, the grad-merge add fused into the reduction; needs ws). */
int pc_layernorm_bwd_acc(int dtype, int64_t rows, int64_t d, const void* dy, const void* x,
                         const float* gamma, const float* mean, const float* rstd,
                         const void* dres, void* dx, float* dgamma, float* dbeta, int accumulate,
                         void* ws, int64_t ws_bytes, void* stream);
/* dgamma (+)= sum_r dy * xhat, dbeta (+)= sum_r dy (dbeta may be NULL; mean NULL =
 * RMSNorm statistics): the LayerNorm parameter gradients alone, so they can run on
 * another stream than the dx chain (pc_layernorm_bwd_acc with dgamma = dbeta = NULL). */
int pc_layernorm_param_grads(int dtype, int64_t rows, int64_t d, const void* dy, const void* x,
                             const float* mean, const float* rstd, float* dgamma, float* dbeta,
                             int accumulate, void* ws, int64_t ws_bytes, void* stream);
/* One pass for a GPT block's LN2 side-stream sums (bf16, [rows, d], ld = d, 16 B rows):
 * dgamma / dbeta as pc_layernorm_param_grads, dsum3 (+)= sum_r y3 (the fc2 bias
 * gradient, y3 = the block's incoming gradient) and dsum4 (+)= sum_r y4 (the
 * attention-output bias gradient, y4 = LN2's output gradient).  Bitwise equal to
 * pc_layernorm_param_grads + two pc_col_sum calls; replaces the bias column sums of
 * the reference backward's `sum-to` rule (executor.py:50-56, 91-92) for those two biases. */
int pc_layernorm_param_bias_grads(int64_t rows, int64_t d, const void* dy, const void* x,
                                  const float* mean, const float* rstd, float* dgamma,
                                  float* dbeta, const void* y3, float* dsum3, const void* y4,
                                  float* dsum4, int accumulate, void* stream);
/* LayerNorm backward in one read of dy and x: dx (+ dres) as pc_layernorm_bwd, plus per-CTA
 * partial rows of dgamma = sum dy*xhat and dbeta = sum dy written to partials [2][n_part][d]
 * (n_part from pc_layernorm_partial_rows); pc_col_sum (fp32, fixed order, accumulate as
 * needed, any stream) over each [n_part, d] half finishes the parameter gradients.  bf16/fp32
 * rows with d % 256 == 0, d <= 1024. */
int pc_layernorm_partial_rows(int64_t rows, int64_t d, int64_t* n_part);
int pc_layernorm_bwd_partials(int dtype, int64_t rows, int64_t d, const void* dy, const void* x,
                              const float* gamma, const float* mean, const float* rstd,
                              const void* dres, void* dx, float* partials, int64_t n_part,
                              void* stream);
/* ---- Llama-style block pieces (BASELINE config C5; oracle/llama.py) ---- */
/* y = x * rsqrt(mean(x^2) + eps) * gamma; rstd [rows] fp32 saved (oracle rms_norm). */
int pc_rmsnorm_fwd(int dtype, int64_t rows, int64_t d, const void* x, const float* gamma,
                   void* y, float* rstd, float eps, void* stream);
/* dx = dres + RMSNorm_bwd(dy) (dres may be NULL); dgamma written (fp32, deterministic
 * two-stage reduction in ws, see pc_reduce_workspace_bytes), or not computed when NULL
 * (pc_layernorm_param_grads with mean = NULL gives it, accumulating, on another stream).
 * (oracle rms_norm_bwd) */
int pc_rmsnorm_bwd(int dtype, int64_t rows, int64_t d, const void* dy, const void* x,
                   const float* gamma, const float* rstd, const void* dres, void* dx,
                   float* dgamma, void* ws, int64_t ws_bytes, void* stream);
/* In-place rotate-half rotary embedding of n_heads consecutive head_dim-wide heads per
 * row (t [rows, ld]), angle = pos[row] * theta^(-2i/head_dim); inverse = 1 applies the
 * transpose rotation (backward). (oracle rope) */
int pc_rope(int dtype, int64_t rows, int64_t n_heads, int64_t head_dim, void* t, int64_t ld,
            const int32_t* pos, float theta, int inverse, void* stream);
/* m = silu(g) * u for gu = [g | u] (f columns each). (oracle silu) */
int pc_swiglu_fwd(int dtype, int64_t rows, int64_t f, const void* gu, int64_t ld_gu, void* m,
                  int64_t ld_m, void* stream);
/* dgu = [dm * u * silu'(g) | dm * silu(g)]. */
int pc_swiglu_bwd(int dtype, int64_t rows, int64_t f, const void* gu, int64_t ld_gu,
                  const void* dm, int64_t ld_dm, void* dgu, int64_t ld_dgu, void* stream);
/* Grouped-query attention heads: reduce = 0 expands [q(H)|k(Hkv)|v(Hkv)] to
 * [q(H)|k(H)|v(H)] (query head h reads kv head h / (H/Hkv)); reduce = 1 maps the
 * expanded gradient back, summing each kv head's group in ascending order. */
int pc_gqa_kv(int dtype, int64_t rows, int64_t n_heads, int64_t n_kv_heads, int64_t head_dim,
              const void* src, int64_t ld_src, void* dst, int64_t ld_dst, int reduce,
              void* stream);
int pc_embedding_fwd(int dtype, int64_t T, int64_t d, int64_t seq, const int32_t* tokens,
                     const float* wte, const float* wpe, void* out, void* stream);
int pc_embedding_bwd_workspace_bytes(int64_t T, int64_t* bytes);
int pc_embedding_bwd(int dtype, int64_t T, int64_t d, int64_t seq, int64_t vocab,
                     const int32_t* tokens, const void* dh, float* dwte, float* dwpe,
                     void* workspace, int64_t ws_bytes, void* stream);
/* As pc_embedding_bwd; accumulate = 1 adds the token-row and position sums onto dwte /
 * dwpe (the running gradient) instead of overwriting (no zero-fill of dwte).  dwpe may be
 * NULL (no position table). */
int pc_embedding_bwd_acc(int dtype, int64_t T_, int64_t d, int64_t seq, int64_t vocab,
                         const int32_t* tokens, const void* dh, float* dwte, float* dwpe,
                         int accumulate, void* workspace, int64_t ws_bytes, void* stream);
/* Next-token cross-entropy per row (targets = tokens shifted by one inside each
 * sequence); overwrites logits with dlogits = softmax - onehot. */
int pc_xent_fwd_bwd(int dtype, int64_t rows, int64_t V, int64_t seq, void* logits, int64_t ld,
                    const int32_t* tokens, float* row_loss, void* stream);
/* Fused LM head + next-token cross-entropy (replaces `sub-sample-loss`, executor.py:72-75,
 * for the GPT / Llama vocabularies; oracle/gpt.py head_loss).  Forward: logits [T, V] =
 * h [T, d] x W[V, d]^T (tcgen05), whose epilogue also leaves per-row partial (max, sum exp)
 * in ws; one streaming pass then writes row_loss [T] and overwrites logits in place with
 * dlogits = softmax - onehot(next token) (zero rows at each sequence's last position).
 * ws: pc_lmhead_xent_workspace bytes.  Backward: dh = dlogits W (B read K-major from
 * W^T [d, V]) and dW (+)= dlogits^T h (fp32; accumulate = 1 adds onto dW). */
int pc_lmhead_xent_workspace(int64_t T, int64_t V, int64_t d, int64_t* ld_stats, int64_t* bytes);
int pc_lmhead_xent_fwd(int64_t T, int64_t V, int64_t d, int64_t seq, const void* h, int64_t ldh,
                       const void* w, int64_t ldw, const int32_t* tokens, void* logits,
                       int64_t ld_logits, void* ws, int64_t ws_bytes, float* row_loss,
                       void* stream);
int pc_lmhead_xent_bwd(int64_t T, int64_t V, int64_t d, const void* dlogits, int64_t ld,
                       const void* h, int64_t ldh, const void* w_t, int64_t ld_wt, void* dh,
                       int64_t ld_dh, float* dw, int64_t ld_dw, int accumulate, void* stream);
/* Causal attention over packed qkv [B*S, ld_qkv]; lse/delta are [B,H,S] fp32. */
int pc_attention_fwd(int dtype, int B, int H, int S, int hd, const void* qkv, int64_t ld_qkv,
                     void* o, int64_t ld_o, float* lse, void* stream);
int pc_attention_bwd(int dtype, int B, int H, int S, int hd, const void* qkv, int64_t ld_qkv,
                     const void* o, const void* dO, int64_t ld_o, const float* lse, float* delta,
                     void* dqkv, int64_t ld_dqkv, void* stream);
/* Grouped-query causal attention (SURVEY §8(b) pc_attention_fwd/bwd with Hkv): qkv packs H
 * query heads, then Hkv key heads, then Hkv value heads, each hd columns; query head h reads
 * kv head h / (H / Hkv); dqkv has qkv's layout and a kv head's gradient sums its group
 * (oracle/llama.py gqa_attention[_bwd]).  Replaces the `matmul` + softmax numpy expressions
 * of a stage forward (executor.py:66-67) for the attention blocks.  bf16 head_dim 64 / 128:
 * tcgen05 kernels; Hkv == H otherwise also served by the legacy / SIMT kernels. */
int pc_attention_gqa_fwd(int dtype, int B, int H, int Hkv, int S, int hd, const void* qkv,
                         int64_t ld_qkv, void* o, int64_t ld_o, float* lse, void* stream);
int pc_attention_gqa_bwd(int dtype, int B, int H, int Hkv, int S, int hd, const void* qkv,
                         int64_t ld_qkv, const void* o, const void* dO, int64_t ld_o,
                         const float* lse, float* delta, void* dqkv, int64_t ld_dqkv,
                         void* stream);
/* 0 = auto (bf16: tcgen05 for head_dim 64 / 128), 1 = force exact SIMT,
 * 2 = force the mma.sync kernels. Test hook. */
int pc_attention_set_impl(int impl);
/* Tuning hook for the tcgen05 attention kernels (bench / A-B tools; the
 * defaults are the measured best).  key 0: head_dim-64 forward design
 * (1 = one-tile-per-CTA fa_fwd_tc5 with P over S, 2 = persistent fa_fwd64_tc5 with one
 * MMA-issuing warp, 3 = the same with scores and PV from two issuing warps, default);
 * key 1: score columns of every 16 whose exp2 runs on the FMA pipe in fa_fwd64_tc5
 * (0, 4, 6 default, 8; 101 / 102 = profiling ablations without the softmax math /
 * without the MMAs, results meaningless); key 2: head_dim-128 forward with one (0) or
 * two (1, default) issuing warps; key 3: backward dQ kernel with one (0) or two (1,
 * default) issuing warps.  The issuer choices are bitwise identical. */
int pc_attention_tune(int key, int value);

/* ---- inter-stage transport over NVLink peer memory (Channel, executor.py:201-254) ----
 * The receiver allocates one slot per plan message plus flag words (pc_peer_alloc: zeroed
 * device memory + a 64-byte CUDA IPC handle); the sender maps them (pc_peer_open), has the
 * producing kernel write the message into the slot (or pc_peer_copy it there), then
 * pc_stream_write_u32(flag, 1); the receiver's stream pc_stream_wait_u32(flag, 1) and
 * re-arms the flag with pc_stream_write_u32(flag, 0).  Graph-capturable. */
int pc_peer_alloc(int64_t bytes, void** ptr, void* handle64);
int pc_peer_free(void* ptr);
int pc_peer_open(const void* handle64, void** ptr);
int pc_peer_close(void* ptr);
int pc_stream_write_u32(void* addr, uint32_t value, void* stream);
int pc_stream_wait_u32(void* addr, uint32_t value, void* stream);
int pc_peer_copy(void* dst, const void* src, int64_t bytes, void* stream);
/* RecvWait of the peer transport (Channel.recv, executor.py:223-240): a one-thread kernel
 * on `stream` spins until *flag == 1 (the sender's pc_stream_write_u32), re-arms it to 0
 * and exits.  It also polls *abort_word_dev (mapped host memory, pc_host_word_alloc):
 * the watchdog (executor.py:443-451) sets the word from the CPU and the wait ends, so a
 * message that will never arrive cannot park the device forever. */
int pc_peer_wait(void* flag, const void* abort_word_dev, void* stream);
/* 64 zeroed bytes of page-locked host memory mapped for the device: *host for CPU
 * stores, *dev for kernels. */
int pc_host_word_alloc(void** host, void** dev);
int pc_host_word_free(void* host);
/* Kernel nodes of a captured CUDA graph (cudaGraph_t), child graphs included. */
int pc_graph_kernel_nodes(void* graph, int64_t* n);

/* ---- inter-stage transport (Channel, executor.py:201-254) over NCCL ---- */
int pc_p2p_available(void);
int pc_p2p_unique_id(void* out128);
int pc_p2p_comm_init(void** comm, int nranks, const void* id128, int rank);
int pc_p2p_send(void* comm, const void* buf, int64_t bytes, int peer, void* stream);
int pc_p2p_recv(void* comm, void* buf, int64_t bytes, int peer, void* stream);
int pc_p2p_abort(void* comm);
int pc_p2p_destroy(void* comm);

#ifdef __cplusplus
}
#endif

#endif /* PP200_H */
