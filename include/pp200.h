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

/* Force the tcgen05 GEMM tile width (0 = heuristic, else 64/128/256). Test hook. */
int pc_gemm_set_tile_n(int bn);

#ifdef __cplusplus
}
#endif

#endif /* PP200_H */
