// cusparse_spmm.cu -- the library baseline of the measurement protocol (the
// paper compares against cuSPARSE 12.0): cusparseSpMM on the same CSR and dense
// row-major X, per algorithm (ALG_DEFAULT, CSR_ALG1, CSR_ALG2, CSR_ALG3), with bufferSize and
// preprocess outside the timed region, timed with CUDA events per call, cold (512 MB scratch
// written + persisting L2 reset before every rep, as Nsight Compute's cache control) or warm
// (back to back).  Not part of the product: bench.py loads it to time the comparison arm.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC -lcusparse
#include <cuda_runtime.h>
#include <cusparse.h>
#include <stdint.h>

extern "C" {

// Make L2 cold: write `bytes` of scratch (larger than L2) and demote persisting lines.
int bl_l2_flush(void* scratch, size_t bytes, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (cudaMemsetAsync(scratch, 0x5a, bytes, s) != cudaSuccess) return -1;
    cudaCtxResetPersistingL2Cache();
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

// Y[n x F] = A[n x n_cols] . X[n_cols x F] with cusparseSpMM, algorithm `alg` (cusparseSpMMAlg_t
// value).  rowptr[n+1] (rowptr[0] == 0), colidx[nnz], vals[nnz], X, Y: DEVICE.  Runs 3 untimed
// calls, then `reps` timed calls; ms[reps] gets each call's CUDA-event time.  cold != 0: every
// rep is preceded by bl_l2_flush(scratch, scratch_bytes).  Returns 0, or the cusparseStatus_t
// (e.g. CUSPARSE_STATUS_NOT_SUPPORTED for an algorithm that does not accept the layout), or
// -1 on a CUDA error.  *buffer_bytes: the external buffer the algorithm asked for.
int bl_cusparse_spmm(const int32_t* rowptr, const int32_t* colidx, const float* vals, int64_t n, int64_t n_cols,
                     int64_t nnz, const float* X, int32_t F, float* Y, int32_t alg, int32_t reps, int32_t cold,
                     void* scratch, size_t scratch_bytes, float* ms, size_t* buffer_bytes, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    cusparseHandle_t h = nullptr;
    cusparseSpMatDescr_t A = nullptr;
    cusparseDnMatDescr_t B = nullptr, C = nullptr;
    void* buf = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    int rc = 0;
    const float one = 1.f, zero = 0.f;
    const cusparseSpMMAlg_t a = (cusparseSpMMAlg_t)alg;
    size_t bsz = 0;
#define CS(x)                                      \
    do {                                           \
        cusparseStatus_t st__ = (x);               \
        if (st__ != CUSPARSE_STATUS_SUCCESS) {     \
            rc = (int)st__;                        \
            goto done;                             \
        }                                          \
    } while (0)
#define CU(x)                      \
    do {                           \
        if ((x) != cudaSuccess) {  \
            rc = -1;               \
            goto done;             \
        }                          \
    } while (0)
    CS(cusparseCreate(&h));
    CS(cusparseSetStream(h, s));
    CS(cusparseCreateCsr(&A, n, n_cols, nnz, (void*)rowptr, (void*)colidx, (void*)vals, CUSPARSE_INDEX_32I,
                         CUSPARSE_INDEX_32I, CUSPARSE_INDEX_BASE_ZERO, CUDA_R_32F));
    CS(cusparseCreateDnMat(&B, n_cols, F, F, (void*)X, CUDA_R_32F, CUSPARSE_ORDER_ROW));
    CS(cusparseCreateDnMat(&C, n, F, F, (void*)Y, CUDA_R_32F, CUSPARSE_ORDER_ROW));
    CS(cusparseSpMM_bufferSize(h, CUSPARSE_OPERATION_NON_TRANSPOSE, CUSPARSE_OPERATION_NON_TRANSPOSE, &one, A, B,
                               &zero, C, CUDA_R_32F, a, &bsz));
    if (buffer_bytes) *buffer_bytes = bsz;
    CU(cudaMalloc(&buf, bsz ? bsz : 16));
    {
        const cusparseStatus_t pst = cusparseSpMM_preprocess(h, CUSPARSE_OPERATION_NON_TRANSPOSE,
                                                             CUSPARSE_OPERATION_NON_TRANSPOSE, &one, A, B, &zero, C,
                                                             CUDA_R_32F, a, buf);
        if (pst != CUSPARSE_STATUS_SUCCESS && pst != CUSPARSE_STATUS_NOT_SUPPORTED) {
            rc = (int)pst;
            goto done;
        }
    }
    for (int i = 0; i < 3; ++i)
        CS(cusparseSpMM(h, CUSPARSE_OPERATION_NON_TRANSPOSE, CUSPARSE_OPERATION_NON_TRANSPOSE, &one, A, B, &zero, C,
                        CUDA_R_32F, a, buf));
    CU(cudaEventCreate(&e0));
    CU(cudaEventCreate(&e1));
    for (int r = 0; r < reps; ++r) {
        if (cold && bl_l2_flush(scratch, scratch_bytes, s) != 0) {
            rc = -1;
            goto done;
        }
        CU(cudaEventRecord(e0, s));
        CS(cusparseSpMM(h, CUSPARSE_OPERATION_NON_TRANSPOSE, CUSPARSE_OPERATION_NON_TRANSPOSE, &one, A, B, &zero, C,
                        CUDA_R_32F, a, buf));
        CU(cudaEventRecord(e1, s));
        CU(cudaEventSynchronize(e1));
        CU(cudaEventElapsedTime(ms + r, e0, e1));
    }
done:
    cudaStreamSynchronize(s);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (buf) cudaFree(buf);
    if (A) cusparseDestroySpMat(A);
    if (B) cusparseDestroyDnMat(B);
    if (C) cusparseDestroyDnMat(C);
    if (h) cusparseDestroy(h);
    return rc;
#undef CS
#undef CU
}

}  // extern "C"
