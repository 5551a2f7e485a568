// gemm_tc.cuh — GEMM dispatcher for the M-huge products of the step.
#pragma once

#include <cuda_runtime.h>

#include "internal.hpp"
#include "nn.cuh"

struct sc_trainer;

namespace sc {

// C[M x N] = A1 op(B1) (+ A2 op(B2)) with an epilogue on the tcgen05 tensor
// cores in bf16x3 split precision (gemm_tc.cu). A rows must be 16-byte
// aligned (ld % 4 == 0); N <= 256. `bimg` is scratch for the pre-split B image.
void gemm_bf16x3(const MatA& a1, const MatB& b1, const MatA* a2, const MatB* b2, float* C, int64_t ldc, int64_t M,
                 int32_t N, int epi, const float* row_scale, DevBuf<uint8_t>& bimg, cudaStream_t s);

// Uses gemm_bf16x3 when the trainer allows it and the shape is supported;
// otherwise the fp32 SIMT kernel (nn.cu).
struct TcGemm {
    bool enabled = false;
    DevBuf<uint8_t> bimg;
    void init(sc_trainer* t);
    void nt(sc_trainer* t, const MatA& a1, const MatB& b1, const MatA* a2, const MatB* b2, float* C, int64_t ldc,
            int64_t M, int32_t N, int epi, const float* row_scale);
};

}  // namespace sc
