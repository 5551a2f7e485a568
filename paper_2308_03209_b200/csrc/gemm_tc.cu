// gemm_tc.cu — tensor-core GEMM path (tcgen05, sm_100a). v0: dispatch only.
#include "gemm_tc.cuh"
#include "internal.hpp"
#include "trainer.hpp"

namespace sc {

void TcGemm::init(sc_trainer* t) { enabled = t->gemm_mode == 0 && false; }

void TcGemm::nt(sc_trainer* t, const MatA& a1, const MatB& b1, const MatA* a2, const MatB* b2, float* C, int64_t ldc,
                int64_t M, int32_t N, int epi, const float* row_scale) {
    gemm_nt(a1, b1, a2, b2, C, ldc, M, N, epi, row_scale, t->ctx->stream);
}

}  // namespace sc
