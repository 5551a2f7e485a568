// gemm_tc.cuh — tensor-core GEMM path (tcgen05 fp16x3, gemm_tc.cu) and its dispatcher.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <tuple>

#include "internal.hpp"
#include "nn.cuh"

struct sc_trainer;

namespace sc {

// A weight operand pre-scaled (by 2^bexp) and pre-split into fp16 hi/lo
// k-block images (32 k, SW64 K-major layout), ready for one bulk copy per stage.
struct BImage {
    DevBuf<uint8_t> img;
    DevBuf<int32_t> bexp;
    DevBuf<float> amax;  // max |B| (prep scratch)
    int32_t N = 0, K = 0, n_pad = 0, kblocks = 0;
};

bool tc_supported(const MatA& a1, const MatA* a2, int32_t N);
bool tc_out_supported(const float* C, int64_t ldc);
bool tn_supported(const MatT& a, const MatT& b1, const MatT* b2);
void prep_bimage(BImage& im, const MatB& b, int32_t N, int32_t K, cudaStream_t s);

// C[M x N] = A1 op(B1) (+ A2 op(B2)) on the tensor cores in fp16x3 split
// precision. amax_i: device scalars holding max|A_i| (upper bounds are fine);
// amax_out (optional): max|C| is atomically reduced into it. relu_pos (optional,
// epi == kEpiRelu): the ReLU decisions as bits, [M][ceil(N / 32)] words.
void gemm_f16x3(const MatA& a1, const float* amax1, const BImage& b1, const MatA* a2, const float* amax2,
                const BImage* b2, float* C, int64_t ldc, int64_t M, int32_t N, int epi, const float* row_scale,
                float* amax_out, cudaStream_t s, uint32_t* relu_pos = nullptr, const float* mask_msg = nullptr,
                const uint32_t* mask_pos = nullptr);

// Weight gradient C[N1 x N2] = A^T [B1 | B2] (K = M rows) on the tensor cores,
// fp16x3, split-K with a fixed-order reduction (deterministic). ws needs
// tn_f16x3_splits(N1, N2, M) * N1 * N2 floats.
int32_t tn_f16x3_splits(int32_t N1, int32_t N2, int64_t M);
void gemm_tn_f16x3(const MatT& a, const float* amax_a, const MatT& b1, const float* amax_b1, const MatT* b2,
                   const float* amax_b2, int64_t M, float* C, int64_t ldc, float* ws, int64_t ws_floats,
                   cudaStream_t s);

// Dual weight-gradient launch of one layer: C1 = A1^T [B1 | B2] and C2 = A2^T B2 in one split-K
// TN launch over A = [A1 | A2] (the A2 x B1 block skipped), so B2 (the layer input) and the
// converted tiles are streamed once for both products (CTA pairs; A1 columns a multiple of 256,
// B1 columns a multiple of 256).
bool tn_dual_supported(const MatT& a1, const MatT& a2, const MatT& b1, const MatT& b2);
void gemm_tn_f16x3_dual(const MatT& a1, const float* amax_a1, const MatT& a2, const float* amax_a2, const MatT& b1,
                        const float* amax_b1, const MatT& b2, const float* amax_b2, int64_t M, float* C1,
                        int64_t ldc1, float* C2, int64_t ldc2, float* ws, int64_t ws_floats, cudaStream_t s);

// Uses gemm_f16x3 when the trainer allows it and the shape is supported,
// otherwise the fp32 SIMT kernel (nn.cu). Weight images are cached per
// operand and rebuilt when `version` changes (after every Adam step).
struct TcGemm {
    bool enabled = false;
    uint64_t version = 1;
    using Key = std::tuple<const float*, int64_t, bool, int32_t, int32_t>;
    struct Entry {
        BImage im;
        uint64_t version = 0;
    };
    std::map<Key, Entry> cache;
    // GEMMs that ran on the fp32 SIMT kernels although the tensor-core path was
    // enabled (operand layout not TMA-compatible): counted, never silent.
    int64_t simt_fallbacks = 0;
    bool dual = false;  // one launch for a layer's dU and dW where shapes allow (SC_TN_DUAL=1; default: two)
    void init(sc_trainer* t);
    void invalidate() { ++version; }
    const BImage& image(const MatB& b, int32_t N, int32_t K, cudaStream_t s);
    void nt(sc_trainer* t, const MatA& a1, const float* amax1, const MatB& b1, const MatA* a2, const float* amax2,
            const MatB* b2, float* C, int64_t ldc, int64_t M, int32_t N, int epi, const float* row_scale,
            float* amax_out, uint32_t* relu_pos = nullptr, const float* mask_msg = nullptr,
            const uint32_t* mask_pos = nullptr);
    // dU and dW of one layer in one launch (false: unsupported here, caller runs tn twice)
    bool tn_dual(sc_trainer* t, const MatT& a1, const float* amax_a1, const MatT& a2, const float* amax_a2,
                 const MatT& b1, const float* amax_b1, const MatT& b2, const float* amax_b2, int64_t M, float* C1,
                 int64_t ldc1, float* C2, int64_t ldc2);
    // s / ws: stream and split-K workspace (default: the context stream, t->ws)
    void tn(sc_trainer* t, const MatT& a, const float* amax_a, const MatT& b1, const float* amax_b1, const MatT* b2,
            const float* amax_b2, int64_t M, float* C, int64_t ldc, cudaStream_t s = nullptr, float* ws = nullptr);
};

}  // namespace sc
