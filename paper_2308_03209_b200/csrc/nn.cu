// nn.cu — SIMT kernels of the per-partition training step (sm_100a).
//
// fp32 everywhere the reference's f32 mode is fp32, f64 where it accumulates
// in f64 (loss total, grad norm). The aggregation kernels keep the reference's
// summation order exactly (CSR order of kept neighbours, then * inv), so their
// outputs are bitwise equal to nn.hpp:222-230 / 277-288 for equal inputs.
//
// The GEMMs here are the fp32 CUDA-core path (exact fp32 products, fp32
// accumulate); gemm_tc.cu holds the tcgen05 tensor-core path that the trainer
// uses for the large M x {H, in} products.
#include <cub/cub.cuh>

#include <cmath>

#include "internal.hpp"
#include "nn.cuh"

namespace sc {
namespace {

// ---------------------------------------------------------------------------
// SIMT GEMM: 128 x 128 x 16 tiles, 256 threads, 8 x 8 outputs per thread.
// ---------------------------------------------------------------------------
constexpr int BM = 128, BN = 128, BK = 16, TM = 8, TN = 8, NT = 256;

struct GemmArgs {
    MatA a[2];
    MatB b[2];
    int nsrc;
    float* C;
    int64_t ldc;
    int64_t M;
    int32_t N;
    int epi;
    const float* row_scale;
    float* amax_out;
    const float* mask_msg;     // kEpiMask (row stride N)
    const uint32_t* mask_pos;  // kEpiMask, sign bits
};

// |v| max-reduction into a float slot: non-negative floats order like their bits.
__device__ __forceinline__ void atomic_max_abs(float* slot, float v) {
    atomicMax(reinterpret_cast<unsigned int*>(slot), __float_as_uint(fabsf(v)));
}
__device__ __forceinline__ float warp_max_f(float x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, o));
    return x;
}

__device__ __forceinline__ float load_a(const MatA& a, int64_t r, int32_t k, int64_t M) {
    if (r >= M || k >= a.K) return 0.f;
    const int64_t row = a.rows ? a.rows[r] : r;
    return __ldg(a.ptr + row * a.ld + k);
}
__device__ __forceinline__ float load_b(const MatB& b, int32_t n, int32_t k, int32_t N, int32_t K) {
    if (n >= N || k >= K) return 0.f;
    return b.nn ? __ldg(b.ptr + int64_t(k) * b.ld + n) : __ldg(b.ptr + int64_t(n) * b.ld + k);
}

__global__ void __launch_bounds__(NT) gemm_nt_kernel(GemmArgs args) {
    __shared__ float As[BK][BM + 4];
    __shared__ float Bs[BK][BN + 4];
    const int tid = threadIdx.x;
    const int64_t m0 = int64_t(blockIdx.x) * BM;
    const int32_t n0 = blockIdx.y * BN;
    const int ty = tid / 16, tx = tid % 16;
    float acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;

    for (int src = 0; src < args.nsrc; ++src) {
        const MatA& A = args.a[src];
        const MatB& B = args.b[src];
        const int32_t K = A.K;
        for (int32_t k0 = 0; k0 < K; k0 += BK) {
            // A tile: 128 rows x 16 k; thread loads 8 (row = tid/2, k = (tid%2)*8 ..)
            {
                const int r = tid >> 1, kc = (tid & 1) * 8;
#pragma unroll
                for (int j = 0; j < 8; ++j) As[kc + j][r] = load_a(A, m0 + r, k0 + kc + j, args.M);
            }
            if (B.nn) {  // B[k][n]: coalesced along n
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int idx = tid + j * NT;  // 0..2047
                    const int kk = idx / BN, nn = idx % BN;
                    Bs[kk][nn] = load_b(B, n0 + nn, k0 + kk, args.N, K);
                }
            } else {
                const int nn = tid >> 1, kc = (tid & 1) * 8;
#pragma unroll
                for (int j = 0; j < 8; ++j) Bs[kc + j][nn] = load_b(B, n0 + nn, k0 + kc + j, args.N, K);
            }
            __syncthreads();
#pragma unroll
            for (int kk = 0; kk < BK; ++kk) {
                float av[TM], bv[TN];
#pragma unroll
                for (int i = 0; i < TM; ++i) av[i] = As[kk][ty * TM + i];
#pragma unroll
                for (int j = 0; j < TN; ++j) bv[j] = Bs[kk][tx * TN + j];
#pragma unroll
                for (int i = 0; i < TM; ++i)
#pragma unroll
                    for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
            }
            __syncthreads();
        }
    }
    float mx = 0.f;
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const int64_t r = m0 + ty * TM + i;
        if (r >= args.M) continue;
        const float sc = args.epi == kEpiRowScale ? args.row_scale[r] : 1.f;
#pragma unroll
        for (int j = 0; j < TN; ++j) {
            const int32_t c = n0 + tx * TN + j;
            if (c >= args.N) continue;
            float v = acc[i][j];
            if (args.epi == kEpiRelu) v = fmaxf(v, 0.f);
            else if (args.epi == kEpiRowScale) v = sc * v;
            else if (args.epi == kEpiMask) {
                const bool keep = args.mask_pos ? ((args.mask_pos[r * ((args.N + 31) >> 5) + (c >> 5)] >> (c & 31)) & 1u)
                                                : args.mask_msg[r * args.N + c] > 0.f;
                v = keep ? v : 0.f;
            }
            args.C[r * args.ldc + c] = v;
            mx = fmaxf(mx, fabsf(v));
        }
    }
    if (args.amax_out) {
        mx = warp_max_f(mx);
        if ((threadIdx.x & 31) == 0) atomic_max_abs(args.amax_out, mx);
    }
}

__global__ void gather_rows_kernel(int64_t n, int32_t d, const int32_t* __restrict__ rows, const float* __restrict__ src,
                                   float* __restrict__ dst) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n * d; i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = i / d;
        dst[i] = src[int64_t(rows[r]) * d + (i - r * d)];
    }
}

// 16-byte variant (d % 4 == 0, 16-byte aligned rows): one float4 per thread.
__global__ void gather_rows4_kernel(int64_t n, int32_t d4, const int32_t* __restrict__ rows,
                                    const float4* __restrict__ src, float4* __restrict__ dst) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n * d4; i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = i / d4;
        dst[i] = __ldg(src + int64_t(rows[r]) * d4 + (i - r * d4));
    }
}

__global__ void absmax_kernel(int64_t n, const float* __restrict__ x, float* out) {
    float mx = 0.f;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        mx = fmaxf(mx, fabsf(x[i]));
    mx = warp_max_f(mx);
    if ((threadIdx.x & 31) == 0) atomic_max_abs(out, mx);
}

// Weight-gradient GEMM, split-K: block (tile, split) accumulates a 128 x 128
// tile of A^T B over its row range and writes it to workspace[split].
struct TnArgs {
    MatT a;
    MatT b[2];
    int32_t n2a;  // columns from b[0]; the rest from b[1]
    int32_t N1, N2;
    int64_t M;
    int64_t rows_per_split;
    float* ws;
};
__device__ __forceinline__ float load_t(const MatT& x, int64_t r, int32_t c) {
    const int64_t row = x.rows ? x.rows[r] : r;
    return __ldg(x.ptr + row * x.ld + c);
}

__global__ void __launch_bounds__(NT) gemm_tn_kernel(TnArgs args) {
    __shared__ float As[BK][BM + 4];
    __shared__ float Bs[BK][BN + 4];
    const int tid = threadIdx.x;
    const int32_t tiles_n2 = (args.N2 + BN - 1) / BN;
    const int32_t t1 = blockIdx.x / tiles_n2, t2 = blockIdx.x % tiles_n2;
    const int32_t n10 = t1 * BM, n20 = t2 * BN;
    const int64_t r_begin = int64_t(blockIdx.y) * args.rows_per_split;
    const int64_t r_end = min(args.M, r_begin + args.rows_per_split);
    const int ty = tid / 16, tx = tid % 16;
    float acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;
    for (int64_t k0 = r_begin; k0 < r_end; k0 += BK) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int idx = tid + j * NT;
            const int kk = idx / BM, cc = idx % BM;
            const int64_t r = k0 + kk;
            const int32_t c1 = n10 + cc, c2 = n20 + cc;
            float av = 0.f, bv = 0.f;
            if (r < r_end) {
                if (c1 < args.N1) av = load_t(args.a, r, c1);
                if (c2 < args.N2) bv = c2 < args.n2a ? load_t(args.b[0], r, c2) : load_t(args.b[1], r, c2 - args.n2a);
            }
            As[kk][cc] = av;
            Bs[kk][cc] = bv;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            float av[TM], bv[TN];
#pragma unroll
            for (int i = 0; i < TM; ++i) av[i] = As[kk][ty * TM + i];
#pragma unroll
            for (int j = 0; j < TN; ++j) bv[j] = Bs[kk][tx * TN + j];
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        }
        __syncthreads();
    }
    float* out = args.ws + int64_t(blockIdx.y) * args.N1 * args.N2;
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const int32_t r = n10 + ty * TM + i;
        if (r >= args.N1) continue;
#pragma unroll
        for (int j = 0; j < TN; ++j) {
            const int32_t c = n20 + tx * TN + j;
            if (c < args.N2) out[int64_t(r) * args.N2 + c] = acc[i][j];
        }
    }
}

__global__ void splitk_reduce_kernel(int32_t S, int32_t N1, int32_t N2, const float* ws, float* C, int64_t ldc) {
    const int64_t total = int64_t(N1) * N2;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
        float acc = 0.f;
        for (int32_t s = 0; s < S; ++s) acc += ws[int64_t(s) * total + i];
        C[(i / N2) * ldc + (i % N2)] = acc;
    }
}

constexpr int kMaxSplits = 256;

int32_t tn_splits(int32_t N1, int32_t N2, int64_t M) {
    const int32_t tiles = ((N1 + BM - 1) / BM) * ((N2 + BN - 1) / BN);
    int64_t s = (int64_t(num_sms()) * 3 + tiles - 1) / tiles;  // ~3 waves
    s = std::min<int64_t>(s, (M + 2047) / 2048);                  // >= 2048 rows per split
    s = std::max<int64_t>(s, 1);
    return static_cast<int32_t>(std::min<int64_t>(s, kMaxSplits));
}

// ---------------------------------------------------------------------------
// Aggregation (warp per row; lanes own float4 column chunks).
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool slot_kept(const uint32_t* bits, int64_t k) {
    return bits == nullptr || ((__ldg(bits + (k >> 5)) >> (k & 31)) & 1u);
}

__global__ void inv_degree_kernel(int64_t n, const int64_t* __restrict__ off, const uint32_t* __restrict__ bits,
                                  float* inv) {
    for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < n; v += int64_t(gridDim.x) * blockDim.x) {
        const int64_t a = off[v], b = off[v + 1];
        int32_t d = 0;
        if (!bits) {
            d = static_cast<int32_t>(b - a);
        } else {  // popcount of the row's slot range, word by word (hub rows span many words)
            for (int64_t k = a; k < b;) {
                const int64_t wbase = k & ~int64_t(31);
                const int lo = static_cast<int>(k - wbase);
                const int hi = static_cast<int>(min(b - wbase, int64_t(32)));
                uint32_t word = __ldg(bits + (k >> 5));
                word >>= lo;
                if (hi - lo < 32) word &= (1u << (hi - lo)) - 1u;
                d += __popc(word);
                k = wbase + hi;
            }
        }
        inv[v] = d > 0 ? 1.f / static_cast<float>(d) : 0.f;
    }
}

// Sum of the kept source rows over CSR slots [a, b) in slot order (the
// reference's order); lanes own float4 column chunks, up to 4 row loads in flight.
// kScale: every gathered row is scaled by inv[nbr] first (spmm_sum_scaled's hub segments)
template <int NCH, bool kScale = false>
__device__ __forceinline__ void gather_rows_sum(int64_t a, int64_t b, int lane, int32_t H, int32_t H4,
                                                const int32_t* __restrict__ nbrs, const uint32_t* __restrict__ bits,
                                                const float* __restrict__ src, float4 (&acc)[NCH],
                                                const float* __restrict__ inv = nullptr) {
    for (int64_t base = a; base < b; base += 32) {
        const int64_t k = base + lane;
        const bool valid = k < b;
        const int32_t nb = valid ? __ldg(nbrs + k) : 0;
        const bool kept = valid && slot_kept(bits, k);
        unsigned ballot = __ballot_sync(0xffffffffu, kept);
        while (ballot) {
            int32_t u[4];
            int cnt = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (ballot) {
                    const int sl = __ffs(ballot) - 1;
                    ballot &= ballot - 1;
                    u[q] = __shfl_sync(0xffffffffu, nb, sl);
                    ++cnt;
                } else {
                    u[q] = -1;
                }
            }
            float4 vals[4][NCH];
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int c = 0; c < NCH; ++c) {
                    const int32_t ch = lane + 32 * c;
                    if (q < cnt && ch < H4)
                        vals[q][c] = __ldg(reinterpret_cast<const float4*>(src + int64_t(u[q]) * H) + ch);
                    else
                        vals[q][c] = make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (q < cnt) {
                    const float sq = kScale ? __ldg(inv + u[q]) : 1.f;
#pragma unroll
                    for (int c = 0; c < NCH; ++c) {
                        float4 x = vals[q][c];
                        if (kScale) {  // separately rounded products, as in spmm_narrow_kernel
                            x.x = __fmul_rn(sq, x.x);
                            x.y = __fmul_rn(sq, x.y);
                            x.z = __fmul_rn(sq, x.z);
                            x.w = __fmul_rn(sq, x.w);
                        }
                        acc[c].x += x.x;
                        acc[c].y += x.y;
                        acc[c].z += x.z;
                        acc[c].w += x.w;
                    }
                }
        }
    }
}

// Output row v: forward mean = inv[v] * sum (nn.hpp:229); backward dz =
// 1[msg > 0] * sum (nn.hpp:287-288). Returns max|out| of the lane's chunks.
// The ReLU decision comes from the msg row, or (compact activations) from its
// sign bits: word [v][c / 32], bit c % 32, written by the msg GEMM's epilogue.
// kX (variants of the composed top layer, trainer.cu): 0 as above; 1 forward, added to the row
// already in out (logits = h Z_R^T + inv * sum P[nbr]); 2 the plain sum (no inv, no mask: the pull
// form of the transposed aggregation of rows pre-scaled by inv).
template <int NCH, bool kBwd, bool kPos, int kX = 0>
__device__ __forceinline__ float finish_row(int64_t v, int lane, int32_t H, int32_t H4, const float* __restrict__ inv,
                                            const float* __restrict__ msg, const uint32_t* __restrict__ pos,
                                            float* __restrict__ out, const float4 (&acc)[NCH]) {
    float amx = 0.f;
    const float s = (kBwd || kX >= 2) ? 1.f : inv[v];
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
        const int32_t ch = lane + 32 * c;
        if (ch >= H4) continue;
        float4 r = acc[c];
        if (kX >= 2) {
        } else if (!kBwd) {
            r.x *= s;
            r.y *= s;
            r.z *= s;
            r.w *= s;
        } else if (kPos) {
            const uint32_t b = __ldg(pos + v * ((H + 31) >> 5) + (ch >> 3)) >> ((4 * ch) & 31);
            r.x = (b & 1u) ? r.x : 0.f;
            r.y = (b & 2u) ? r.y : 0.f;
            r.z = (b & 4u) ? r.z : 0.f;
            r.w = (b & 8u) ? r.w : 0.f;
        } else {
            const float4 mv = __ldg(reinterpret_cast<const float4*>(msg + v * H) + ch);
            r.x = mv.x > 0.f ? r.x : 0.f;
            r.y = mv.y > 0.f ? r.y : 0.f;
            r.z = mv.z > 0.f ? r.z : 0.f;
            r.w = mv.w > 0.f ? r.w : 0.f;
        }
        if (kX == 1) {  // (inv * sum) rounded, then added: no FMA contraction
            const float4 o = reinterpret_cast<const float4*>(out + v * H)[ch];
            r.x = __fadd_rn(o.x, r.x);
            r.y = __fadd_rn(o.y, r.y);
            r.z = __fadd_rn(o.z, r.z);
            r.w = __fadd_rn(o.w, r.w);
        }
        reinterpret_cast<float4*>(out + v * H)[ch] = r;
        amx = fmaxf(amx, fmaxf(fmaxf(fabsf(r.x), fabsf(r.y)), fmaxf(fabsf(r.z), fabsf(r.w))));
    }
    return amx;
}

// Warp per row over rows with at most `max_slots` CSR slots (heavier rows go
// through the segmented path below).
template <int NCH, bool kBwd, bool kPos = false, int kX = 0, bool kList = false>
__global__ void __launch_bounds__(256) spmm_kernel(int64_t n, int32_t H, const int64_t* __restrict__ off,
                                                   const int32_t* __restrict__ nbrs,
                                                   const uint32_t* __restrict__ bits, const float* __restrict__ inv,
                                                   const float* __restrict__ src, const float* __restrict__ msg,
                                                   const uint32_t* __restrict__ pos, float* __restrict__ out,
                                                   float* amax_out, int64_t max_slots, int64_t min_slots = -1,
                                                   const int32_t* __restrict__ rowlist = nullptr) {
    float amx = 0.f;
    const int lane = threadIdx.x & 31;
    const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
    const int32_t H4 = H >> 2;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += warps) {
        const int64_t v = kList ? rowlist[i] : i;  // (kList: n = the list's length)
        const int64_t a = off[v], b = off[v + 1];
        if (b - a > max_slots || (!kList && b - a <= min_slots)) continue;  // hub rows / the narrow kernel's rows
        float4 acc[NCH];
#pragma unroll
        for (int c = 0; c < NCH; ++c) acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
        gather_rows_sum<NCH, kX == 3>(a, b, lane, H, H4, nbrs, bits, src, acc, inv);
        amx = fmaxf(amx, finish_row<NCH, kBwd, kPos, kX>(v, lane, H, H4, inv, msg, pos, out, acc));
    }
    if (amax_out) {
        amx = warp_max_f(amx);
        if (lane == 0) atomic_max_abs(amax_out, amx);
    }
}

// Narrow rows (H <= 4 * LPR * CPL floats, e.g. the projected top layer's Cp = 48): a warp serves
// 32 / LPR rows at once, LPR lanes each, CPL float4 chunks per lane, so many more neighbour rows are
// in flight per warp. Per row the kept slots are summed in CSR order exactly as in spmm_kernel (the
// same bits). kX == 3: every gathered row is first scaled by inv[nbr] (the pull form of the
// transposed aggregation of inv-scaled rows, nn.hpp:284: inv_d * dmean.row(v)).
#ifndef SC_NARROW_MINB
#define SC_NARROW_MINB 4
#endif
// (minimum resident blocks: the kernel is bound by the dependent offset -> index -> row chain, so
// resident warps matter more than registers; CPL = 8 keeps its wider accumulators at 2)
template <int LPR, int CPL, bool kBwd, bool kPos, int kX, bool kList = false>
__global__ void __launch_bounds__(256, CPL <= 4 ? SC_NARROW_MINB : 2) spmm_narrow_kernel(int64_t n, int32_t H, const int64_t* __restrict__ off,
                                                          const int32_t* __restrict__ nbrs,
                                                          const uint32_t* __restrict__ bits,
                                                          const float* __restrict__ inv, const float* __restrict__ src,
                                                          const float* __restrict__ msg,
                                                          const uint32_t* __restrict__ pos, float* __restrict__ out,
                                                          float* amax_out, int64_t max_slots,
                                                          const int32_t* __restrict__ rowlist = nullptr) {
    constexpr int G = 32 / LPR;
    const int lane = threadIdx.x & 31;
    const int grp = lane / LPR, gl = lane % LPR;
    const unsigned gmask = (LPR == 32 ? 0xffffffffu : ((1u << LPR) - 1u)) << (grp * LPR);
    const int32_t H4 = H >> 2;
    float amx = 0.f;
    const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
    for (int64_t v0 = (blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5)) * G; v0 < n; v0 += warps * G) {
        const int64_t vi = v0 + grp;  // (kList: an index into the row list, n its length)
        bool skip = vi >= n;
        const int64_t v = kList ? (skip ? 0 : rowlist[vi]) : vi;
        int64_t a = 0, b = 0;
        if (!skip) {
            a = off[v];
            b = off[v + 1];
            skip = b - a > max_slots;  // hub row: the segmented path writes it
            if (skip) b = a;
        }
        float4 acc[CPL];
#pragma unroll
        for (int c = 0; c < CPL; ++c) acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int64_t base = a; base < b; base += LPR) {  // uniform within the group
            const int64_t k = base + gl;
            const bool valid = k < b;
            const int32_t nb = valid ? __ldg(nbrs + k) : 0;
            const bool kept = valid && slot_kept(bits, k);
            unsigned ballot = (__ballot_sync(gmask, kept) & gmask) >> (grp * LPR);
            constexpr int QN = CPL > 4 ? 2 : 4;  // neighbour rows in flight per batch (register budget)
            while (ballot) {
                int32_t u[QN];
                int cnt = 0;
#pragma unroll
                for (int q = 0; q < QN; ++q) {
                    if (ballot) {
                        const int sl = __ffs(ballot) - 1;
                        ballot &= ballot - 1;
                        u[q] = __shfl_sync(gmask, nb, grp * LPR + sl);
                        ++cnt;
                    } else {
                        u[q] = -1;
                    }
                }
                float4 vals[QN][CPL];
                float sc[QN];
#pragma unroll
                for (int q = 0; q < QN; ++q) {
                    sc[q] = (kX == 3 && q < cnt) ? __ldg(inv + u[q]) : 1.f;
#pragma unroll
                    for (int c = 0; c < CPL; ++c) {
                        const int32_t ch = gl + LPR * c;
                        vals[q][c] = (q < cnt && ch < H4)
                                         ? __ldg(reinterpret_cast<const float4*>(src + int64_t(u[q]) * H) + ch)
                                         : make_float4(0.f, 0.f, 0.f, 0.f);
                    }
                }
#pragma unroll
                for (int q = 0; q < QN; ++q)
                    if (q < cnt)
#pragma unroll
                        for (int c = 0; c < CPL; ++c) {
                            float4 x = vals[q][c];
                            if (kX == 3) {  // separately rounded products (no FMA contraction): the
                                x.x = __fmul_rn(sc[q], x.x);  // reference's inv_d * dmean.row(v), then +=
                                x.y = __fmul_rn(sc[q], x.y);
                                x.z = __fmul_rn(sc[q], x.z);
                                x.w = __fmul_rn(sc[q], x.w);
                            }
                            acc[c].x += x.x;
                            acc[c].y += x.y;
                            acc[c].z += x.z;
                            acc[c].w += x.w;
                        }
            }
        }
        if (!skip) {
            // finish_row's chunk index is lane + 32 c; here chunk c of this lane is gl + LPR c
#pragma unroll
            for (int c = 0; c < CPL; ++c) {
                float4 one[1] = {acc[c]};
                const int32_t ch = gl + LPR * c;
                if (ch < H4) amx = fmaxf(amx, finish_row<1, kBwd, kPos, kX>(v, ch, H, H4, inv, msg, pos, out, one));
            }
        }
    }
    if (amax_out) {
        amx = warp_max_f(amx);
        if (lane == 0) atomic_max_abs(amax_out, amx);
    }
}

// Skewed degrees (hubs): a row with more than kHeavySlots slots is cut into
// kSegSlots-slot segments, one warp each, whose partial sums are then added in
// segment order by one warp per row (deterministic; the association differs
// from the reference's single running sum only for these rows).
template <int NCH, bool kScale = false>
__global__ void __launch_bounds__(256) spmm_segments_kernel(int32_t nseg, int32_t H, const int64_t* __restrict__ off,
                                                            const int32_t* __restrict__ nbrs,
                                                            const uint32_t* __restrict__ bits,
                                                            const int32_t* __restrict__ seg_row,
                                                            const int64_t* __restrict__ seg_begin,
                                                            const float* __restrict__ src, float* __restrict__ partial,
                                                            const float* __restrict__ inv = nullptr) {
    const int lane = threadIdx.x & 31;
    const int32_t H4 = H >> 2;
    const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
    for (int64_t sg = blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5); sg < nseg; sg += warps) {
        const int64_t a = seg_begin[sg];
        const int64_t b = min(a + int64_t(kSegSlots), off[seg_row[sg] + 1]);
        float4 acc[NCH];
#pragma unroll
        for (int c = 0; c < NCH; ++c) acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
        gather_rows_sum<NCH, kScale>(a, b, lane, H, H4, nbrs, bits, src, acc, inv);
#pragma unroll
        for (int c = 0; c < NCH; ++c)
            if (lane + 32 * c < H4) reinterpret_cast<float4*>(partial + sg * H)[lane + 32 * c] = acc[c];
    }
}

template <int NCH, bool kBwd, bool kPos, int kX = 0>
__global__ void __launch_bounds__(256) spmm_heavy_finish_kernel(int32_t nh, int32_t H,
                                                                const int32_t* __restrict__ rows,
                                                                const int32_t* __restrict__ seg_first,
                                                                const float* __restrict__ partial,
                                                                const float* __restrict__ inv,
                                                                const float* __restrict__ msg,
                                                                const uint32_t* __restrict__ pos,
                                                                float* __restrict__ out, float* amax_out) {
    const int lane = threadIdx.x & 31;
    const int32_t H4 = H >> 2;
    float amx = 0.f;
    const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
    for (int64_t h = blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5); h < nh; h += warps) {
        float4 acc[NCH];
#pragma unroll
        for (int c = 0; c < NCH; ++c) acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int32_t sg = seg_first[h]; sg < seg_first[h + 1]; ++sg)
#pragma unroll
            for (int c = 0; c < NCH; ++c)
                if (lane + 32 * c < H4) {
                    const float4 p = reinterpret_cast<const float4*>(partial + int64_t(sg) * H)[lane + 32 * c];
                    acc[c].x += p.x;
                    acc[c].y += p.y;
                    acc[c].z += p.z;
                    acc[c].w += p.w;
                }
        amx = fmaxf(amx, finish_row<NCH, kBwd, kPos, kX>(rows[h], lane, H, H4, inv, msg, pos, out, acc));
    }
    if (amax_out) {
        amx = warp_max_f(amx);
        if (lane == 0) atomic_max_abs(amax_out, amx);
    }
}

__global__ void heavy_count_kernel(int32_t nh, const int32_t* __restrict__ rows, const int64_t* __restrict__ off,
                                   int32_t* __restrict__ nseg) {
    for (int64_t h = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; h < nh; h += int64_t(gridDim.x) * blockDim.x) {
        const int64_t d = off[rows[h] + 1] - off[rows[h]];
        nseg[h] = static_cast<int32_t>((d + kSegSlots - 1) / kSegSlots);
    }
}
__global__ void heavy_fill_kernel(int32_t nh, const int32_t* __restrict__ rows, const int64_t* __restrict__ off,
                                  const int32_t* __restrict__ seg_first, int32_t* __restrict__ seg_row,
                                  int64_t* __restrict__ seg_begin) {
    for (int64_t h = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; h < nh; h += int64_t(gridDim.x) * blockDim.x) {
        const int32_t v = rows[h];
        for (int32_t sg = seg_first[h], j = 0; sg < seg_first[h + 1]; ++sg, ++j) {
            seg_row[sg] = v;
            seg_begin[sg] = off[v] + int64_t(j) * kSegSlots;
        }
    }
}
struct IsHeavy {
    const int64_t* off;
    __device__ bool operator()(int64_t v) const { return off[v + 1] - off[v] > kHeavySlots; }
};
struct IsMid {
    const int64_t* off;
    __device__ bool operator()(int64_t v) const {
        const int64_t d = off[v + 1] - off[v];
        return d > kNarrowSlots && d <= kHeavySlots;
    }
};

template <bool kBwd>
__global__ void spmm_scalar_kernel(int64_t n, int32_t H, const int64_t* __restrict__ off,
                                   const int32_t* __restrict__ nbrs, const uint32_t* __restrict__ bits,
                                   const float* __restrict__ inv, const float* __restrict__ src,
                                   const float* __restrict__ msg, const uint32_t* __restrict__ pos,
                                   float* __restrict__ out, float* amax_out) {
    const int64_t total = n * H;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t v = i / H;
        const int32_t c = static_cast<int32_t>(i % H);
        float acc = 0.f;
        for (int64_t k = off[v]; k < off[v + 1]; ++k)
            if (slot_kept(bits, k)) acc += src[int64_t(nbrs[k]) * H + c];
        const bool on = !kBwd || (pos ? ((pos[v * ((H + 31) >> 5) + (c >> 5)] >> (c & 31)) & 1u) != 0 : msg[i] > 0.f);
        out[i] = kBwd ? (on ? acc : 0.f) : acc * inv[v];
        if (amax_out) atomic_max_abs(amax_out, out[i]);
    }
}

// rows of H <= 128 floats and <= kNarrowSlots CSR slots run several per warp (spmm_narrow_kernel)
// unless SC_SPMM_NARROW=0
bool narrow_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("SC_SPMM_NARROW");
        return !(e && e[0] == '0');
    }();
    return on;
}

// rows per warp for 68 .. 128-float rows: 8 (4 lanes x 8 chunks, two neighbour rows per batch; default:
// papers-shaped partitions 0.60 -> 0.75 of HBM, profiles/r02_spmm_narrow_ab.txt) or 4 (SC_SPMM_NARROW128=4)
int narrow_wide_rows() {
    static const int r = [] {
        const char* e = std::getenv("SC_SPMM_NARROW128");
        return e ? std::atoi(e) : 8;
    }();
    return r;
}

template <int NCH, bool kBwd, bool kPos, int kX = 0>
void spmm_vec(int64_t n, int32_t H, const int64_t* off, const int32_t* nbrs, const uint32_t* bits, const float* inv,
              const float* src, const float* msg, const uint32_t* pos, float* out, cudaStream_t s, float* amax_out,
              const HeavyRows* hv, float* partial) {
    // 64 blocks of 8 warps per SM: ~13 waves at 5 resident blocks, so the grid-stride tail is short
    // (A/B, profiles/r01_spmm_grid_ab.txt: x16 -> x64 blocks per SM = 0.82 -> 0.92 of HBM peak)
    const bool heavy = hv && hv->nh > 0;
    const int64_t max_slots = heavy ? int64_t(kHeavySlots) : INT64_MAX;
    const int32_t H4 = H / 4;
    if (NCH == 1 && H4 <= 32 && narrow_enabled()) {
        // several rows per warp for rows of at most kNarrowSlots CSR slots (a warp's rows finish together,
        // so long rows — skewed degrees — would hold the other lanes); a warp-per-row pass takes the rest
        const int64_t nmax = std::min<int64_t>(max_slots, kNarrowSlots);
        auto go = [&](auto lpr_tag, auto cpl_tag) {
            constexpr int LPR = decltype(lpr_tag)::value, CPL = decltype(cpl_tag)::value;
            const unsigned grid = grid_for((n + 32 / LPR - 1) / (32 / LPR) * 32, 256, int64_t(num_sms()) * 64);
            spmm_narrow_kernel<LPR, CPL, kBwd, kPos, kX><<<grid, 256, 0, s>>>(n, H, off, nbrs, bits, inv, src, msg,
                                                                              pos, out, amax_out, nmax);
        };
        using I4 = std::integral_constant<int, 4>;
        using I8 = std::integral_constant<int, 8>;
        if (H4 <= 8) go(I4{}, std::integral_constant<int, 2>{});
        else if (H4 <= 12) go(I4{}, std::integral_constant<int, 3>{});
        else if (H4 <= 16) go(I4{}, I4{});
        else if (narrow_wide_rows() == 8) go(I4{}, I8{});  // 128 floats: 8 rows per warp
        else go(I8{}, I4{});
        SC_LAUNCH_CHECK();
        if (hv && hv->built) {  // the mid rows, from their list
            if (hv->nmid > 0 && H4 <= 16) {  // two 16-lane rows per warp (rows of similar length)
                const unsigned grid = grid_for((int64_t(hv->nmid) + 1) / 2 * 32, 256, int64_t(num_sms()) * 64);
                spmm_narrow_kernel<16, 1, kBwd, kPos, kX, true><<<grid, 256, 0, s>>>(
                    hv->nmid, H, off, nbrs, bits, inv, src, msg, pos, out, amax_out, max_slots, hv->mid.get());
                count_launch();
            } else if (hv->nmid > 0) {
                const unsigned grid = grid_for(int64_t(hv->nmid) * 32, 256, int64_t(num_sms()) * 64);
                spmm_kernel<NCH, kBwd, kPos, kX, true><<<grid, 256, 0, s>>>(hv->nmid, H, off, nbrs, bits, inv, src,
                                                                           msg, pos, out, amax_out, max_slots, nmax,
                                                                           hv->mid.get());
                count_launch();
            }
        } else if (max_slots > nmax) {  // no row table: a pass over every row picks them out
            const unsigned grid = grid_for(n * 32, 256, int64_t(num_sms()) * 64);
            spmm_kernel<NCH, kBwd, kPos, kX><<<grid, 256, 0, s>>>(n, H, off, nbrs, bits, inv, src, msg, pos, out,
                                                                 amax_out, max_slots, nmax);
            count_launch();
        }
    } else {
        const unsigned grid = grid_for(n * 32, 256, int64_t(num_sms()) * 64);
        spmm_kernel<NCH, kBwd, kPos, kX><<<grid, 256, 0, s>>>(n, H, off, nbrs, bits, inv, src, msg, pos, out,
                                                             amax_out, max_slots);
    }
    SC_LAUNCH_CHECK();
    count_launch();
    if (!heavy) return;
    spmm_segments_kernel<NCH, kX == 3><<<grid_for(int64_t(hv->nseg) * 32, 256, int64_t(num_sms()) * 16), 256, 0, s>>>(
        hv->nseg, H, off, nbrs, bits, hv->seg_row.get(), hv->seg_begin.get(), src, partial, inv);
    SC_LAUNCH_CHECK();
    spmm_heavy_finish_kernel<NCH, kBwd, kPos, kX><<<grid_for(int64_t(hv->nh) * 32, 256), 256, 0, s>>>(
        hv->nh, H, hv->rows.get(), hv->seg_first.get(), partial, inv, msg, pos, out, amax_out);
    SC_LAUNCH_CHECK();
    count_launch(2);
}

// the ReLU-bits variant is a separate instantiation: the msg path keeps its own code
template <int NCH, bool kBwd>
void spmm_vec_pos(int64_t n, int32_t H, const int64_t* off, const int32_t* nbrs, const uint32_t* bits,
                  const float* inv, const float* src, const float* msg, const uint32_t* pos, float* out,
                  cudaStream_t s, float* amax_out, const HeavyRows* hv, float* partial) {
    if (kBwd && pos) spmm_vec<NCH, kBwd, true>(n, H, off, nbrs, bits, inv, src, msg, pos, out, s, amax_out, hv, partial);
    else spmm_vec<NCH, kBwd, false>(n, H, off, nbrs, bits, inv, src, msg, pos, out, s, amax_out, hv, partial);
}

template <bool kBwd>
void spmm_launch(int64_t n, int32_t H, const int64_t* off, const int32_t* nbrs, const uint32_t* bits, const float* inv,
                 const float* src, const float* msg, const uint32_t* pos, float* out, cudaStream_t s,
                 float* amax_out, const HeavyRows* hv, float* partial) {
    if (n <= 0) return;
    if (H % 4 != 0) {  // scalar fallback: thread per output element (any H, any degree)
        spmm_scalar_kernel<kBwd><<<grid_for(n * H, 256), 256, 0, s>>>(n, H, off, nbrs, bits, inv, src, msg, pos, out,
                                                                      amax_out);
        SC_LAUNCH_CHECK();
        count_launch();
        return;
    }
    const int nch = (H / 4 + 31) / 32;
    if (nch <= 1) spmm_vec_pos<1, kBwd>(n, H, off, nbrs, bits, inv, src, msg, pos, out, s, amax_out, hv, partial);
    else if (nch == 2) spmm_vec_pos<2, kBwd>(n, H, off, nbrs, bits, inv, src, msg, pos, out, s, amax_out, hv, partial);
    else if (nch <= 4) spmm_vec_pos<4, kBwd>(n, H, off, nbrs, bits, inv, src, msg, pos, out, s, amax_out, hv, partial);
    else spmm_vec_pos<8, kBwd>(n, H, off, nbrs, bits, inv, src, msg, pos, out, s, amax_out, hv, partial);
}

// The composed top layer's aggregations (kX = 1, 2; H a multiple of 4, the padded class count).
template <int kX>
void spmm_variant(int64_t n, int32_t H, const int64_t* off, const int32_t* nbrs, const uint32_t* bits,
                  const float* inv, const float* src, float* out, cudaStream_t s, float* amax_out, const HeavyRows* hv,
                  float* partial) {
    if (n <= 0) return;
    if (H % 4 != 0) throw std::logic_error("spmm variant: row width must be a multiple of 4");
    const int nch = (H / 4 + 31) / 32;
    constexpr bool kB = kX >= 2;
    if (nch <= 1) spmm_vec<1, kB, false, kX>(n, H, off, nbrs, bits, inv, src, nullptr, nullptr, out, s, amax_out, hv, partial);
    else if (nch == 2) spmm_vec<2, kB, false, kX>(n, H, off, nbrs, bits, inv, src, nullptr, nullptr, out, s, amax_out, hv, partial);
    else if (nch <= 4) spmm_vec<4, kB, false, kX>(n, H, off, nbrs, bits, inv, src, nullptr, nullptr, out, s, amax_out, hv, partial);
    else spmm_vec<8, kB, false, kX>(n, H, off, nbrs, bits, inv, src, nullptr, nullptr, out, s, amax_out, hv, partial);
}

__global__ void mask_bits_kernel(int64_t nnz, const int32_t* __restrict__ eids, const uint8_t* __restrict__ mask,
                                 uint32_t* bits) {
    const int64_t words = (nnz + 31) / 32;
    for (int64_t w = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; w < words; w += int64_t(gridDim.x) * blockDim.x) {
        uint32_t x = 0;
        for (int b = 0; b < 32; ++b) {
            const int64_t k = w * 32 + b;
            if (k < nnz && mask[eids[k]]) x |= 1u << b;
        }
        bits[w] = x;
    }
}

// ---------------------------------------------------------------------------
// Loss (warp per row).
// ---------------------------------------------------------------------------
__device__ __forceinline__ float warp_max(float x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, o));
    return x;
}
__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}
__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long x) {
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}
__device__ __forceinline__ double warp_sum_d(double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

__global__ void softmax_ce_kernel(int64_t n, int32_t C, int32_t ld, const float* __restrict__ logits,
                                  const int32_t* __restrict__ labels, const int32_t* __restrict__ rows,
                                  const double* __restrict__ w, const float* __restrict__ scale, float* G,
                                  double* row_loss) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
    for (int64_t r = blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += warps) {
        const float* z = logits + r * ld;
        float* g = G + r * ld;
        const double wr = w[r];
        for (int32_t c = C + lane; c < ld; c += 32) g[c] = 0.f;  // padding columns (row stride ld)
        if (wr == 0.0) {  // nn.hpp:330 rows with zero weight contribute nothing
            for (int32_t c = lane; c < C; c += 32) g[c] = 0.f;
            if (lane == 0) row_loss[r] = 0.0;
            continue;
        }
        const int32_t y = labels[rows ? rows[r] : r];
        float mx = -INFINITY;
        for (int32_t c = lane; c < C; c += 32) mx = fmaxf(mx, z[c]);
        mx = warp_max(mx);
        float se = 0.f;
        for (int32_t c = lane; c < C; c += 32) se += expf(z[c] - mx);
        se = warp_sum(se);
        const float lse = mx + logf(se);
        const float sc = scale[r];
        for (int32_t c = lane; c < C; c += 32) g[c] = sc * (expf(z[c] - lse) - (c == y ? 1.f : 0.f));
        if (lane == 0) row_loss[r] = wr * static_cast<double>(lse - z[y]);
    }
}

// Thread per row for C <= 4 * NV (the bench's 47 classes: 12 float4 per row):
// the row lives in registers, max / sum-exp run sequentially in column order
// exactly like nn.hpp:333-336, and the gradient row is written with 16-byte
// stores (padding columns zeroed). Warp-per-row above handles wide C.
template <int NV>
__global__ void __launch_bounds__(128) softmax_ce_rows_kernel(int64_t n, int32_t C, int32_t ld,
                                                              const float* __restrict__ logits,
                                                              const int32_t* __restrict__ labels,
                                                              const int32_t* __restrict__ rows,
                                                              const double* __restrict__ w,
                                                              const float* __restrict__ scale, float* __restrict__ G,
                                                              double* __restrict__ row_loss) {
    const int32_t nv = ld >> 2;  // float4 per (padded) row
    for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < n; r += int64_t(gridDim.x) * blockDim.x) {
        float4* g = reinterpret_cast<float4*>(G + r * ld);
        const double wr = w[r];
        if (wr == 0.0) {  // nn.hpp:330
#pragma unroll
            for (int j = 0; j < NV; ++j)
                if (j < nv) g[j] = make_float4(0.f, 0.f, 0.f, 0.f);
            row_loss[r] = 0.0;
            continue;
        }
        const float4* zr = reinterpret_cast<const float4*>(logits + r * ld);
        float z[4 * NV];
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            const float4 v = j < nv ? __ldg(zr + j) : make_float4(0.f, 0.f, 0.f, 0.f);
            z[4 * j] = v.x;
            z[4 * j + 1] = v.y;
            z[4 * j + 2] = v.z;
            z[4 * j + 3] = v.w;
        }
        const int32_t y = labels[rows ? rows[r] : r];
        float mx = -INFINITY;
#pragma unroll
        for (int c = 0; c < 4 * NV; ++c)
            if (c < C) mx = fmaxf(mx, z[c]);
        float se = 0.f;
#pragma unroll
        for (int c = 0; c < 4 * NV; ++c)
            if (c < C) se += expf(z[c] - mx);
        const float lse = mx + logf(se);
        const float sc = scale[r];
        float zy = 0.f;
#pragma unroll
        for (int c = 0; c < 4 * NV; ++c) {
            if (c == y) zy = z[c];
            z[c] = c < C ? sc * (expf(z[c] - lse) - (c == y ? 1.f : 0.f)) : 0.f;
        }
#pragma unroll
        for (int j = 0; j < NV; ++j)
            if (j < nv) g[j] = make_float4(z[4 * j], z[4 * j + 1], z[4 * j + 2], z[4 * j + 3]);
        row_loss[r] = wr * static_cast<double>(lse - zy);
    }
}

// Warp per row for 64 < C <= 32 NV (e.g. 172 classes): the row lives in registers (lane l holds
// columns l, l + 32, ...), so logits are read once; the same per-lane column order and butterfly
// reductions as softmax_ce_kernel (identical bits).
template <int NV>
__global__ void softmax_ce_warp_regs_kernel(int64_t n, int32_t C, int32_t ld, const float* __restrict__ logits,
                                            const int32_t* __restrict__ labels, const int32_t* __restrict__ rows,
                                            const double* __restrict__ w, const float* __restrict__ scale, float* G,
                                            double* row_loss) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
    for (int64_t r = blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += warps) {
        const float* z = logits + r * ld;
        float* g = G + r * ld;
        const double wr = w[r];
        for (int32_t c = C + lane; c < ld; c += 32) g[c] = 0.f;  // padding columns (row stride ld)
        if (wr == 0.0) {  // nn.hpp:330
            for (int32_t c = lane; c < C; c += 32) g[c] = 0.f;
            if (lane == 0) row_loss[r] = 0.0;
            continue;
        }
        float zr[NV];
#pragma unroll
        for (int j = 0; j < NV; ++j) zr[j] = (lane + 32 * j < C) ? z[lane + 32 * j] : -INFINITY;
        const int32_t y = labels[rows ? rows[r] : r];
        float mx = -INFINITY;
#pragma unroll
        for (int j = 0; j < NV; ++j)
            if (lane + 32 * j < C) mx = fmaxf(mx, zr[j]);
        mx = warp_max(mx);
        float se = 0.f;
#pragma unroll
        for (int j = 0; j < NV; ++j)
            if (lane + 32 * j < C) se += expf(zr[j] - mx);
        se = warp_sum(se);
        const float lse = mx + logf(se);
        const float sc = scale[r];
        float zy = 0.f;
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            const int32_t c = lane + 32 * j;
            if (c < C) {
                if (c == y) zy = zr[j];
                g[c] = sc * (expf(zr[j] - lse) - (c == y ? 1.f : 0.f));
            }
        }
        zy = __shfl_sync(0xffffffffu, zy, y & 31);
        if (lane == 0) row_loss[r] = wr * static_cast<double>(lse - zy);
    }
}

// targets (optional): the graph's n x C 0/1 multi-label matrix (graph.hpp:64);
// without it the target row is the one-hot of the class id (label_targets,
// graph.cpp:91-98).
__global__ void bce_kernel(int64_t n, int32_t C, int32_t ld, const float* __restrict__ logits,
                           const int32_t* __restrict__ labels, const uint8_t* __restrict__ targets,
                           const int32_t* __restrict__ rows, const double* __restrict__ w,
                           const float* __restrict__ scale, float* G, double* row_loss) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
    for (int64_t r = blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += warps) {
        const float* z = logits + r * ld;
        float* g = G + r * ld;
        const double wr = w[r];
        for (int32_t c = C + lane; c < ld; c += 32) g[c] = 0.f;  // padding columns (row stride ld)
        if (wr == 0.0) {
            for (int32_t c = lane; c < C; c += 32) g[c] = 0.f;
            if (lane == 0) row_loss[r] = 0.0;
            continue;
        }
        const int64_t node = rows ? rows[r] : r;
        const int32_t yl = targets ? -1 : labels[node];
        const uint8_t* trow = targets ? targets + node * C : nullptr;
        const float sc = scale[r];
        double acc = 0.0;
        for (int32_t c = lane; c < C; c += 32) {
            const float zc = z[c];
            const float y = trow ? static_cast<float>(trow[c]) : (c == yl ? 1.f : 0.f);
            const float sp = fmaxf(zc, 0.f) + log1pf(expf(-fabsf(zc)));
            acc += wr * static_cast<double>(sp - zc * y);
            const float sg = zc >= 0.f ? 1.f / (1.f + expf(-zc)) : expf(zc) / (1.f + expf(zc));
            g[c] = sc * (sg - y);
        }
        acc = warp_sum_d(acc);
        if (lane == 0) row_loss[r] = acc;
    }
}

constexpr int kRedBlocks = 512;
constexpr int kRedThreads = 256;

__global__ void sum_f64_partial_kernel(int64_t n, const double* __restrict__ x, double* partial) {
    __shared__ double sh[kRedThreads];
    double acc = 0.0;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        acc += x[i];
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int s = kRedThreads / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}
__global__ void sum_f64_final_kernel(const double* partial, int nb, double* out, double divisor) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double acc = 0.0;
        for (int i = 0; i < nb; ++i) acc += partial[i];
        *out = acc / divisor;
    }
}

// Gradient slots are bucket-major (one bucket per parameter matrix, in
// for_each_matrix order): bucket b holds pp consecutive per-partition copies of
// its len_b floats, so one all-gather per (round, bucket) exchanges a
// contiguous range. Element k of bucket b for partition i lives at
// b_off[b] * pp + i * len_b + (k - b_off[b]).
__global__ void gather_kernel(int64_t P, int32_t p, int32_t pp, int32_t nb, const int64_t* __restrict__ b_off,
                              const float* __restrict__ slots, float* gathered, double* partial, int* nonfinite) {
    __shared__ double sh[kRedThreads];
    double acc = 0.0;
    bool bad = false;
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < P; k += int64_t(gridDim.x) * blockDim.x) {
        int32_t lo = 0, hi = nb - 1;  // last bucket with b_off <= k
        while (lo < hi) {
            const int32_t mid = (lo + hi + 1) >> 1;
            if (b_off[mid] <= k) lo = mid;
            else hi = mid - 1;
        }
        const int64_t o = b_off[lo], len = b_off[lo + 1] - o;
        const float* src = slots + o * pp + (k - o);
        float g = src[0];
        for (int32_t i = 1; i < p; ++i) g += src[int64_t(i) * len];  // ascending partition order (trainer.hpp:79-94)
        gathered[k] = g;
        bad |= !isfinite(g);
        acc += static_cast<double>(g) * static_cast<double>(g);
    }
    if (bad) *nonfinite = 1;
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int s = kRedThreads / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}

__global__ void finalize_kernel(const double* partial, int nb, const double* part_loss, int32_t p, double* out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double sq = 0.0;
        for (int i = 0; i < nb; ++i) sq += partial[i];
        double l = 0.0;
        for (int32_t i = 0; i < p; ++i) l += part_loss[i];
        out[0] = sqrt(sq);
        out[1] = l;
    }
}

__global__ void adam_kernel(int64_t P, float* theta, float* m1, float* m2, const float* __restrict__ g, float b1,
                            float b2, float c1, float c2, float lr, float eps, const int* nonfinite) {
    if (*nonfinite) return;  // adam_step throws before touching anything (nn.hpp:404)
    const float ob1 = 1.f - b1, ob2 = 1.f - b2;
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < P; k += int64_t(gridDim.x) * blockDim.x) {
        const float gi = g[k];
        // Separate multiply/add roundings as in the reference (no FMA contraction).
        const float m = __fadd_rn(__fmul_rn(b1, m1[k]), __fmul_rn(ob1, gi));
        const float v = __fadd_rn(__fmul_rn(b2, m2[k]), __fmul_rn(ob2, __fmul_rn(gi, gi)));
        m1[k] = m;
        m2[k] = v;
        const float mh = __fdiv_rn(m, c1), vh = __fdiv_rn(v, c2);
        theta[k] = __fsub_rn(theta[k], __fdiv_rn(__fmul_rn(lr, mh), __fadd_rn(__fsqrt_rn(vh), eps)));
    }
}

__global__ void correct_kernel(int64_t n, int32_t C, int32_t ld, const float* __restrict__ logits,
                               const int32_t* __restrict__ labels,
                               const uint8_t* __restrict__ mask, unsigned long long* out) {
    unsigned long long corr = 0, tot = 0;
    for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < n; r += int64_t(gridDim.x) * blockDim.x) {
        if (!mask[r]) continue;
        ++tot;
        const float* z = logits + r * ld;
        int32_t best = 0;
        for (int32_t c = 1; c < C; ++c)
            if (z[c] > z[best]) best = c;
        corr += best == labels[r];
    }
    atomicAdd(&out[0], corr);
    atomicAdd(&out[1], tot);
}

// Micro-F1 counts over masked rows (trainer.cpp:72-87): prediction = logit > 0,
// truth = target != 0; out[0..2] += (tp, fp, fn), out[3] += masked rows.
__global__ void f1_counts_kernel(int64_t n, int32_t C, int32_t ld, const float* __restrict__ logits,
                                 const uint8_t* __restrict__ targets, const uint8_t* __restrict__ mask,
                                 unsigned long long* out) {
    unsigned long long tp = 0, fp = 0, fn = 0, tot = 0;
    const int64_t total = n * C;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = i / C;
        const int32_t c = static_cast<int32_t>(i - r * C);
        if (!mask[r]) continue;
        tot += c == 0;
        const bool pred = logits[r * ld + c] > 0.f;
        const bool truth = targets[i] != 0;
        tp += pred && truth;
        fp += pred && !truth;
        fn += !pred && truth;
    }
    tp = warp_sum_u64(tp);
    fp = warp_sum_u64(fp);
    fn = warp_sum_u64(fn);
    tot = warp_sum_u64(tot);
    if ((threadIdx.x & 31) == 0 && (tp | fp | fn | tot)) {
        atomicAdd(&out[0], tp);
        atomicAdd(&out[1], fp);
        atomicAdd(&out[2], fn);
        atomicAdd(&out[3], tot);
    }
}

}  // namespace

void gemm_nt(const MatA& a1, const MatB& b1, const MatA* a2, const MatB* b2, float* C, int64_t ldc, int64_t M,
             int32_t N, int epi, const float* row_scale, cudaStream_t s, float* amax_out, const float* mask_msg,
             const uint32_t* mask_pos) {
    if (M <= 0 || N <= 0) return;
    GemmArgs args{};
    args.amax_out = amax_out;
    args.mask_msg = mask_msg;
    args.mask_pos = mask_pos;
    args.a[0] = a1;
    args.b[0] = b1;
    args.nsrc = 1;
    if (a2) {
        args.a[1] = *a2;
        args.b[1] = *b2;
        args.nsrc = 2;
    }
    args.C = C;
    args.ldc = ldc;
    args.M = M;
    args.N = N;
    args.epi = epi;
    args.row_scale = row_scale;
    dim3 grid(static_cast<unsigned>((M + BM - 1) / BM), static_cast<unsigned>((N + BN - 1) / BN));
    gemm_nt_kernel<<<grid, NT, 0, s>>>(args);
    SC_LAUNCH_CHECK();
    count_launch();
}

int64_t gemm_tn_workspace_floats(int32_t N1, int32_t N2) { return int64_t(kMaxSplits) * N1 * N2; }

void gemm_tn(const MatT& a, const MatT& b1, const MatT* b2, int64_t M, float* C, int64_t ldc, float* ws,
             int64_t ws_floats, cudaStream_t s) {
    const int32_t N1 = a.cols, N2 = b1.cols + (b2 ? b2->cols : 0);
    if (N1 <= 0 || N2 <= 0) return;
    if (M <= 0) {  // no rows: zero gradient
        for (int32_t r = 0; r < N1; ++r) SC_CUDA(cudaMemsetAsync(C + int64_t(r) * ldc, 0, sizeof(float) * N2, s));
        return;
    }
    const int32_t S = tn_splits(N1, N2, M);
    if (int64_t(S) * N1 * N2 > ws_floats) throw std::logic_error("gemm_tn: workspace too small");
    TnArgs args{};
    args.a = a;
    args.b[0] = b1;
    if (b2) args.b[1] = *b2;
    args.n2a = b1.cols;
    args.N1 = N1;
    args.N2 = N2;
    args.M = M;
    args.rows_per_split = ((M + S - 1) / S + BK - 1) / BK * BK;
    args.ws = ws;
    const int32_t tiles = ((N1 + BM - 1) / BM) * ((N2 + BN - 1) / BN);
    gemm_tn_kernel<<<dim3(tiles, S), NT, 0, s>>>(args);
    SC_LAUNCH_CHECK();
    splitk_reduce_kernel<<<grid_for(int64_t(N1) * N2, 256), 256, 0, s>>>(S, N1, N2, ws, C, ldc);
    SC_LAUNCH_CHECK();
    count_launch(2);
}

void inv_degree(int64_t n, const int64_t* offsets, const uint32_t* bits, float* inv, cudaStream_t s) {
    if (n <= 0) return;
    inv_degree_kernel<<<grid_for(n, 256), 256, 0, s>>>(n, offsets, bits, inv);
    SC_LAUNCH_CHECK();
    count_launch();
}
void spmm_fwd(int64_t n, int32_t H, const int64_t* offsets, const int32_t* nbrs, const uint32_t* bits, const float* inv,
              const float* msg, float* mean, cudaStream_t s, const HeavyRows* hv, float* partial) {
    spmm_launch<false>(n, H, offsets, nbrs, bits, inv, msg, nullptr, nullptr, mean, s, nullptr, hv, partial);
}
void spmm_fwd_add(int64_t n, int32_t H, const int64_t* offsets, const int32_t* nbrs, const uint32_t* bits,
                  const float* inv, const float* src, float* out, cudaStream_t s, const HeavyRows* hv, float* partial) {
    spmm_variant<1>(n, H, offsets, nbrs, bits, inv, src, out, s, nullptr, hv, partial);
}
void spmm_sum_scaled(int64_t n, int32_t H, const int64_t* offsets, const int32_t* nbrs, const uint32_t* bits,
                     const float* inv, const float* src, float* out, cudaStream_t s, float* amax_out,
                     const HeavyRows* hv, float* partial) {
    spmm_variant<3>(n, H, offsets, nbrs, bits, inv, src, out, s, amax_out, hv, partial);
}
void spmm_bwd(int64_t n, int32_t H, const int64_t* offsets, const int32_t* nbrs, const uint32_t* bits,
              const float* dmean_s, const float* msg, float* dz, cudaStream_t s, float* amax_out, const HeavyRows* hv,
              float* partial, const uint32_t* relu_pos) {
    spmm_launch<true>(n, H, offsets, nbrs, bits, nullptr, dmean_s, msg, relu_pos, dz, s, amax_out, hv, partial);
}

__global__ void relu_sign_bits_kernel(int64_t M, int32_t N, const float* __restrict__ C, int64_t ldc,
                                      uint32_t* __restrict__ pos) {
    const int32_t W = (N + 31) >> 5;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < M * W; i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = i / W;
        const int32_t w = static_cast<int32_t>(i - r * W);
        uint32_t b = 0;
        for (int q = 0; q < 32 && 32 * w + q < N; ++q) b |= (C[r * ldc + 32 * w + q] > 0.f ? 1u : 0u) << q;
        pos[i] = b;
    }
}
void relu_sign_bits(int64_t M, int32_t N, const float* C, int64_t ldc, uint32_t* pos, cudaStream_t s) {
    if (M <= 0 || N <= 0) return;
    relu_sign_bits_kernel<<<grid_for(M * ((N + 31) / 32), 256), 256, 0, s>>>(M, N, C, ldc, pos);
    SC_LAUNCH_CHECK();
    count_launch();
}

void build_heavy_rows(sc_ctx* ctx, int64_t n, const int64_t* off, HeavyRows& hv) {
    cudaStream_t s = ctx->stream;
    hv.nh = hv.nseg = hv.nmid = 0;
    hv.built = true;
    if (n <= 0) return;
    DevBuf<int32_t> cnt(1);
    hv.rows.alloc(1);
    cub::CountingInputIterator<int64_t> it(0);
    {  // mid rows (warp-per-row pass next to the narrow kernel)
        cub::TransformInputIterator<bool, IsMid, cub::CountingInputIterator<int64_t>> mflags(it, IsMid{off});
        DevBuf<int32_t> midx(n);
        cub::CountingInputIterator<int32_t> ids(0);
        size_t tmp = 0;
        SC_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, ids, mflags, midx.get(), cnt.get(), n, s));
        SC_CUDA(cub::DeviceSelect::Flagged(ctx->temp(tmp), tmp, ids, mflags, midx.get(), cnt.get(), n, s));
        int32_t nm = 0;
        d2h(&nm, cnt.get(), 1, s);
        SC_CUDA(cudaStreamSynchronize(s));
        count_launch(1);
        if (nm > 0) {
            hv.mid.alloc(nm);
            SC_CUDA(cudaMemcpyAsync(hv.mid.get(), midx.get(), sizeof(int32_t) * nm, cudaMemcpyDeviceToDevice, s));
            SC_CUDA(cudaStreamSynchronize(s));
        }
        hv.nmid = nm;
    }
    IsHeavy pred{off};
    // pass 1: count heavy rows
    cub::TransformInputIterator<bool, IsHeavy, cub::CountingInputIterator<int64_t>> flags(it, pred);
    DevBuf<int32_t> idx(n);
    cub::CountingInputIterator<int32_t> ids(0);
    size_t tmp = 0;
    SC_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, ids, flags, idx.get(), cnt.get(), n, s));
    SC_CUDA(cub::DeviceSelect::Flagged(ctx->temp(tmp), tmp, ids, flags, idx.get(), cnt.get(), n, s));
    int32_t nh = 0;
    d2h(&nh, cnt.get(), 1, s);
    SC_CUDA(cudaStreamSynchronize(s));
    count_launch(1);
    if (nh == 0) return;
    hv.rows.alloc(nh);
    SC_CUDA(cudaMemcpyAsync(hv.rows.get(), idx.get(), sizeof(int32_t) * nh, cudaMemcpyDeviceToDevice, s));
    hv.seg_first.alloc(nh + 1);
    DevBuf<int32_t> nseg(nh + 1);
    heavy_count_kernel<<<grid_for(nh, 256), 256, 0, s>>>(nh, hv.rows.get(), off, nseg.get());
    SC_LAUNCH_CHECK();
    SC_CUDA(cudaMemsetAsync(nseg.get() + nh, 0, sizeof(int32_t), s));
    tmp = 0;
    SC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, nseg.get(), hv.seg_first.get(), nh + 1, s));
    SC_CUDA(cub::DeviceScan::ExclusiveSum(ctx->temp(tmp), tmp, nseg.get(), hv.seg_first.get(), nh + 1, s));
    int32_t total = 0;
    d2h(&total, hv.seg_first.get() + nh, 1, s);
    SC_CUDA(cudaStreamSynchronize(s));
    hv.seg_row.alloc(total);
    hv.seg_begin.alloc(total);
    heavy_fill_kernel<<<grid_for(nh, 256), 256, 0, s>>>(nh, hv.rows.get(), off, hv.seg_first.get(), hv.seg_row.get(),
                                                        hv.seg_begin.get());
    SC_LAUNCH_CHECK();
    count_launch(3);
    hv.nh = nh;
    hv.nseg = total;
}
__global__ void gather_rows_pad_kernel(int64_t n, int32_t d, int32_t dp, const int32_t* __restrict__ rows,
                                       const float* __restrict__ src, float* __restrict__ dst) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n * dp; i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = i / dp;
        const int32_t c = static_cast<int32_t>(i - r * dp);
        dst[i] = c < d ? __ldg(src + (rows ? int64_t(rows[r]) : r) * d + c) : 0.f;
    }
}

void gather_rows(int64_t n, int32_t d, const int32_t* rows, const float* src, float* dst, cudaStream_t s,
                 int32_t dst_ld) {
    if (n <= 0) return;
    if (dst_ld > d) {  // padded destination rows (zeros beyond d)
        gather_rows_pad_kernel<<<grid_for(n * dst_ld, 256, int64_t(num_sms()) * 64), 256, 0, s>>>(n, d, dst_ld, rows,
                                                                                                   src, dst);
        SC_LAUNCH_CHECK();
        count_launch();
        return;
    }
    if (d % 4 == 0 && reinterpret_cast<uintptr_t>(src) % 16 == 0 && reinterpret_cast<uintptr_t>(dst) % 16 == 0)
        gather_rows4_kernel<<<grid_for(n * (d / 4), 256, int64_t(num_sms()) * 64), 256, 0, s>>>(
            n, d / 4, rows, reinterpret_cast<const float4*>(src), reinterpret_cast<float4*>(dst));
    else
        gather_rows_kernel<<<grid_for(n * d, 256), 256, 0, s>>>(n, d, rows, src, dst);
    SC_LAUNCH_CHECK();
    count_launch();
}
// ---- small weight-space products (the composed top layer, trainer.cu) --------------------------
// C[M x N] = op(A) op(B): a(i, k) = ta ? A[k lda + i] : A[i lda + k], b(k, j) = tb ? B[j ldb + k] :
// B[k ldb + j]. fp64 accumulation, k ascending per lane, fixed-shape lane reduction: deterministic.
// (!ta, tb): k is contiguous in both operands -> a warp per output, lanes stride k; otherwise a
// thread per output with j across the warp (coalesced B rows, broadcast A).
namespace {
__global__ void small_gemm_warp_kernel(int M, int N, int K, const float* __restrict__ A, int64_t lda,
                                       const float* __restrict__ B, int64_t ldb, float* C, int64_t ldc) {
    const int64_t w = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= int64_t(M) * N) return;
    const int i = static_cast<int>(w / N), j = static_cast<int>(w % N);
    double acc = 0.0;
    for (int k = lane; k < K; k += 32) acc += double(A[i * lda + k]) * double(B[j * ldb + k]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) C[i * ldc + j] = static_cast<float>(acc);
}
__global__ void small_gemm_thread_kernel(int M, int N, int K, const float* __restrict__ A, int64_t lda, bool ta,
                                         const float* __restrict__ B, int64_t ldb, bool tb, float* C, int64_t ldc) {
    const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (t >= int64_t(M) * N) return;
    const int i = static_cast<int>(t / N), j = static_cast<int>(t % N);
    double acc = 0.0;
    for (int k = 0; k < K; ++k) {
        const float a = ta ? A[int64_t(k) * lda + i] : A[i * lda + k];
        const float b = tb ? B[j * ldb + k] : B[int64_t(k) * ldb + j];
        acc += double(a) * double(b);
    }
    C[i * ldc + j] = static_cast<float>(acc);
}
}  // namespace

void small_gemm(int M, int N, int K, const float* A, int64_t lda, bool ta, const float* B, int64_t ldb, bool tb,
                float* C, int64_t ldc, cudaStream_t s) {
    const int64_t outs = int64_t(M) * N;
    if (outs <= 0) return;
    if (!ta && tb) {
        small_gemm_warp_kernel<<<static_cast<unsigned>((outs * 32 + 255) / 256), 256, 0, s>>>(M, N, K, A, lda, B, ldb,
                                                                                              C, ldc);
    } else {
        small_gemm_thread_kernel<<<static_cast<unsigned>((outs + 255) / 256), 256, 0, s>>>(M, N, K, A, lda, ta, B, ldb,
                                                                                          tb, C, ldc);
    }
    SC_LAUNCH_CHECK();
    count_launch();
}

void absmax(int64_t n, const float* x, float* out, cudaStream_t s) {
    if (n <= 0) return;
    absmax_kernel<<<grid_for(n, 256), 256, 0, s>>>(n, x, out);
    SC_LAUNCH_CHECK();
    count_launch();
}
void mask_to_bits(int64_t nnz, const int32_t* eids, const uint8_t* mask, uint32_t* bits, cudaStream_t s) {
    if (nnz <= 0) return;
    mask_bits_kernel<<<grid_for((nnz + 31) / 32, 256), 256, 0, s>>>(nnz, eids, mask, bits);
    SC_LAUNCH_CHECK();
    count_launch();
}
void softmax_ce(int64_t n, int32_t C, int32_t ld, const float* logits, const int32_t* labels, const int32_t* rows, const double* w,
                const float* scale, float* G, double* row_loss, cudaStream_t s) {
    if (n <= 0) return;
    const bool vec = ld % 4 == 0 && reinterpret_cast<uintptr_t>(logits) % 16 == 0 &&
                     reinterpret_cast<uintptr_t>(G) % 16 == 0;
    const unsigned grid = grid_for(n, 128);
    if (vec && ld <= 16)
        softmax_ce_rows_kernel<4><<<grid, 128, 0, s>>>(n, C, ld, logits, labels, rows, w, scale, G, row_loss);
    else if (vec && ld <= 32)
        softmax_ce_rows_kernel<8><<<grid, 128, 0, s>>>(n, C, ld, logits, labels, rows, w, scale, G, row_loss);
    else if (vec && ld <= 48)
        softmax_ce_rows_kernel<12><<<grid, 128, 0, s>>>(n, C, ld, logits, labels, rows, w, scale, G, row_loss);
    else if (vec && ld <= 64)
        softmax_ce_rows_kernel<16><<<grid, 128, 0, s>>>(n, C, ld, logits, labels, rows, w, scale, G, row_loss);
    else if (C <= 128)
        softmax_ce_warp_regs_kernel<4><<<grid_for(n * 32, 256), 256, 0, s>>>(n, C, ld, logits, labels, rows, w, scale,
                                                                            G, row_loss);
    else if (C <= 256)
        softmax_ce_warp_regs_kernel<8><<<grid_for(n * 32, 256), 256, 0, s>>>(n, C, ld, logits, labels, rows, w, scale,
                                                                            G, row_loss);
    else
        softmax_ce_kernel<<<grid_for(n * 32, 256), 256, 0, s>>>(n, C, ld, logits, labels, rows, w, scale, G,
                                                                  row_loss);
    SC_LAUNCH_CHECK();
    count_launch();
}
void bce(int64_t n, int32_t C, int32_t ld, const float* logits, const int32_t* labels, const uint8_t* targets,
         const int32_t* rows, const double* w, const float* scale, float* G, double* row_loss, cudaStream_t s) {
    if (n <= 0) return;
    bce_kernel<<<grid_for(n * 32, 256), 256, 0, s>>>(n, C, ld, logits, labels, targets, rows, w, scale, G, row_loss);
    SC_LAUNCH_CHECK();
    count_launch();
}
void sum_f64(int64_t n, const double* x, double* partial, double* out, double divisor, cudaStream_t s) {
    sum_f64_partial_kernel<<<kRedBlocks, kRedThreads, 0, s>>>(n, x, partial);
    SC_LAUNCH_CHECK();
    sum_f64_final_kernel<<<1, 32, 0, s>>>(partial, kRedBlocks, out, divisor);
    SC_LAUNCH_CHECK();
    count_launch(2);
}
void gather_grads(int64_t P, int32_t p, int32_t pp, int32_t nb, const int64_t* b_off, const float* slots,
                  float* gathered, double* partial, int* nonfinite, cudaStream_t s) {
    gather_kernel<<<kRedBlocks, kRedThreads, 0, s>>>(P, p, pp, nb, b_off, slots, gathered, partial, nonfinite);
    SC_LAUNCH_CHECK();
    count_launch();
}
void finalize_step(const double* partial, const double* part_loss, int32_t p, double* out, cudaStream_t s) {
    finalize_kernel<<<1, 32, 0, s>>>(partial, kRedBlocks, part_loss, p, out);
    SC_LAUNCH_CHECK();
    count_launch();
}
void adam(int64_t P, float* theta, float* m1, float* m2, const float* g, float b1, float b2, float c1, float c2,
          float lr, float eps, const int* nonfinite, cudaStream_t s) {
    adam_kernel<<<grid_for(P, 256), 256, 0, s>>>(P, theta, m1, m2, g, b1, b2, c1, c2, lr, eps, nonfinite);
    SC_LAUNCH_CHECK();
    count_launch();
}
void count_correct(int64_t n, int32_t C, int32_t ld, const float* logits, const int32_t* labels, const uint8_t* mask,
                   unsigned long long* out, cudaStream_t s) {
    if (n <= 0) return;
    correct_kernel<<<grid_for(n, 256), 256, 0, s>>>(n, C, ld, logits, labels, mask, out);
    SC_LAUNCH_CHECK();
    count_launch();
}

void f1_counts(int64_t n, int32_t C, int32_t ld, const float* logits, const uint8_t* targets, const uint8_t* mask,
               unsigned long long* out, cudaStream_t s) {
    if (n <= 0 || C <= 0) return;
    f1_counts_kernel<<<grid_for(n * C, 256), 256, 0, s>>>(n, C, ld, logits, targets, mask, out);
    SC_LAUNCH_CHECK();
    count_launch();
}

}  // namespace sc
