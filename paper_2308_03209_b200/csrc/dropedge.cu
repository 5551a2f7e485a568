// dropedge.cu — DropEdge-K masks on the device, bit-exact with the reference.
//
// Reference: precompute_masks (proj/src/dropedge.cpp:9-33). Mask k shuffles
// iota(m) with Rng(substream(seed,"dropedge.mask",k)).shuffle (rng.hpp:69-74:
// for i = m..2, swap(a[i-1], a[next_below(i)])) and keeps a[0..keep).
//
// Parallel restatement. Position i-1 is final after step i, so the dropped set
// is exactly the set of values placed by the first D = m - keep steps
// (i = m..keep+1). Step t (i = m - t) places at i-1 the value held at
// j_t = next_below(i) just before step t. That value is found by walking back
// in time: the latest earlier step t' < t with j_{t'} == j_t had moved there
// the value then at position m-t'-1; recurse on (m-t'-1, t'); with no such
// step the value is the position itself (iota). All j_t are counter-based
// draws (draw t + #rejections-before-t), so every step resolves in parallel
// after one stable radix sort of (j_t, t). next_below rejections
// (r < 2^64 mod i, probability < i/2^64 per draw) are detected and the draw
// indices of all later steps shifted, exactly as the sequential stream would.
#include <cub/cub.cuh>

#include <cmath>

#include "internal.hpp"

namespace sc {
namespace {

constexpr int kBlock = 256;

__global__ void draw_steps_kernel(int64_t m, int64_t D, uint64_t s, int64_t start, int64_t shift, int32_t* j,
                                  int32_t* t_idx, unsigned long long* first_reject) {
    for (int64_t t = start + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < D;
         t += int64_t(gridDim.x) * blockDim.x) {
        const uint64_t i = static_cast<uint64_t>(m - t);
        const uint64_t r = draw_u64(s, static_cast<uint64_t>(t + shift));
        if (r < below_threshold(i)) atomicMin(first_reject, static_cast<unsigned long long>(t));
        j[t] = static_cast<int32_t>(r % i);
        t_idx[t] = static_cast<int32_t>(t);
    }
}

__global__ void ones_kernel(uint8_t* p, int64_t n) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        p[i] = 1;
}

// sorted (js, ts): stable by j, so for a fixed j the ts are ascending.
__device__ __forceinline__ int64_t lower_bound_i32(const int32_t* a, int64_t n, int32_t x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (a[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void resolve_kernel(int64_t m, int64_t D, const int32_t* __restrict__ j, const int32_t* __restrict__ js,
                               const int32_t* __restrict__ ts, uint8_t* mask) {
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < D; t += int64_t(gridDim.x) * blockDim.x) {
        int64_t pos = j[t];
        int64_t time = t;
        for (;;) {
            // latest step t' < time with j_{t'} == pos
            const int64_t lo = lower_bound_i32(js, D, static_cast<int32_t>(pos));
            int64_t best = -1;
            for (int64_t q = lo; q < D && js[q] == pos; ++q) {
                if (ts[q] < time) best = ts[q];
                else break;
            }
            if (best < 0) break;
            pos = m - best - 1;
            time = best;
        }
        mask[pos] = 0;
    }
}

}  // namespace

void precompute_masks_device(sc_ctx* ctx, int64_t m, int32_t k, double ratio, uint64_t seed, uint8_t* out) {
    if (k < 1) throw std::invalid_argument("precompute_masks: need at least one mask");
    if (ratio < 0.0 || ratio >= 1.0) throw std::invalid_argument("precompute_masks: ratio must lie in [0, 1)");
    cudaStream_t st = ctx->stream;
    const auto keep = static_cast<int64_t>(std::ceil((1.0 - ratio) * static_cast<double>(m)));
    const int64_t D = m - keep;
    if (m > 0) {
        ones_kernel<<<grid_for(m * k, kBlock), kBlock, 0, st>>>(out, m * k);
        SC_LAUNCH_CHECK();
        count_launch();
    }
    if (D <= 0) return;
    DevBuf<int32_t> j(D), t_idx(D), js(D), ts(D);
    DevBuf<unsigned long long> first(1);
    int eb = 1;
    while (eb < 32 && (static_cast<uint64_t>(m) >> eb) != 0) ++eb;
    for (int32_t mk = 0; mk < k; ++mk) {
        const uint64_t s = substream(seed, "dropedge.mask", static_cast<uint64_t>(mk));
        int64_t start = 0, shift = 0;
        for (;;) {
            const unsigned long long none = static_cast<unsigned long long>(D);
            h2d(first.get(), &none, 1, st);
            draw_steps_kernel<<<grid_for(D - start, kBlock), kBlock, 0, st>>>(m, D, s, start, shift, j.get(),
                                                                              t_idx.get(), first.get());
            SC_LAUNCH_CHECK();
            count_launch();
            unsigned long long f = 0;
            d2h(&f, first.get(), 1, st);
            SC_CUDA(cudaStreamSynchronize(st));
            if (f >= static_cast<unsigned long long>(D)) break;
            start = static_cast<int64_t>(f);
            shift += 1;
        }
        size_t tb = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tb, j.get(), js.get(), t_idx.get(), ts.get(), D, 0, eb, st);
        cub::DeviceRadixSort::SortPairs(ctx->temp(tb), tb, j.get(), js.get(), t_idx.get(), ts.get(), D, 0, eb, st);
        count_launch(4);
        resolve_kernel<<<grid_for(D, kBlock), kBlock, 0, st>>>(m, D, j.get(), js.get(), ts.get(),
                                                               out + static_cast<int64_t>(mk) * m);
        SC_LAUNCH_CHECK();
        count_launch();
    }
    SC_CUDA(cudaStreamSynchronize(st));
}

}  // namespace sc
