// common.cuh — shared device/host helpers for libsagecut_cuda.so (sm_100a).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace sc {

// ---- errors: the reference's exception taxonomy, carried across the C ABI ----
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct NcclError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define SC_CUDA(expr)                                                                                   \
    do {                                                                                                \
        cudaError_t sc_e_ = (expr);                                                                     \
        if (sc_e_ != cudaSuccess)                                                                       \
            throw ::sc::CudaError(std::string(#expr) + ": " + cudaGetErrorString(sc_e_) + " (" __FILE__ \
                                  ":" + std::to_string(__LINE__) + ")");                                \
    } while (0)

#define SC_LAUNCH_CHECK() SC_CUDA(cudaGetLastError())

// Host-side launch counter (bench.py reports "gpu_launches").
extern thread_local int64_t g_launches;
inline void count_launch(int64_t n = 1) { g_launches += n; }

// ---- RNG: the reference's splitmix64 stream (proj/include/sagecut/rng.hpp) ----
constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ULL;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {  // rng.hpp:11-16
    x += kGamma;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
// t-th (0-based) next_u64() of Rng(seed): state = seed + (t+1)γ, output =
// finalizer(state) = mix64(seed + tγ). Counter-based, so every draw of the
// reference's sequential stream is computable in parallel.
__host__ __device__ __forceinline__ uint64_t draw_u64(uint64_t seed, uint64_t t) { return mix64(seed + t * kGamma); }
// next_below's rejection threshold (rng.hpp:43-49): draws r < (2^64 mod n) are redrawn.
__host__ __device__ __forceinline__ uint64_t below_threshold(uint64_t n) { return (0 - n) % n; }
__host__ __device__ __forceinline__ double u64_to_double(uint64_t r) {  // next_double, rng.hpp:31-33
    return static_cast<double>(r >> 11) * 0x1.0p-53;
}

inline uint64_t fnv1a64(const char* s) {  // rng.hpp:83-90
    uint64_t h = 0xcbf29ce484222325ULL;
    for (; *s; ++s) {
        h ^= static_cast<unsigned char>(*s);
        h *= 0x100000001b3ULL;
    }
    return h;
}
inline uint64_t substream(uint64_t seed, const char* tag) { return mix64(seed ^ fnv1a64(tag)); }
inline uint64_t substream(uint64_t seed, const char* tag, uint64_t a) {
    return mix64(substream(seed, tag) ^ mix64(a + kGamma));
}
inline uint64_t substream(uint64_t seed, const char* tag, uint64_t a, uint64_t b) {
    return mix64(substream(seed, tag, a) ^ mix64(b + 0x2545f4914f6cdd1dULL));
}
// Sequential host Rng, used only for scalar control draws (mask selection).
struct HostRng {
    uint64_t s;
    explicit HostRng(uint64_t seed) : s(seed) {}
    uint64_t next_u64() {
        s += kGamma;
        return mix64(s - kGamma);
    }
    uint64_t next_below(uint64_t n) {
        const uint64_t thr = below_threshold(n);
        for (;;) {
            const uint64_t r = next_u64();
            if (r >= thr) return r % n;
        }
    }
};

inline int num_sms() {
    static int n = [] {
        int dev = 0, v = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    }();
    return n;
}

inline unsigned grid_for(int64_t n, int block, int64_t max_blocks = 0) {
    int64_t g = (n + block - 1) / block;
    if (max_blocks <= 0) max_blocks = int64_t(num_sms()) * 32;
    if (g > max_blocks) g = max_blocks;
    if (g < 1) g = 1;
    return static_cast<unsigned>(g);
}

}  // namespace sc
