// mma_rate.cu — tcgen05 kind::f16 issue-rate probe (CTA pairs, cta_group::2) on B200.
//
// Times back-to-back MMAs (M = 256 across the pair, K = 16) with the A operand in shared
// memory (SS) or in TMEM (TS), for N = 256 and N = 128, on every SM pair at once, to decide
// the shapes of the fp16x3 GEMM pipelines (gemm_tc.cu): does an N = 128 MMA with A in TMEM
// run at the same MAC rate as N = 256?
//
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o mma_rate mma_rate.cu -lcuda
//   ./mma_rate            -> one line per variant: clocks per MMA, MACs/clk/SM, TFLOP/s at the measured clock
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) {                                                                \
            std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            return 1;                                                                           \
        }                                                                                       \
    } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void csync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint64_t desc_sw64(uint32_t saddr) {
    return static_cast<uint64_t>((saddr & 0x3FFFF) >> 4) | (uint64_t(1) << 16) | (uint64_t(512 >> 4) << 32) |
           (uint64_t(1) << 46) | (uint64_t(4) << 61);
}
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
    return (1u << 4) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

template <bool TS, int N>
__global__ void __launch_bounds__(128, 1) probe(int iters, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
    uint8_t* a_s = smem;            // 128 rows x 64 B (SW64, K = 32)
    uint8_t* b_s = smem + 8192;     // N / 2 rows x 64 B
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t rank = ctarank();
    // random-ish fp16 operands (|x| < 1): data-dependent power matters under the power cap
    for (int i = tid; i < (8192 + N * 32) / 4; i += blockDim.x) {
        uint32_t h = (i * 2654435761u) ^ (blockIdx.x * 40503u);
        const uint32_t e = 0x3000u | (h & 0x0BFFu);  // exponent 12..14, random mantissa
        reinterpret_cast<uint32_t*>(smem)[i] = e | ((e ^ (h >> 7)) & 0x83FFu) << 16;
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    csync();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tslot;
    if (TS) {  // A' (128 lanes x 16 columns) at column 256
        uint32_t v[8];
        for (int q = 0; q < 8; ++q) v[q] = 0x3C003800u ^ ((tid * 977u + q * 131u) & 0x03FF03FFu);
        for (int c = 0; c < 16; c += 8)
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                             tmem + ((32u * warp) << 16) + 256 + c),
                         "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                         : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    csync();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (rank == 0 && tid == 0) {
        const uint32_t idesc = idesc_f16(256, N);
        const uint64_t da = desc_sw64(su32(a_s)), db = desc_sw64(su32(b_s));
        const long long t0 = clock64();
        unsigned long long g0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const uint32_t d = tmem + ((it & 1) ? (N == 256 ? 0 : 128) : 0);
                if (TS)
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
                        "r"(tmem + 256 + k * 8), "l"(db + (k * 32 >> 4)), "r"(idesc), "r"(1));
                else
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
                        "l"(da + (k * 32 >> 4)), "l"(db + (k * 32 >> 4)), "r"(idesc), "r"(1));
            }
        }
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                su32(&bar)),
            "h"(uint16_t(3))
            : "memory");
        asm volatile(
            "{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(
                su32(&bar))
            : "memory");
        const long long t1 = clock64();
        unsigned long long g1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
        out[2 * (blockIdx.x >> 1)] = static_cast<unsigned long long>(t1 - t0);
        out[2 * (blockIdx.x >> 1) + 1] = g1 - g0;
    } else if (rank == 1 && tid == 0) {
        asm volatile(
            "{\n\t.reg .pred p;\nW1:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W1;\n}" ::"r"(
                su32(&bar))
            : "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    csync();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <bool TS, int N>
int run(const char* name, int sms) {
    const int pairs = sms / 2, iters = 20000;
    unsigned long long* d;
    CK(cudaMalloc(&d, sizeof(unsigned long long) * 2 * pairs));
    auto k = probe<TS, N>;
    const int smem = 8192 + 128 * 64 + 2048;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(2 * pairs);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    for (int rep = 0; rep < 3; ++rep) {
        CK(cudaLaunchKernelEx(&cfg, k, iters, d));
        CK(cudaDeviceSynchronize());
    }
    std::vector<unsigned long long> h(2 * pairs);
    CK(cudaMemcpy(h.data(), d, h.size() * 8, cudaMemcpyDeviceToHost));
    double clk = 0, ns = 0;
    for (int p = 0; p < pairs; ++p) {
        clk += double(h[2 * p]);
        ns += double(h[2 * p + 1]);
    }
    clk /= pairs;
    ns /= pairs;
    const double mmas = 2.0 * iters;
    const double macs_per_sm = mmas * 256.0 * N * 16 / 2.0;  // per SM of the pair
    const double ghz = clk / ns;
    std::printf("%-8s N=%3d  clk/MMA %7.1f  MACs/clk/SM %7.1f  SM clock %.3f GHz  dense %.1f TFLOP/s (all SMs)\n",
                name, N, clk / mmas, macs_per_sm / clk, ghz, 2.0 * macs_per_sm * sms / ns / 1e3);
    CK(cudaFree(d));
    return 0;
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    sms &= ~1;
    run<false, 256>("SS", sms);
    run<false, 128>("SS", sms);
    run<true, 256>("TS", sms);
    run<true, 128>("TS", sms);
    run<false, 64>("SS", sms);
    run<true, 64>("TS", sms);
    return 0;
}
