// gemm_tc.cu — fp32-grade GEMMs on the 5th-gen tensor cores (tcgen05, sm_100a).
//
//   NT:  C[M x N] = A1 op(B1) (+ A2 op(B2)), M huge (partition rows), N <= 256
//        (forward msg / update / head, backward dgrad)
//   TN:  C[N1 x N2] = A^T [B1 | B2], K = M rows (weight gradients)
//
// Precision ("fp16x3"). The reference's f32 mode needs ~fp32 products: its
// parity bar is 1e-4 relative after 5 Adam steps, and Adam amplifies small
// gradient errors. Each fp32 operand is scaled by a power of two (exact) so its
// |max| lands in [2^14, 2^15), then split into fp16 hi = rn(x s) and
// lo = rn(x s - hi) (|x s - hi - lo| <= 2^-22 |x s|); the product is
// hi*hi + hi*lo + lo*hi (three kind::f16 MMAs at the full 16-bit tensor rate,
// fp32 accumulation in TMEM). Measured ~1e-6 relative vs fp64 (bf16 splitting:
// 4.5e-6, which compounded to 2.5e-4 in 5-step gradients). The |max| values
// come from the kernels that produced each operand (no host sync).
//
// Data movement (persistent, one CTA (pair) per SM (pair)):
//   loader warp      2D TMA boxes HBM -> fp32 staging ring in shared memory
//   converter warps  staging fp32 -> scaled fp16 hi/lo tiles in the canonical
//                    SWIZZLE_64B K-major (NT) or SWIZZLE_128B MN-major (TN)
//                    layout; TN CTA pairs write the A' halves to TMEM instead;
//                    NT thread 0 also bulk-copies the pre-split weight image
//   MMA warp         TMEM allocator + single-thread MMA issuer (tcgen05.mma/commit)
//   epilogue warps   tcgen05.ld -> unscale / ReLU / row-scale / |max| -> smem
//                    transpose -> TMA stores (NT), or periodic TMEM drains into
//                    an fp32 split-K partial (TN)
// NT: 8 converter + 8 epilogue warps, two TMEM accumulators (2 x 256 columns) so
// one tile's epilogue overlaps the next tile's main loop. TN: TnCfg (8 or 16
// converter warps, 4 epilogue warps).
#include <cuda.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "gemm_tc.cuh"
#include "internal.hpp"
#include "trainer.hpp"

namespace sc {
namespace tc {

constexpr int kBM = 128;  // UMMA M (cta_group::1)
constexpr int kMaxN = 256;
constexpr int kConvWarps = 8;  // TN converter warps (NT: NtCfg::kCW)
// NT uses 8 epilogue warps (after the converters: two per TMEM lane quarter, even / odd
// 32-column chunks), then the MMA and loader warps.
constexpr int kNtEpiWarps = 8;

// NT: 32-deep k-stages, fp16 SW64 tiles (64 B rows)
constexpr int kNtBK = 32;
constexpr int kNtATile = kBM * 64;                    // one (hi or lo) A tile
constexpr int kNtStgBytes = kBM * kNtBK * 4;          // 128 rows x 32 fp32
constexpr int kNtEpiBuf = 32 * 32 * 4;                // one 32 x 32 fp32 output box (SW128)
constexpr int kNtEpiBytes = kNtEpiWarps * kNtEpiBuf;  // one store box per epilogue warp

// TN: 32-row stages, fp16 MN-major SW128 tiles
constexpr int kTnBK = 32;
constexpr int kTnATile = kBM * kTnBK * 2;             // 128 cols x 32 rows fp16 = 8 KB
constexpr int kTnStgA = kTnBK * kBM * 4;              // 32 rows x 128 fp32 = 16 KB
constexpr int kChunkKb = 32;                          // 1024 rows per TMEM accumulation (TN)
constexpr int kTnBox = kTnBK * 128;                   // one 32-column x 32-row fp32 TMA box

struct Src {
    CUtensorMap tmap;     // 2D map over A (box 32 k x 128 rows, fp32, SWIZZLE_128B, OOB -> 0)
    const float* a;
    int64_t lda;
    int32_t K;            // valid k (multiple of 4)
    int32_t kblocks;      // ceil(K / 32)
    const uint8_t* bimg;  // kblocks x [hi tile | lo tile], each n_pad x 64 B (32 k, SW64)
    CUtensorMap tmap_b;   // the same image as 2D [kblocks * 2 * n_pad rows x 64 B] (pair kernel: half-tile boxes)
    const float* amax_a;  // max|A| (device scalar)
    const int32_t* bexp;  // power-of-two exponent B was scaled by (device scalar)
};

struct alignas(64) Params {
    Src src[2];
    CUtensorMap tmap_c;   // 2D map over C (box 32 cols x 32 rows, fp32, SWIZZLE_128B; stores clip at M, N)
    int nsrc;
    int64_t M;
    int32_t N, n_pad;
    float* C;
    int64_t ldc;
    int epi;
    const float* row_scale;
    float* amax_out;
    uint32_t* relu_pos;  // optional (EPI == kEpiRelu): bit c % 32 of word [row][c / 32] = C[row][c] > 0
    const float* mask_msg;     // EPI == kEpiMask: C = 1[msg > 0] acc, msg row stride N ...
    const uint32_t* mask_pos;  // ... or its sign bits ([row][ceil(N / 32)] words)
    int64_t tiles;
    unsigned long long* trace;  // optional (SC_TN_TRACE_BUILD + SC_TN_TRACE=1), as TnParams::trace
    int32_t prefetch;           // L2-prefetch the CTA's next tile's A rows at the start of each tile
};

// ---- PTX helpers -------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// Instruction descriptor, kind::f16: D f32 (bits 4-5 = 1), A f16 (7-9 = 0),
// B f16 (10-12 = 0), both K-major, N>>3 at [17,23), M>>4 at [24,29).
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
    return (1u << 4) | (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
}
__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
        "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// (slot, phase) of a circular mbarrier pipeline, advanced without divisions.
struct Ring {
    int idx = 0;
    uint32_t phase = 0;
    __device__ __forceinline__ void next(int n) {
        if (++idx == n) {
            idx = 0;
            phase ^= 1u;
        }
    }
};

// Exponent k such that amax * 2^k lies in [2^14, 2^15) (0 for zero / non-finite).
__host__ __device__ __forceinline__ int scale_exp(float amax) {
    if (!(amax > 0.f) || !(amax < 3.0e38f)) return 0;
    int e;
    frexpf(amax, &e);  // amax = f 2^e, f in [0.5, 1)
    return 15 - e;
}

// x * 2^k split into fp16 (hi, lo); two elements per 32-bit word. Packed fp32x2 arithmetic
// (FMUL2 / FFMA2) and packed conversions (F2FP); x s - hi is exact in fp32.
__device__ __forceinline__ void split2(float x0, float x1, float s, uint32_t& hi, uint32_t& lo) {
    const float2 xs = __fmul2_rn(make_float2(x0, x1), make_float2(s, s));
    const __half2 h = __float22half2_rn(xs);
    const float2 d = __ffma2_rn(__half22float2(h), make_float2(-1.f, -1.f), xs);
    const __half2 l = __float22half2_rn(d);
    hi = *reinterpret_cast<const uint32_t*>(&h);
    lo = *reinterpret_cast<const uint32_t*>(&l);
}

// kEpiMask: bit q = 1[msg[row][c0 + q] > 0] for the 32 columns from c0 (all-ones past M / N).
__device__ __forceinline__ uint32_t mask_bits32(const Params& p, int64_t row, int32_t c0) {
    if (row >= p.M || c0 >= p.N) return ~0u;
    if (p.mask_pos) return p.mask_pos[row * ((p.N + 31) >> 5) + (c0 >> 5)];
    const float* m = p.mask_msg + row * p.N + c0;
    uint32_t b = 0;
    if (c0 + 32 <= p.N && (p.N & 3) == 0) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(m) + j);
            b |= (v.x > 0.f ? 1u : 0u) << (4 * j) | (v.y > 0.f ? 1u : 0u) << (4 * j + 1) |
                 (v.z > 0.f ? 1u : 0u) << (4 * j + 2) | (v.w > 0.f ? 1u : 0u) << (4 * j + 3);
        }
    } else {
        for (int q = 0; q < 32 && c0 + q < p.N; ++q) b |= (m[q] > 0.f ? 1u : 0u) << q;
    }
    return b;
}

// K-major SWIZZLE_64B descriptor: 8-row core groups of 512 B (SBO), swizzle mode 4.
__device__ __forceinline__ uint64_t desc_sw64(uint32_t saddr) {
    return static_cast<uint64_t>((saddr & 0x3FFFF) >> 4) | (static_cast<uint64_t>(1) << 16) |
           (static_cast<uint64_t>(512 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) |
           (static_cast<uint64_t>(4) << 61);
}
// Byte offset of (row, 16-byte chunk c in 0..3) in a K-major SW64 tile
// (Swizzle<2,4,3>: chunk bits [4,6) ^= address bits [7,9)).
__host__ __device__ __forceinline__ uint32_t sw64_off(uint32_t row, uint32_t c) {
    return (row >> 3) * 512 + (row & 7) * 64 + ((c ^ ((row >> 1) & 3)) << 4);
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int32_t x, int32_t y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int32_t x, int32_t y) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(x), "r"(y), "r"(smem_u32(src))
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// L2 prefetch of a 2D TMA box (no shared memory, no barrier): raises the HBM bytes in flight beyond
// what the shared-memory staging ring can hold, so the later tensor load hits L2.
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int32_t x, int32_t y) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(x), "r"(y)
                 : "memory");
}
// 3D TMA store / reduce-add of one smem box (the weight-gradient partials [split][N1][N2]; the N1 and
// N2 extents clip a box's rows / columns beyond the matrix). One bulk group each.
// (pol: an L2 eviction policy — the split partials stay L2-resident until tn_reduce_kernel sums them)
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int32_t x, int32_t y, int32_t z,
                                             uint64_t pol) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2, %3}], [%4], %5;" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(x), "r"(y), "r"(z), "r"(smem_u32(src)), "l"(pol)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void tma_reduce_add_3d(const CUtensorMap* map, const void* src, int32_t x, int32_t y,
                                                  int32_t z, uint64_t pol) {
    asm volatile(
        "cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group.L2::cache_hint [%0, {%1, %2, %3}], [%4], "
        "%5;" ::"l"(reinterpret_cast<uint64_t>(map)),
        "r"(x), "r"(y), "r"(z), "r"(smem_u32(src)), "l"(pol)
        : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// all of this thread's bulk groups complete (writes performed), not just their source reads
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
// L2 eviction-priority policies (createpolicy) for streamed operands and L2-resident partials.
__device__ __forceinline__ uint64_t l2_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void st_l2hint(float* ptr, float v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(ptr), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_v4_l2hint(float* ptr, float a, float b, float c, float d, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(ptr), "f"(a), "f"(b), "f"(c),
                 "f"(d), "l"(pol)
                 : "memory");
}
// fire-and-forget fp32 adds performed at L2 (round-to-nearest)
__device__ __forceinline__ void red_add_v4_l2hint(float* ptr, float a, float b, float c, float d, uint64_t pol) {
    asm volatile("red.global.add.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(ptr), "f"(a), "f"(b),
                 "f"(c), "f"(d), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void red_add_l2hint(float* ptr, float a, uint64_t pol) {
    asm volatile("red.global.add.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(ptr), "f"(a), "l"(pol) : "memory");
}
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const CUtensorMap* map, int32_t x, int32_t y,
                                                 uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
        "%3}], [%4], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void split8_store(const float4& x0, const float4& x1, float s, uint8_t* hi_base,
                                             uint8_t* lo_base, uint32_t off) {
    uint4 hi, lo;
    split2(x0.x, x0.y, s, hi.x, lo.x);
    split2(x0.z, x0.w, s, hi.y, lo.y);
    split2(x1.x, x1.y, s, hi.z, lo.z);
    split2(x1.z, x1.w, s, hi.w, lo.w);
    *reinterpret_cast<uint4*>(hi_base + off) = hi;
    *reinterpret_cast<uint4*>(lo_base + off) = lo;
}
// Zero the elements of an 8-wide chunk at or beyond `valid` (0..8).
__device__ __forceinline__ void mask8(float4& x0, float4& x1, int valid) {
    if (valid >= 8) return;
    float v[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
#pragma unroll
    for (int q = 0; q < 8; ++q)
        if (q >= valid) v[q] = 0.f;
    x0 = make_float4(v[0], v[1], v[2], v[3]);
    x1 = make_float4(v[4], v[5], v[6], v[7]);
}


// ---- CTA-pair (cta_group::2) helpers ----------------------------------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// shared::cluster address of the same shared variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
// Arrive on a barrier of either CTA of the cluster. Default (.release.cta) semantics, as the
// tensor-core pipelines use: the data it publishes was written to the arriving CTA's own shared
// memory and made visible to the async proxy by fence.proxy.async beforehand.
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAITC_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAITC_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// 2D TMA issued by either CTA of a pair; completion bytes are counted on the leader's barrier.
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, int32_t x, int32_t y,
                                                 uint32_t leader_bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
        "%3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(leader_bar)
        : "memory");
}
template <bool PAIR>
__device__ __forceinline__ void mma_f16_g(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    if constexpr (PAIR)
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
            "l"(a), "l"(b), "r"(idesc), "r"(acc));
    else
        mma_f16(d_tmem, a, b, idesc, acc);
}
// A operand from TMEM (K-major: lane = M row, K packed two fp16 per 32-bit column), B from smem.
__device__ __forceinline__ void mma_f16_ts_pair(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                                uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}
template <int N>
__device__ __forceinline__ void tmem_st(uint32_t taddr, const uint32_t (&v)[N]) {
    static_assert(N == 4 || N == 8, "tmem_st: 4 or 8 columns");
    if constexpr (N == 8) {
        tmem_st8(taddr, v);
    } else {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(v[0]), "r"(v[1]),
                     "r"(v[2]), "r"(v[3])
                     : "memory");
    }
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// MMA completion -> barrier at the same offset in both CTAs of the pair (or the local one).
template <bool PAIR>
__device__ __forceinline__ void mma_commit_g(uint64_t* bar) {
    if constexpr (PAIR)
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(bar)),
            "h"(static_cast<uint16_t>(3))
            : "memory");
    else
        mma_commit(bar);
}
template <bool PAIR>
__device__ __forceinline__ void tmem_alloc_g(uint32_t* slot) {
    if constexpr (PAIR) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
}
template <bool PAIR>
__device__ __forceinline__ void tmem_dealloc_g(uint32_t base) {
    if constexpr (PAIR)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(512));
    else
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(512));
}

// Shared-memory plan of the NT kernel. PAIR: a CTA pair (cluster of 2, cta_group::2)
// computes a 256-row tile with one M=256 MMA stream; each CTA converts its own
// 128 A rows and holds half of the weight image's rows, so the per-SM operand
// bytes (TMA in, tensor-core reads) drop by a third and the freed shared memory
// deepens both rings.
template <bool PAIR>
struct NtCfg {
    // warp roles: converters 0 .. kCW-1, epilogue kCW .. kCW+7, MMA issuer, TMA loader
    // (16 converter warps measured ~1 % slower than 8: the converters are not the limit)
    static constexpr int kCW = 8;
    static constexpr int kC = kCW * 32;
    static constexpr int kMma = kCW + kNtEpiWarps, kLoad = kMma + 1, kThr = (kLoad + 1) * 32;
    static constexpr int kStages = PAIR ? 4 : 3;                    // MMA operand stages
    static constexpr int kStg = PAIR ? 4 : 3;                       // fp32 staging stages
    static constexpr int kBTile = (PAIR ? kMaxN / 2 : kMaxN) * 64;  // one (hi or lo) B tile, this CTA's rows
    static constexpr int kStage = 2 * kNtATile + 2 * kBTile;
    static constexpr int kStgOff = kStages * kStage;
    static constexpr int kEpiOff = kStgOff + kStg * kNtStgBytes;
    static constexpr int kBarOff = kEpiOff + kNtEpiBytes;
    static constexpr int kSmem = kBarOff + 256 + 1024;
    static constexpr int kRows = PAIR ? 2 * kBM : kBM;              // output rows per tile
};
static_assert(NtCfg<true>::kSmem <= 232448 && NtCfg<false>::kSmem <= 232448, "NT shared memory");

// Diagnostics (build with -DSC_TN_TRACE_BUILD, run with SC_TN_TRACE=1): cycles each
// role spends in its barrier waits, summed over CTAs and printed per launch (TN and NT).
#ifdef SC_TN_TRACE_BUILD
#define TN_TIMED_WAIT(acc_var, call)                                              \
    do {                                                                          \
        const long long t0_ = p.trace ? clock64() : 0;                            \
        call;                                                                     \
        if (p.trace) acc_var += static_cast<unsigned long long>(clock64() - t0_); \
    } while (0)
#else
#define TN_TIMED_WAIT(acc_var, call) call
#endif

template <int EPI, bool AMAX, bool PAIR>
__global__ void __launch_bounds__(NtCfg<PAIR>::kThr, 1) gemm_f16x3_kernel(const __grid_constant__ Params p) {
    using Cfg = NtCfg<PAIR>;
    extern __shared__ __align__(16) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* stg_base = smem + Cfg::kStgOff;
    uint8_t* epi_base = smem + Cfg::kEpiOff;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::kBarOff);
    uint64_t* full = bars;                              // [kStages] converters + B TMA -> MMA (leader's)
    uint64_t* empty = full + Cfg::kStages;              // [kStages] MMA -> converters
    uint64_t* sfull = empty + Cfg::kStages;             // [kStg] loader (tx) -> converters
    uint64_t* sempty = sfull + Cfg::kStg;               // [kStg] converters -> loader
    uint64_t* tfull = sempty + Cfg::kStg;               // [2] MMA -> epilogue
    uint64_t* tempty = tfull + 2;                       // [2] epilogue -> MMA (leader's)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = PAIR ? cluster_ctarank() : 0u;
#ifdef SC_TN_TRACE_BUILD
    unsigned long long w_a = 0, w_b = 0;
    const long long t_start = p.trace ? clock64() : 0;
#endif
    const int64_t tile0 = PAIR ? (blockIdx.x >> 1) : blockIdx.x;
    const int64_t tstep = PAIR ? (gridDim.x >> 1) : gridDim.x;
    const int32_t nloc = PAIR ? (p.n_pad >> 1) : p.n_pad;  // weight rows held by this CTA
    const uint32_t bh = static_cast<uint32_t>(nloc) * 64u;  // bytes of one local (hi or lo) B tile

    // Per-source operand scales: A_s gets 2^(kt - kB_s) so that every source's
    // products carry the same total scale 2^kt (they share one accumulator).
    int kt = 1 << 20;
    int kb_exp[2] = {0, 0};
    for (int s = 0; s < p.nsrc; ++s) {
        kb_exp[s] = *p.src[s].bexp;
        kt = min(kt, scale_exp(*p.src[s].amax_a) + kb_exp[s]);
    }

    if (warp == Cfg::kMma) {
        if (lane == 0) {
            for (int s = 0; s < Cfg::kStages; ++s) {
                mbar_init(&full[s], Cfg::kCW * (PAIR ? 2 : 1));
                mbar_init(&empty[s], 1);
            }
            for (int s = 0; s < Cfg::kStg; ++s) {
                mbar_init(&sfull[s], 1);
                mbar_init(&sempty[s], Cfg::kCW);
            }
            for (int s = 0; s < 2; ++s) {
                mbar_init(&tfull[s], 1);
                mbar_init(&tempty[s], kNtEpiWarps * (PAIR ? 2 : 1));
            }
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
        tmem_alloc_g<PAIR>(tmem_slot);
    }
    tc_fence_before();
    if constexpr (PAIR) cluster_sync();  // peer barriers initialised before any remote arrive
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // the pair's leader (rank 0) owns the barriers the MMA issuer waits on
    const uint32_t full_l = PAIR ? mapa(smem_u32(full), 0) : smem_u32(full);
    const uint32_t tempty_l = PAIR ? mapa(smem_u32(tempty), 0) : smem_u32(tempty);

    int kb_total = 0;
    for (int s = 0; s < p.nsrc; ++s) kb_total += p.src[s].kblocks;

    if (warp == Cfg::kLoad) {
        // ================= loader: one 2D TMA per stage, HBM -> fp32 staging =================
        // box 32 k (128 B) x 128 rows, SWIZZLE_128B; out-of-range rows / k are zero-filled
        Ring ring;
        for (int64_t tile = tile0; tile < p.tiles; tile += tstep) {
            if (p.prefetch && tile + tstep < p.tiles) {  // the next tile's rows: one box per (source, k-block)
                const int32_t y = static_cast<int32_t>((tile + tstep) * Cfg::kRows + rank * kBM);
                int j = 0;
                for (int src = 0; src < p.nsrc; ++src)
                    for (int kb = 0; kb < p.src[src].kblocks; ++kb, ++j)
                        if ((j & 31) == lane) tma_prefetch_2d(&p.src[src].tmap, kb * kNtBK, y);
            }
            for (int src = 0; src < p.nsrc; ++src)
                for (int kb = 0; kb < p.src[src].kblocks; ++kb, ring.next(Cfg::kStg)) {
                    TN_TIMED_WAIT(w_a, mbar_wait(&sempty[ring.idx], ring.phase ^ 1));
                    if (lane == 0) {
                        mbar_arrive_expect_tx(&sfull[ring.idx], kNtStgBytes);
                        tma_load_2d(stg_base + ring.idx * kNtStgBytes, &p.src[src].tmap, kb * kNtBK,
                                    static_cast<int32_t>(tile * Cfg::kRows + rank * kBM), &sfull[ring.idx]);
                    }
                    __syncwarp();
                }
        }
    } else if (warp < Cfg::kCW) {
        // ================= converters: staging fp32 -> scaled fp16 hi/lo (SW64) =================
        // Row-fastest mapping: 8 consecutive threads read the same chunk of 8 different rows, which
        // the 128 B swizzle spreads over distinct banks (conflict-free loads and SW64 stores).
        // Thread 0 also fetches this CTA's rows of the stage's weight image.
        const int tid = threadIdx.x;
        const float sa0 = ldexpf(1.f, kt - kb_exp[0]), sa1 = ldexpf(1.f, kt - kb_exp[1]);
        Ring mr, sr;  // MMA-operand ring, staging ring
        for (int64_t tile = tile0; tile < p.tiles; tile += tstep)
            for (int src = 0; src < p.nsrc; ++src) {
                const Src& S = p.src[src];
                const float sa = src ? sa1 : sa0;
                for (int kb = 0; kb < S.kblocks; ++kb, mr.next(Cfg::kStages), sr.next(Cfg::kStg)) {
                    uint8_t* st = smem + mr.idx * Cfg::kStage;
                    const uint8_t* sg = stg_base + sr.idx * kNtStgBytes;
                    TN_TIMED_WAIT(w_a, mbar_wait(&empty[mr.idx], mr.phase ^ 1));
                    if (tid == 0) {
                        if constexpr (PAIR) {
                            // image rows: [kb][plane][n_pad]; this CTA's half starts at rank * nloc
                            const uint32_t fb = full_l + mr.idx * 8;
                            if (rank == 0) mbar_expect_tx(&full[mr.idx], 4 * bh);  // both halves, hi + lo
                            const int32_t r0 = (kb * 2) * p.n_pad + static_cast<int32_t>(rank) * nloc;
                            tma_load_2d_pair(st + 2 * kNtATile, &S.tmap_b, 0, r0, fb);
                            tma_load_2d_pair(st + 2 * kNtATile + bh, &S.tmap_b, 0, r0 + p.n_pad, fb);
                        } else {
                            mbar_expect_tx(&full[mr.idx], 2 * bh);
                            bulk_g2s(st + 2 * kNtATile, S.bimg + static_cast<int64_t>(kb) * 2 * bh, 2 * bh,
                                     &full[mr.idx]);
                        }
                    }
                    TN_TIMED_WAIT(w_b, mbar_wait(&sfull[sr.idx], sr.phase));
                    // all of the stage's shared loads first (4 x LDS.128 in flight), then convert
                    constexpr int kItems = 4 * kBM / Cfg::kC;  // (row, 8-float chunk) items per thread
                    float4 xv[kItems][2];
#pragma unroll
                    for (int j = 0; j < kItems; ++j) {
                        const int idx = tid + j * Cfg::kC;
                        const int r = idx & 127, c = idx >> 7;  // row, 8-float chunk (0..3)
                        const uint8_t* rowp = sg + r * (kNtBK * 4);
                        xv[j][0] = *reinterpret_cast<const float4*>(rowp + (((2 * c) ^ (r & 7)) << 4));
                        xv[j][1] = *reinterpret_cast<const float4*>(rowp + (((2 * c + 1) ^ (r & 7)) << 4));
                    }
#pragma unroll
                    for (int j = 0; j < kItems; ++j) {
                        const int idx = tid + j * Cfg::kC;
                        split8_store(xv[j][0], xv[j][1], sa, st, st + kNtATile, sw64_off(idx & 127, idx >> 7));
                    }
                    fence_proxy_async();
                    __syncwarp();
                    if (lane == 0) {
                        if constexpr (PAIR) mbar_arrive_cluster(full_l + mr.idx * 8);
                        else mbar_arrive(&full[mr.idx]);
                        mbar_arrive(&sempty[sr.idx]);
                    }
                }
            }
    } else if (warp == Cfg::kMma) {
        // ================= MMA issuer (the pair's leader only) =================
        if (PAIR && rank != 0) {
            // the peer's tensor core work is issued by the leader
        } else {
            const uint32_t idesc = idesc_f16(Cfg::kRows, p.n_pad);
            Ring mr;
            uint32_t t = 0;
            for (int64_t tile = tile0; tile < p.tiles; tile += tstep, ++t) {
                const uint32_t acc = t & 1;
                const uint32_t d_tmem = tmem_base + acc * 256;
                if constexpr (PAIR) TN_TIMED_WAIT(w_b, mbar_wait_cluster(&tempty[acc], ((t >> 1) & 1) ^ 1));
                else TN_TIMED_WAIT(w_b, mbar_wait(&tempty[acc], ((t >> 1) & 1) ^ 1));
                tc_fence_after();
                for (int kbg = 0; kbg < kb_total; ++kbg, mr.next(Cfg::kStages)) {
                    if constexpr (PAIR) TN_TIMED_WAIT(w_a, mbar_wait_cluster(&full[mr.idx], mr.phase));
                    else TN_TIMED_WAIT(w_a, mbar_wait(&full[mr.idx], mr.phase));
                    tc_fence_after();
                    if (lane == 0) {
                        const uint8_t* st = smem + mr.idx * Cfg::kStage;
                        const uint64_t ahi = desc_sw64(smem_u32(st)), alo = desc_sw64(smem_u32(st + kNtATile));
                        const uint64_t bhi = desc_sw64(smem_u32(st + 2 * kNtATile));
                        const uint64_t blo = desc_sw64(smem_u32(st + 2 * kNtATile + bh));
#pragma unroll
                        for (int k = 0; k < kNtBK / 16; ++k) {
                            const uint64_t adv = static_cast<uint64_t>(k * 32) >> 4;  // 16 fp16 = 32 B along K
                            mma_f16_g<PAIR>(d_tmem, ahi + adv, bhi + adv, idesc, (kbg | k) ? 1u : 0u);
                            mma_f16_g<PAIR>(d_tmem, ahi + adv, blo + adv, idesc, 1u);
                            mma_f16_g<PAIR>(d_tmem, alo + adv, bhi + adv, idesc, 1u);
                        }
                        mma_commit_g<PAIR>(&empty[mr.idx]);
                        if (kbg == kb_total - 1) mma_commit_g<PAIR>(&tfull[acc]);
                    }
                    __syncwarp();
                }
            }
        }
    } else {
        // ================= epilogue (warps 8-15) =================
        // tcgen05.ld (lane = row) -> unscale / ReLU / row-scale / |max| -> SW128 smem box -> TMA store
        // (the store clips rows >= M and columns >= N). n_pad is a multiple of 32 and the B image
        // is zero beyond N, as are TMA-filled A rows beyond M, so every chunk is full and padded
        // entries are exactly 0 (they cannot raise |max|).
        const int ew = warp & 3;                    // TMEM lanes 32*ew .. 32*ew+31
        const int half = (warp - Cfg::kCW) >> 2;  // even / odd 32-column chunks
        const float unscale = ldexpf(1.f, -kt);
        uint8_t* box = epi_base + (warp - Cfg::kCW) * kNtEpiBuf;
        float amx = 0.f;
        uint32_t t = 0;
        for (int64_t tile = tile0; tile < p.tiles; tile += tstep, ++t) {
            const uint32_t acc = t & 1;
            TN_TIMED_WAIT(w_a, mbar_wait(&tfull[acc], (t >> 1) & 1));
            tc_fence_after();
            const int64_t row0 = tile * Cfg::kRows + rank * kBM + ew * 32;  // this warp's 32 output rows
            float sc = 1.f;
            if (EPI == kEpiRowScale && row0 + lane < p.M) sc = p.row_scale[row0 + lane];
            for (int c0 = half * 32; c0 < p.n_pad; c0 += 64) {
                uint32_t r[32];
                tmem_ld32(tmem_base + acc * 256 + (static_cast<uint32_t>(ew * 32) << 16) + c0, r);
                if (lane == 0) TN_TIMED_WAIT(w_b, bulk_wait_read<0>());  // the previous store has read the box
                __syncwarp();
                uint32_t keep = ~0u;  // kEpiMask: the ReLU decisions of this row's 32 columns
                if (EPI == kEpiMask) keep = mask_bits32(p, row0 + lane, c0);
                uint32_t pos = 0;  // ReLU decisions of this row's 32 columns (compact activations)
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    float x[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        float v = __uint_as_float(r[4 * j + q]) * unscale;
                        if (EPI == kEpiRelu) {
                            v = fmaxf(v, 0.f);
                            pos |= (v > 0.f ? 1u : 0u) << (4 * j + q);
                        }
                        if (EPI == kEpiRowScale) v = sc * v;
                        if (EPI == kEpiMask) v = ((keep >> (4 * j + q)) & 1u) ? v : 0.f;
                        if (AMAX) amx = fmaxf(amx, fabsf(v));
                        x[q] = v;
                    }
                    *reinterpret_cast<float4*>(box + lane * 128 + ((j ^ (lane & 7)) << 4)) =
                        make_float4(x[0], x[1], x[2], x[3]);
                }
                if (EPI == kEpiRelu && p.relu_pos && c0 < p.N && row0 + lane < p.M)
                    p.relu_pos[(row0 + lane) * ((p.N + 31) >> 5) + (c0 >> 5)] = pos;
                fence_proxy_async();
                __syncwarp();
                if (lane == 0 && row0 < p.M) tma_store_2d(&p.tmap_c, box, c0, static_cast<int32_t>(row0));
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if constexpr (PAIR) mbar_arrive_cluster(tempty_l + acc * 8);
                else mbar_arrive(&tempty[acc]);
            }
        }
        if (lane == 0) bulk_wait_read<0>();
        if (AMAX) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) amx = fmaxf(amx, __shfl_xor_sync(0xffffffffu, amx, o));
            if (lane == 0) atomicMax(reinterpret_cast<unsigned int*>(p.amax_out), __float_as_uint(amx));
        }
    }
#ifdef SC_TN_TRACE_BUILD
    if (p.trace && lane == 0) {  // roles: 0 converters, 1 epilogue, 2 MMA, 3 loader
        const int role = warp < Cfg::kCW ? 0 : warp < Cfg::kMma ? 1 : warp == Cfg::kMma ? 2 : 3;
        if (role != 2 || !PAIR || rank == 0) {
            atomicAdd(p.trace + 4 * role + 0, w_a);
            atomicAdd(p.trace + 4 * role + 1, w_b);
            atomicAdd(p.trace + 4 * role + 2, static_cast<unsigned long long>(clock64() - t_start));
            atomicAdd(p.trace + 4 * role + 3, 1ull);
        }
    }
#endif
    tc_fence_before();
    if constexpr (PAIR) cluster_sync();  // no remote arrivals / tensor-core work left in flight
    else __syncthreads();
    if (warp == Cfg::kMma) {
        tc_fence_after();
        tmem_dealloc_g<PAIR>(tmem_base);
    }
}

// ---- NT, single source, K <= 256: A' in TMEM, weight image resident in shared memory -----------
// The general NT kernel above is shared-memory-bandwidth bound: per 32-k stage a CTA writes the
// fp32 staging (TMA) and reads it (converters), writes the fp16 hi / lo A tiles and the stage's
// weight-image rows (TMA), and the tensor core reads A and B three times — ~146 B/clk at full MMA
// rate against the SM's 128 B/clk. Here, for one source with K <= 256 (msg, dmean, head and head
// dgrad GEMMs):
//   * the whole weight image (this CTA's B' rows, every k-block, hi + lo: <= 128 KB) is loaded
//     into shared memory once per launch and stays there;
//   * the converters write A' (the tile's 128 rows x K, hi / lo) into TMEM with tcgen05.st
//     (lane = row, two fp16 per column), and the MMAs read A from TMEM;
// leaving the staging write + read and the B' operand reads: ~73 B/clk at full MMA rate.
// TMEM: A' for the whole K (kblocks x 32 columns, <= 256) + two accumulators of Np columns.
// N > 128 runs as two passes of Np = n_pad / 2 over the same A' (accumulator h), so the second
// pass's MMAs overlap the first pass's epilogue; N <= 128: one pass, accumulators alternate by tile.
// A' stage kb is released for the next tile after the tile's last pass has read it.
struct NtTmCfg {
    static constexpr int kCW = 8;                       // converter warps
    static constexpr int kMma = kCW + kNtEpiWarps, kLoad = kMma + 1, kThr = (kLoad + 1) * 32;
    static constexpr int kMaxStg = 12;                  // fp32 staging slots (as many as fit after B')
    static constexpr int kMaxKb = 8;                    // A' stages in TMEM (256 columns)
    static constexpr int kBOff = 0;                     // resident B' (<= kBBytes per CTA), then the staging ring
    static constexpr int kBBytes = kMaxKb * 2 * (kMaxN / 2) * 64;  // k-blocks x {hi, lo} x this CTA's rows x 64 B
    static constexpr int kSmem = kBBytes + 4 * kNtStgBytes + kNtEpiBytes + 512 + 1024;
    static constexpr int kBarOff = kSmem - 1024 - 512;  // barriers + TMEM slot (after the 1 KB alignment slack)
    static constexpr int kEpiOff = kBarOff - kNtEpiBytes;
    static constexpr int kRows = 2 * kBM;
};
static_assert(NtTmCfg::kSmem <= 232448, "NT (A in TMEM) shared memory");

template <int EPI, bool AMAX>
__global__ void __launch_bounds__(NtTmCfg::kThr, 1) gemm_nt_tm_kernel(const __grid_constant__ Params p) {
    using Cfg = NtTmCfg;
    extern __shared__ __align__(16) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* bres = smem + Cfg::kBOff;
    uint8_t* epi_base = smem + Cfg::kEpiOff;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::kBarOff);
    uint64_t* full = bars;                       // [kMaxKb] converters -> MMA (leader's)
    uint64_t* empty = full + Cfg::kMaxKb;        // [kMaxKb] MMA -> converters
    uint64_t* sfull = empty + Cfg::kMaxKb;       // [kMaxStg] loader (tx) -> converters
    uint64_t* sempty = sfull + Cfg::kMaxStg;     // [kMaxStg] converters -> loader
    uint64_t* tfull = sempty + Cfg::kMaxStg;     // [2] MMA -> epilogue
    uint64_t* tempty = tfull + 2;                // [2] epilogue -> MMA (leader's)
    uint64_t* bready = tempty + 2;               // resident B' landed
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bready + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const int64_t tile0 = blockIdx.x >> 1, tstep = gridDim.x >> 1;
    const int kb0 = p.src[0].kblocks;                           // k-blocks of source 0 (source 1 follows)
    const int kbl = kb0 + (p.nsrc > 1 ? p.src[1].kblocks : 0);  // per tile, both sources
    const int np = p.n_pad > kBM ? 2 : 1;                       // passes
    const int Np = p.n_pad / np;                                // MMA N (multiple of 32)
    // A' stage ring: one pass -> kMaxKb stages, each released after its MMAs; two passes -> the
    // tile's whole K stays resident (kbl stages) until the second pass has read it.
    const int R = np > 1 ? kbl : Cfg::kMaxKb;
    const uint32_t bt = static_cast<uint32_t>(Np / 2) * 64u;    // one resident (pass, kb, plane) tile
    // the staging ring takes the shared memory the resident B' leaves (a small weight image -> more
    // fp32 rows in flight: the narrow-N GEMMs stream A and are bound by the HBM bytes in flight)
    const uint32_t stg_off = (static_cast<uint32_t>(np * kbl * 2) * bt + 1023u) & ~1023u;
    const int nstg = min(Cfg::kMaxStg, static_cast<int>((Cfg::kEpiOff - stg_off) / kNtStgBytes));
    uint8_t* stg_base = smem + stg_off;
    int kt = 1 << 20;
    int bexp[2] = {0, 0};
    for (int q = 0; q < p.nsrc; ++q) {
        bexp[q] = *p.src[q].bexp;
        kt = min(kt, scale_exp(*p.src[q].amax_a) + bexp[q]);
    }
    const float sa0 = ldexpf(1.f, kt - bexp[0]), sa1 = ldexpf(1.f, kt - bexp[1]);

    if (warp == Cfg::kMma) {
        if (lane == 0) {
            for (int s = 0; s < Cfg::kMaxKb; ++s) {
                mbar_init(&full[s], Cfg::kCW * 2);
                mbar_init(&empty[s], 1);
            }
            for (int s = 0; s < Cfg::kMaxStg; ++s) {
                mbar_init(&sfull[s], 1);
                mbar_init(&sempty[s], Cfg::kCW);
            }
            for (int s = 0; s < 2; ++s) {
                mbar_init(&tfull[s], 1);
                mbar_init(&tempty[s], kNtEpiWarps * 2);
            }
            mbar_init(bready, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
        tmem_alloc_g<true>(tmem_slot);
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t full_l = mapa(smem_u32(full), 0);
    const uint32_t tempty_l = mapa(smem_u32(tempty), 0);

    if (warp == Cfg::kLoad) {
        if (lane == 0) {
            // resident B': for pass h, k-block kb (both sources), plane q, this CTA's Np / 2 rows of the
            // source's image (rows [kb][q][n_pad]; pass h covers columns h Np .. h Np + Np - 1, split by
            // rank). Both CTAs' bytes are counted on the leader's barrier (its MMAs read both halves).
            if (rank == 0) mbar_arrive_expect_tx(bready, 2u * static_cast<uint32_t>(np * kbl * 2) * bt);
            const uint32_t bready_l = mapa(smem_u32(bready), 0);
            for (int h = 0; h < np; ++h)
                for (int kb = 0; kb < kbl; ++kb)
                    for (int q = 0; q < 2; ++q) {
                        const int src = kb < kb0 ? 0 : 1, kl = kb < kb0 ? kb : kb - kb0;
                        tma_load_2d_pair(bres + ((h * kbl + kb) * 2 + q) * bt, &p.src[src].tmap_b, 0,
                                         (kl * 2 + q) * p.n_pad + h * Np + static_cast<int32_t>(rank) * (Np / 2),
                                         bready_l);
                    }
        }
        __syncwarp();
        Ring ring;
        for (int64_t tile = tile0; tile < p.tiles; tile += tstep)
            for (int kb = 0; kb < kbl; ++kb, ring.next(nstg)) {
                const int src = kb < kb0 ? 0 : 1, kl = kb < kb0 ? kb : kb - kb0;
                mbar_wait(&sempty[ring.idx], ring.phase ^ 1);
                if (lane == 0) {
                    mbar_arrive_expect_tx(&sfull[ring.idx], kNtStgBytes);
                    tma_load_2d(stg_base + ring.idx * kNtStgBytes, &p.src[src].tmap, kl * kNtBK,
                                static_cast<int32_t>(tile * Cfg::kRows + rank * kBM), &sfull[ring.idx]);
                }
                __syncwarp();
            }
    } else if (warp < Cfg::kCW) {
        // converters: warp w owns TMEM lane quarter q = w & 3 (rows 32q + lane) and k half kh = w >> 2
        // of each 32-k stage: 16 fp32 of its row (4 x LDS.128 from the SW128 staging) -> 8 hi + 8 lo
        // columns of A' stage st (hi at column 32 st + 8 kh, lo 16 columns further).
        const int q = warp & 3, kh = warp >> 2;
        const int r = 32 * q + lane;
        Ring sr;
        uint32_t g = 0;  // k-blocks converted so far (A' ring position)
        for (int64_t tile = tile0; tile < p.tiles; tile += tstep)
            for (int kb = 0; kb < kbl; ++kb, sr.next(nstg), ++g) {
                const uint32_t st = g % R;
                const float sa = kb < kb0 ? sa0 : sa1;
                mbar_wait(&empty[st], ((g / R) & 1) ^ 1);  // the MMAs that read this stage last are done
                mbar_wait(&sfull[sr.idx], sr.phase);
                const uint8_t* rowp = stg_base + sr.idx * kNtStgBytes + r * (kNtBK * 4);
                float4 x[4];
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    x[c] = *reinterpret_cast<const float4*>(rowp + (((4 * kh + c) ^ (r & 7)) << 4));
                uint32_t hi[8], lo[8];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    split2(x[c].x, x[c].y, sa, hi[2 * c], lo[2 * c]);
                    split2(x[c].z, x[c].w, sa, hi[2 * c + 1], lo[2 * c + 1]);
                }
                tc_fence_after();  // orders the stores after the MMAs that read this stage last
                const uint32_t tcol = tmem_base + (static_cast<uint32_t>(32 * q) << 16) + st * 32 + 8 * kh;
                tmem_st8(tcol, hi);
                tmem_st8(tcol + 16, lo);
                tmem_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive_cluster(full_l + st * 8);
                    mbar_arrive(&sempty[sr.idx]);
                }
            }
    } else if (warp == Cfg::kMma) {
        if (rank == 0) {
            mbar_wait(bready, 0);
            const uint32_t idesc = idesc_f16(Cfg::kRows, Np);
            uint32_t t = 0;
            for (int64_t tile = tile0; tile < p.tiles; tile += tstep, ++t)
                for (int h = 0; h < np; ++h) {
                    const uint32_t u = t * np + h, acc = u & 1;
                    mbar_wait_cluster(&tempty[acc], ((u >> 1) & 1) ^ 1);
                    tc_fence_after();
                    const uint32_t d_tmem = tmem_base + 256 + acc * Np;
                    for (int kb = 0; kb < kbl; ++kb) {
                        const uint32_t g = t * kbl + kb, st = g % R;
                        if (h == 0) {
                            mbar_wait_cluster(&full[st], (g / R) & 1);
                            tc_fence_after();
                        }
                        if (lane == 0) {
                            const uint8_t* bt0 = bres + ((h * kbl + kb) * 2) * bt;
                            const uint64_t bhi = desc_sw64(smem_u32(bt0)), blo = desc_sw64(smem_u32(bt0 + bt));
#pragma unroll
                            for (int k = 0; k < kNtBK / 16; ++k) {
                                const uint64_t adv = static_cast<uint64_t>(k * 32) >> 4;
                                const uint32_t tah = tmem_base + st * 32 + k * 8;  // lo plane 16 columns after hi
                                mma_f16_ts_pair(d_tmem, tah, bhi + adv, idesc, (kb | k) ? 1u : 0u);
                                mma_f16_ts_pair(d_tmem, tah, blo + adv, idesc, 1u);
                                mma_f16_ts_pair(d_tmem, tah + 16, bhi + adv, idesc, 1u);
                            }
                            if (h == np - 1) mma_commit_g<true>(&empty[st]);
                            if (kb == kbl - 1) mma_commit_g<true>(&tfull[acc]);
                        }
                        __syncwarp();
                    }
                }
        }
    } else {
        // epilogue (8 warps): as the general kernel, per pass: TMEM columns 256 + acc Np + c0 are output
        // columns h Np + c0.
        const int ew = warp & 3;
        const int half = (warp - Cfg::kCW) >> 2;
        const float unscale = ldexpf(1.f, -kt);
        uint8_t* box = epi_base + (warp - Cfg::kCW) * kNtEpiBuf;
        float amx = 0.f;
        uint32_t t = 0;
        for (int64_t tile = tile0; tile < p.tiles; tile += tstep, ++t) {
            const int64_t row0 = tile * Cfg::kRows + rank * kBM + ew * 32;
            float sc = 1.f;
            if (EPI == kEpiRowScale && row0 + lane < p.M) sc = p.row_scale[row0 + lane];
            for (int h = 0; h < np; ++h) {
                const uint32_t u = t * np + h, acc = u & 1;
                mbar_wait(&tfull[acc], (u >> 1) & 1);
                tc_fence_after();
                for (int c0 = half * 32; c0 < Np; c0 += 64) {
                    uint32_t rr[32];
                    tmem_ld32(tmem_base + 256 + acc * Np + (static_cast<uint32_t>(ew * 32) << 16) + c0, rr);
                    if (lane == 0) bulk_wait_read<0>();
                    __syncwarp();
                    const int col = h * Np + c0;
                    uint32_t pos = 0;
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        float x[4];
#pragma unroll
                        for (int qq = 0; qq < 4; ++qq) {
                            float v = __uint_as_float(rr[4 * j + qq]) * unscale;
                            if (EPI == kEpiRelu) {
                                v = fmaxf(v, 0.f);
                                pos |= (v > 0.f ? 1u : 0u) << (4 * j + qq);
                            }
                            if (EPI == kEpiRowScale) v = sc * v;
                            if (AMAX) amx = fmaxf(amx, fabsf(v));
                            x[qq] = v;
                        }
                        *reinterpret_cast<float4*>(box + lane * 128 + ((j ^ (lane & 7)) << 4)) =
                            make_float4(x[0], x[1], x[2], x[3]);
                    }
                    if (EPI == kEpiRelu && p.relu_pos && col < p.N && row0 + lane < p.M)
                        p.relu_pos[(row0 + lane) * ((p.N + 31) >> 5) + (col >> 5)] = pos;
                    fence_proxy_async();
                    __syncwarp();
                    if (lane == 0 && row0 < p.M) tma_store_2d(&p.tmap_c, box, col, static_cast<int32_t>(row0));
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(tempty_l + acc * 8);
            }
        }
        if (lane == 0) bulk_wait_read<0>();
        if (AMAX) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) amx = fmaxf(amx, __shfl_xor_sync(0xffffffffu, amx, o));
            if (lane == 0) atomicMax(reinterpret_cast<unsigned int*>(p.amax_out), __float_as_uint(amx));
        }
    }
    tc_fence_before();
    cluster_sync();
    if (warp == Cfg::kMma) {
        tc_fence_after();
        tmem_dealloc_g<true>(tmem_base);
    }
}

// ---- B image prep (two grid-wide passes): |B| max -> exponent kB, then fp32 B
// (NT [N x K] or NN [K x N]) * 2^kB split into per-k-block [hi tile | lo tile],
// each n_pad rows x 32 k fp16 in the SW64 K-major layout.
__global__ void prep_b_amax_kernel(const float* __restrict__ B, int64_t ldb, int nn, int32_t N, int32_t K,
                                   float* amax) {
    float mx = 0.f;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < int64_t(N) * K;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int32_t a = static_cast<int32_t>(i / K), b = static_cast<int32_t>(i % K);
        mx = fmaxf(mx, fabsf(nn ? B[int64_t(b) * ldb + a] : B[int64_t(a) * ldb + b]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) atomicMax(reinterpret_cast<unsigned int*>(amax), __float_as_uint(mx));
}
__global__ void prep_b_split_kernel(const float* __restrict__ B, int64_t ldb, int nn, int32_t N, int32_t K,
                                    int32_t n_pad, int32_t kblocks, const float* amax, uint8_t* img,
                                    int32_t* bexp) {
    const int kexp = scale_exp(*amax);
    const float s = ldexpf(1.f, kexp);
    if (blockIdx.x == 0 && threadIdx.x == 0) *bexp = kexp;
    const int64_t total = int64_t(kblocks) * n_pad * 4;  // 16-byte chunks per (hi) image
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
        const int32_t kb = static_cast<int32_t>(i / (int64_t(n_pad) * 4));
        const int32_t rem = static_cast<int32_t>(i % (int64_t(n_pad) * 4));
        const int32_t n = rem >> 2, c = rem & 3;
        float v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int32_t k = kb * kNtBK + c * 8 + q;
            v[q] = (n < N && k < K) ? (nn ? B[int64_t(k) * ldb + n] : B[int64_t(n) * ldb + k]) : 0.f;
        }
        uint4 hi, lo;
        split2(v[0], v[1], s, hi.x, lo.x);
        split2(v[2], v[3], s, hi.y, lo.y);
        split2(v[4], v[5], s, hi.z, lo.z);
        split2(v[6], v[7], s, hi.w, lo.w);
        uint8_t* base = img + int64_t(kb) * 2 * n_pad * 64;
        const uint32_t off = sw64_off(n, c);
        *reinterpret_cast<uint4*>(base + off) = hi;
        *reinterpret_cast<uint4*>(base + int64_t(n_pad) * 64 + off) = lo;
    }
}

// =============================================================================
// Weight-gradient GEMM:  C[N1 x N2] = A^T Bcat,  A [M x N1], Bcat = [B1 | B2]
// [M x N2], K = M (partition rows, millions). The MMA's "M" is N1 (tiles of
// 128), its "N" is N2 (tiles of <= 256), its K runs over rows. Row-major
// activations are MN-major operands, so row slices are bulk-copied straight to
// staging and converted into the MN-major SWIZZLE_128B layout. Split-K over
// rows; inside a CTA the TMEM accumulator is drained every kChunkKb k-blocks
// (1024 rows) into an fp32 partial (the tensor-core accumulate is not
// round-to-nearest, so long K runs in TMEM would bias the sum); splits are
// summed in a fixed order afterwards (deterministic).
// =============================================================================
struct TnB {
    const float* ptr;
    int64_t ld;
    const int32_t* rows;
    int32_t cols;
    const float* amax;
};
struct alignas(64) TnParams {
    CUtensorMap tm_a, tm_b1, tm_b2;  // 2D fp32 maps, box 32 columns x 32 rows, SWIZZLE_128B
    const float* a;
    int64_t lda;
    int32_t N1;
    const float* amax_a;
    TnB b[2];
    int nb;          // number of B sources
    int32_t n2a;     // columns of B1 (B2 follows)
    int32_t N2;
    int64_t M;
    int64_t rows_per_split;
    int32_t tiles1, tiles2;
    // Second A source (dual weight-gradient launch, A = [A1 | A2]: dU and dW of one layer share
    // their B columns and stream every operand once): A' columns >= n1a come from tm_a2.
    CUtensorMap tm_a2;
    const float* amax_a2;
    int32_t n1a;
    // The (A' tile, B' tile) pairs computed per split (a dual launch skips A2 x B1).
    int32_t ntiles;
    int8_t tile_a[8], tile_b[8];
    int32_t stagger;    // A' in TMEM, one accumulator: stagger the pairs' drain points (tn_run_end)
    int32_t pf_dist;    // L2-prefetch the operand boxes of k-block kb + pf_dist when loading kb (0: off)
    int32_t split_acc;  // A' in TMEM: split full tiles' accumulator into two staggered halves
    float* ws;       // [splits][N1][N2] fp32 partials
    CUtensorMap tm_ws;  // 3D map over ws (box 32 x 32 x 1, SW128): the drains' TMA stores / reduce-adds
    int32_t ws_tma;     // use tm_ws (N2 % 4 == 0, one accumulator, SC_TN_TMA_DRAIN != 0)
    unsigned long long* trace;  // optional (SC_TN_TRACE=1): per-role wait / total cycles, summed over CTAs
};

// MN-major SW128 descriptor: LBO = stride between 64-element MN atoms,
// SBO = stride between 8-row K groups (validated against fp64 in tests).
__device__ __forceinline__ uint64_t desc_mn_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return static_cast<uint64_t>((saddr & 0x3FFFF) >> 4) | (static_cast<uint64_t>(lbo >> 4) << 16) |
           (static_cast<uint64_t>(sbo >> 4) << 32) | (static_cast<uint64_t>(1) << 46) |
           (static_cast<uint64_t>(2) << 61);
}
// kind::f16, D f32, A/B f16, A and B MN-major (bits 15, 16).
__host__ __device__ constexpr uint32_t idesc_f16_mn(int M, int N) {
    return (1u << 4) | (1u << 15) | (1u << 16) | (static_cast<uint32_t>(N >> 3) << 17) |
           (static_cast<uint32_t>(M >> 4) << 24);
}
// Same with A K-major (A read from TMEM), B MN-major.
__host__ __device__ constexpr uint32_t idesc_f16_at(int M, int N) {
    return (1u << 4) | (1u << 16) | (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
}
// Byte offset of the 16-byte chunk (8 consecutive mn at one k) in an MN-major
// SW128 tile of 32 k rows laid out [mn_atom][k_atom(4)][8 k rows][128 B].
constexpr uint32_t kTnLbo = 4 * 1024;  // MN atom stride
constexpr uint32_t kTnSbo = 1024;      // K group stride
__device__ __forceinline__ uint32_t mn_off(uint32_t mn, uint32_t k) {
    return (mn >> 6) * kTnLbo + (k >> 3) * kTnSbo + (k & 7) * 128 + ((((mn & 63) >> 3) ^ (k & 7)) << 4);
}

// Shared-memory plan of the TN kernel. PAIR: a CTA pair (cta_group::2) owns a
// 256-column slice of A' (M = 256, 128 per CTA) and splits the B' tile's columns
// between its two CTAs, so each B' element is converted once per pair instead
// of once per 128-column A' tile, and per-SM conversion work drops by a third.
// AT (pairs only): the A' operand lives in TMEM instead of shared memory. The
// converters write its fp16 hi / lo halves with tcgen05.st (TMEM lane = A'
// column = output row) and the MMAs read A from TMEM, which removes the A'
// fp16 stores and two thirds of the MMA operand reads from the SM's shared-
// memory bandwidth (the TN kernel's limit). TMEM then holds one 256-column
// accumulator plus kStages 32-column A' stages (hi 16 + lo 16), so the
// accumulator is single-buffered: the MMAs wait for each 1024-row drain.
template <bool PAIR, bool AT = false>
struct TnCfg {
// A'-in-TMEM stages (TMEM ring + B' smem tiles) / fp32 staging slots: 5 / 4 (6 / 3 and 4 / 4 measured
// 1-1.5 ms per epoch slower, profiles/r02_tn_stages_ab.txt)
#ifndef SC_TN_AT_STAGES
#define SC_TN_AT_STAGES 5
#define SC_TN_AT_STG 4
#endif
    static constexpr int kStages = AT ? SC_TN_AT_STAGES : (PAIR ? 3 : 2);
    static constexpr int kStg = AT ? SC_TN_AT_STG : (PAIR ? 3 : 2);
    static constexpr int kAcc = AT ? 1 : 2;                  // TMEM accumulators
    // warp roles: converters 0 .. kCW-1, epilogue kCW .. kCW+3, MMA issuer, TMA loader
    static constexpr int kCW = kConvWarps;  // (16 with A' in TMEM measured 2 % slower: converters are not the limit)
    static constexpr int kC = kCW * 32;
    static constexpr int kMma = kCW + 4, kLoad = kCW + 5, kThr = (kCW + 6) * 32;
    static constexpr int kChunk = AT ? 2 * kChunkKb : kChunkKb;  // k-blocks per accumulation
    static constexpr int kBLoc = PAIR ? kMaxN / 2 : kMaxN;  // B' columns held per CTA
    static constexpr int kBTile = kBLoc * kTnBK * 2;        // one (hi or lo) B' tile
    static constexpr int kStage = (AT ? 0 : 2 * kTnATile) + 2 * kBTile;  // smem per stage
    static constexpr int kStgB = kTnBK * kBLoc * 4;
    static constexpr int kStgSlot = kTnStgA + kStgB;
    static constexpr int kStgOff = kStages * kStage;
    static constexpr int kEpiOff = kStgOff + kStg * kStgSlot;
    static constexpr int kEpiPitch = 33;                     // drain transpose tile: 32 x 33 floats per warp
    static constexpr int kBarOff = kEpiOff + 4 * 32 * kEpiPitch * 4;
    static constexpr int kSmem = kBarOff + 256 + 1024;
    static constexpr int kACols = PAIR ? 2 * kBM : kBM;      // A' columns per tile
};
static_assert(TnCfg<true>::kSmem <= 232448 && TnCfg<false>::kSmem <= 232448, "TN shared memory");
static_assert(TnCfg<true, true>::kSmem <= 232448 && 256 + 32 * TnCfg<true, true>::kStages <= 512, "TN (A in TMEM)");


// Accumulation runs of half h (A' in TMEM, split accumulator): runs end at the k-blocks where
// (kb + off_h) % kRun == 0, off_1 = kRun / 2 (staggered), and at kblocks. Returns the (exclusive)
// end of the run that starts at `start`.
constexpr int kRun = 2 * kChunkKb;
// `stag` (one accumulator) shifts a CTA pair's run boundaries so that the pairs' drains, during
// which their tensor pipe and HBM stream pause, do not all fall on the same k-blocks.
__device__ __forceinline__ int tn_run_end(int h, int start, int kblocks, int nh, int stag) {
    const int off = nh > 1 ? (h == 1 ? kRun / 2 : 0) : stag;
    const int end = start + (kRun - (start + off) % kRun);
    return end < kblocks ? end : kblocks;
}

template <bool PAIR, bool AT = false>
__global__ void __launch_bounds__(TnCfg<PAIR, AT>::kThr, 1) gemm_tn_f16x3_kernel(const __grid_constant__ TnParams p) {
    static_assert(!AT || PAIR, "A in TMEM needs the CTA-pair layout");
    using Cfg = TnCfg<PAIR, AT>;
    extern __shared__ __align__(16) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* stg_base = smem + Cfg::kStgOff;  // kStg x [A' rows | B' rows]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::kBarOff);
    uint64_t* full = bars;                     // [kStages] converters -> MMA (leader's)
    uint64_t* empty = full + Cfg::kStages;     // [kStages] MMA -> converters
    uint64_t* sfull = empty + Cfg::kStages;    // [kStg] loader (tx) -> converters
    uint64_t* sempty = sfull + Cfg::kStg;      // [kStg] converters -> loader
    uint64_t* tfull = sempty + Cfg::kStg;      // [2] MMA -> epilogue
    uint64_t* tempty = tfull + 2;              // [2] epilogue -> MMA (leader's)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    const uint32_t rank = PAIR ? cluster_ctarank() : 0u;
#ifdef SC_TN_TRACE_BUILD
    unsigned long long w_a = 0, w_b = 0;  // diagnostics: wait cycles of this thread's role
    const long long t_start = p.trace ? clock64() : 0;
#endif
    const int unit = PAIR ? static_cast<int>(blockIdx.x >> 1) : static_cast<int>(blockIdx.x);
    const int split = unit / p.ntiles, tile = unit % p.ntiles;
    const int32_t n10 = p.tile_a[tile] * Cfg::kACols + static_cast<int32_t>(rank) * kBM;  // this CTA's A' cols
    const int32_t n20 = p.tile_b[tile] * kMaxN;                                           // tile's B' cols
    const bool a_second = n10 >= p.n1a;  // this CTA's A' columns come from A2 (dual launch)
    const CUtensorMap* tm_a = a_second ? &p.tm_a2 : &p.tm_a;
    const int32_t a_col0 = a_second ? n10 - p.n1a : n10;  // first A' column within its source
    const int32_t na = max(0, min(kBM, p.N1 - n10));  // valid A' columns of this CTA
    const int32_t nb = min(kMaxN, p.N2 - n20);        // valid B' columns of the tile
    // MMA N; a pair splits it into two 32-column-aligned halves (TMA boxes never straddle B1 | B2)
    const int32_t nb_pad = PAIR ? (nb + 63) / 64 * 64 : (nb + 15) / 16 * 16;
    const int32_t nloc = PAIR ? nb_pad / 2 : nb_pad;                  // B' columns held by this CTA
    const int32_t nb0 = n20 + static_cast<int32_t>(rank) * nloc;      // first of them
    const int32_t nbl = max(0, min(nloc, nb - static_cast<int32_t>(rank) * nloc));  // valid ones
    const int64_t r0 = int64_t(split) * p.rows_per_split;
    const int64_t r1 = min(p.M, r0 + p.rows_per_split);
    const int kblocks = r1 > r0 ? static_cast<int>((r1 - r0 + kTnBK - 1) / kTnBK) : 0;
    const int nchunks = (kblocks + Cfg::kChunk - 1) / Cfg::kChunk;
    // A' in TMEM: a full 256-column tile splits its accumulator into two staggered halves
    const int nh = (AT && p.split_acc && nb_pad == 2 * kBM) ? 2 : 1;
    const int stag = p.stagger ? (unit & 3) * (kRun / 4) : 0;

    constexpr int kBOff = AT ? 0 : 2 * kTnATile;  // B' hi / lo tiles within a stage
    const int ka = scale_exp(*(a_second ? p.amax_a2 : p.amax_a));
    int kbx = scale_exp(*p.b[0].amax);
    if (p.nb > 1) kbx = min(kbx, scale_exp(*p.b[1].amax));

    if (warp == Cfg::kMma) {
        if (lane == 0) {
            for (int s = 0; s < Cfg::kStages; ++s) {
                mbar_init(&full[s], Cfg::kCW * (PAIR ? 2 : 1));
                mbar_init(&empty[s], 1);
            }
            for (int s = 0; s < Cfg::kStg; ++s) {
                mbar_init(&sfull[s], 1);
                mbar_init(&sempty[s], Cfg::kCW);
            }
            for (int s = 0; s < 2; ++s) {  // kAcc accumulators, or (A' in TMEM) the two halves of one
                mbar_init(&tfull[s], 1);
                mbar_init(&tempty[s], 4 * (PAIR ? 2 : 1));
            }
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
        tmem_alloc_g<PAIR>(tmem_slot);
    }
    tc_fence_before();
    if constexpr (PAIR) cluster_sync();
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t full_l = PAIR ? mapa(smem_u32(full), 0) : smem_u32(full);
    const uint32_t tempty_l = PAIR ? mapa(smem_u32(tempty), 0) : smem_u32(tempty);

    if (warp == Cfg::kLoad) {
        // ================= loader: 2D TMA boxes (32 columns x 32 rows, SWIZZLE_128B) -> staging =================
        // A' needs ceil(na/32) boxes, B' ceil(nbl/32) (each from B1 or B2; n2a is a multiple of 32).
        const int a_boxes = (na + 31) >> 5, b_boxes = (nbl + 31) >> 5;
        const uint32_t bytes = static_cast<uint32_t>(a_boxes + b_boxes) * kTnBox;
        const uint64_t pol_b = l2_evict_first();
        Ring ring;
        for (int kb = 0; kb < kblocks; ++kb, ring.next(Cfg::kStg)) {
            const int32_t k0 = static_cast<int32_t>(r0 + int64_t(kb) * kTnBK);
            TN_TIMED_WAIT(w_a, mbar_wait(&sempty[ring.idx], ring.phase ^ 1));
            uint8_t* sa = stg_base + ring.idx * Cfg::kStgSlot;
            uint8_t* sb = sa + kTnStgA;
            if (lane == 0) mbar_arrive_expect_tx(&sfull[ring.idx], bytes);
            __syncwarp();
            if (lane < a_boxes) tma_load_2d(sa + lane * kTnBox, tm_a, a_col0 + 32 * lane, k0, &sfull[ring.idx]);
            if (lane < b_boxes) {  // B' columns are read by this CTA only: stream them through L2
                const int32_t c = nb0 + 32 * lane;
                if (c < p.n2a) tma_load_2d_hint(sb + lane * kTnBox, &p.tm_b1, c, k0, &sfull[ring.idx], pol_b);
                else tma_load_2d_hint(sb + lane * kTnBox, &p.tm_b2, c - p.n2a, k0, &sfull[ring.idx], pol_b);
            }
            if (p.pf_dist > 0 && kb + p.pf_dist < kblocks) {  // the same boxes pf_dist k-blocks ahead -> L2
                const int32_t kp = k0 + p.pf_dist * kTnBK;
                if (lane < a_boxes) tma_prefetch_2d(tm_a, a_col0 + 32 * lane, kp);
                if (lane < b_boxes) {
                    const int32_t c = nb0 + 32 * lane;
                    if (c < p.n2a) tma_prefetch_2d(&p.tm_b1, c, kp);
                    else tma_prefetch_2d(&p.tm_b2, c - p.n2a, kp);
                }
            }
        }
    } else if (warp < Cfg::kCW) {
        // ================= converters: swizzled staging -> MN-major fp16 hi/lo =================
        // Row-fastest mapping (idx & 31 = row): 8 consecutive threads read the same logical chunk
        // of 8 rows, which the 128 B swizzle spreads over distinct banks.
        const int tid = threadIdx.x;
        const float sa_ = ldexpf(1.f, ka), sb_ = ldexpf(1.f, kbx);
        const int bch = nloc >> 3;
        Ring mr, sr;
        for (int kb = 0; kb < kblocks; ++kb, mr.next(Cfg::kStages), sr.next(Cfg::kStg)) {
            const int64_t k0 = r0 + int64_t(kb) * kTnBK;
            const int rows_ok = r1 - k0 < kTnBK ? static_cast<int>(r1 - k0) : kTnBK;
            uint8_t* st = smem + mr.idx * Cfg::kStage;
            const uint8_t* sga = stg_base + sr.idx * Cfg::kStgSlot;
            const uint8_t* sgb = sga + kTnStgA;
            TN_TIMED_WAIT(w_a, mbar_wait(&empty[mr.idx], mr.phase ^ 1));
            TN_TIMED_WAIT(w_b, mbar_wait(&sfull[sr.idx], sr.phase));
            // A': 32 rows x 16 chunks of 8 columns; B': 32 rows x bch chunks (this CTA's columns).
            // Interior stages (all rows and columns valid) skip the masking.
            const bool whole = rows_ok == kTnBK && na == kBM && nbl == nloc;  // block-uniform
            auto load8 = [&](const uint8_t* sg, int kr, int ch, int valid, float4& x0, float4& x1) {
                const uint8_t* rowp = sg + (ch >> 2) * kTnBox + kr * 128;
                x0 = *reinterpret_cast<const float4*>(rowp + (((2 * (ch & 3)) ^ (kr & 7)) << 4));
                x1 = *reinterpret_cast<const float4*>(rowp + (((2 * (ch & 3) + 1) ^ (kr & 7)) << 4));
                if (valid < 8) mask8(x0, x1, valid);
            };
            if constexpr (AT) {
                // A' -> TMEM: warp w owns TMEM lane quarter w & 3 (A' columns 32q .. 32q+31, one per
                // lane) and k rows 16 (w >> 2) .. +15 of the stage. Column-wise reads of the row-major
                // staging are conflict-free (one 128 B row per instruction, swizzled chunks).
                constexpr int kRows = kTnBK / (Cfg::kCW / 4);  // k rows per warp (8 with 16 converter warps)
                const int q = warp & 3, kh = warp >> 2;
                const int m = 32 * q + lane;
                const uint8_t* box = sga + q * kTnBox + (((lane & 3)) << 2);
                float x[kRows];
#pragma unroll
                for (int i = 0; i < kRows; ++i) {
                    const int kr = kRows * kh + i;
                    const float v = *reinterpret_cast<const float*>(box + kr * 128 + ((((lane >> 2) ^ (kr & 7))) << 4));
                    x[i] = (whole || (kr < rows_ok && m < na)) ? v : 0.f;
                }
                uint32_t hi[kRows / 2], lo[kRows / 2];
#pragma unroll
                for (int j = 0; j < kRows / 2; ++j) split2(x[2 * j], x[2 * j + 1], sa_, hi[j], lo[j]);
                const uint32_t tcol =
                    tmem_base + (static_cast<uint32_t>(32 * q) << 16) + 256 + mr.idx * 32 + (kRows / 2) * kh;
                tmem_st<kRows / 2>(tcol, hi);
                tmem_st<kRows / 2>(tcol + 16, lo);
            }
            if (whole) {
                // all of the stage's shared loads first (up to 8 x LDS.128 in flight), then convert
                constexpr int kJB = (4 * Cfg::kBLoc + Cfg::kC - 1) / Cfg::kC;  // B' items (row, 8 cols) per thread
                constexpr int kJA = (4 * kBM + Cfg::kC - 1) / Cfg::kC;         // A' items (smem path)
                float4 xa[kJA][2], xb[kJB][2];
#pragma unroll
                for (int j = 0; j < kJA; ++j) {
                    if constexpr (AT) break;
                    const int idx = tid + j * Cfg::kC;
                    load8(sga, idx & 31, idx >> 5, 8, xa[j][0], xa[j][1]);
                }
#pragma unroll
                for (int j = 0; j < kJB; ++j) {
                    const int idx = tid + j * Cfg::kC;
                    if ((idx >> 5) < bch) load8(sgb, idx & 31, idx >> 5, 8, xb[j][0], xb[j][1]);
                }
#pragma unroll
                for (int j = 0; j < kJA; ++j) {
                    if constexpr (AT) break;
                    const int idx = tid + j * Cfg::kC;
                    split8_store(xa[j][0], xa[j][1], sa_, st, st + kTnATile, mn_off((idx >> 5) * 8, idx & 31));
                }
#pragma unroll
                for (int j = 0; j < kJB; ++j) {
                    const int idx = tid + j * Cfg::kC;
                    const int kr = idx & 31, ch = idx >> 5;
                    if (ch < bch)
                        split8_store(xb[j][0], xb[j][1], sb_, st + kBOff, st + kBOff + Cfg::kBTile,
                                     mn_off(ch * 8, kr));
                }
            } else {
#pragma unroll
                for (int j = 0; j < (4 * kBM + Cfg::kC - 1) / Cfg::kC; ++j) {
                    if constexpr (AT) break;
                    const int idx = tid + j * Cfg::kC;
                    const int kr = idx & 31, ch = idx >> 5;
                    float4 x0 = make_float4(0.f, 0.f, 0.f, 0.f), x1 = x0;
                    const int valid = kr < rows_ok ? min(8, na - ch * 8) : 0;
                    if (valid > 0) load8(sga, kr, ch, valid, x0, x1);
                    split8_store(x0, x1, sa_, st, st + kTnATile, mn_off(ch * 8, kr));
                }
#pragma unroll
                for (int j = 0; j < (4 * Cfg::kBLoc + Cfg::kC - 1) / Cfg::kC; ++j) {
                    const int idx = tid + j * Cfg::kC;
                    const int kr = idx & 31, ch = idx >> 5;
                    if (ch >= bch) continue;
                    float4 x0 = make_float4(0.f, 0.f, 0.f, 0.f), x1 = x0;
                    const int valid = kr < rows_ok ? min(8, nbl - ch * 8) : 0;
                    if (valid > 0) load8(sgb, kr, ch, valid, x0, x1);
                    split8_store(x0, x1, sb_, st + kBOff, st + kBOff + Cfg::kBTile, mn_off(ch * 8, kr));
                }
            }
            if constexpr (AT) {
                tmem_wait_st();   // the A' stage is in TMEM
                tc_fence_before();
            }
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
                if constexpr (PAIR) mbar_arrive_cluster(full_l + mr.idx * 8);
                else mbar_arrive(&full[mr.idx]);
                mbar_arrive(&sempty[sr.idx]);
            }
        }
    } else if (warp == Cfg::kMma && AT) {
        // ================= MMA issuer, A' in TMEM: split accumulator (the pair's leader only) =================
        // A full 256-column tile runs as two N = 128 halves with their own accumulation runs, staggered by
        // half a run: half 0 drains after k-blocks 64, 128, ..., half 1 after 32, 96, ... While one half is
        // drained, the issuer keeps the tensor pipe busy with the other half's MMAs on the stages already
        // converted (up to kStages - 1 k-blocks ahead), so the single 256-column accumulator no longer
        // stalls the pipe for a whole drain. Every element still accumulates <= kChunk k-blocks per run.
        if (rank == 0 && lane == 0) {
            // Per-half state in scalars (no runtime-indexed arrays: those live in local memory and
            // made this single-thread loop slower than the tensor pipe it feeds).
            const uint32_t idesc = idesc_f16_at(Cfg::kACols, nb_pad / nh);
            int kb0 = 0, kb1 = nh > 1 ? 0 : kblocks;                 // next k-block of each half
            int beg0 = 0, beg1 = 0;                                  // first k-block of the current run
            int end0 = tn_run_end(0, 0, kblocks, nh, stag), end1 = nh > 1 ? tn_run_end(1, 0, kblocks, nh, stag) : kblocks;
            uint32_t par0 = 1, par1 = 1;                             // tempty parity the next run waits for
            bool fresh0 = true, fresh1 = true;                       // at a run start: accumulator must be free
            auto issue = [&](int h, int& kb, int& beg, int& end, uint32_t& par, bool& fresh, int other_kb) {
                if (fresh) {  // block (suspended in try_wait) until the epilogue has drained this half
                    TN_TIMED_WAIT(w_b, mbar_wait(&tempty[h], par));
                    tc_fence_after();
                    fresh = false;
                }
                const int st = kb % Cfg::kStages;
                TN_TIMED_WAIT(w_a, mbar_wait(&full[st], (kb / Cfg::kStages) & 1));
                tc_fence_after();
                const uint8_t* stp = smem + st * Cfg::kStage;
                const uint32_t bhi = smem_u32(stp) + h * kTnLbo, blo = smem_u32(stp + Cfg::kBTile) + h * kTnLbo;
                const uint32_t d_tmem = tmem_base + h * 128;
#pragma unroll
                for (int k = 0; k < kTnBK / 16; ++k) {
                    const uint32_t adv = k * 2 * kTnSbo;  // 16 rows = 2 K groups
                    const uint64_t dbh = desc_mn_sw128(bhi + adv, kTnLbo, kTnSbo);
                    const uint64_t dbl = desc_mn_sw128(blo + adv, kTnLbo, kTnSbo);
                    const uint32_t tah = tmem_base + 256 + st * 32 + k * 8;  // lo plane 16 columns after hi
                    mma_f16_ts_pair(d_tmem, tah, dbh, idesc, (kb == beg && k == 0) ? 0u : 1u);
                    mma_f16_ts_pair(d_tmem, tah, dbl, idesc, 1u);
                    mma_f16_ts_pair(d_tmem, tah + 16, dbh, idesc, 1u);
                }
                if (kb == end - 1) {  // end of this half's run: hand it to the epilogue
                    mma_commit_g<PAIR>(&tfull[h]);
                    par ^= 1u;
                    fresh = true;
                    beg = end;
                    end = tn_run_end(h, end, kblocks, nh, stag);
                }
                if (other_kb > kb) mma_commit_g<PAIR>(&empty[st]);  // both halves issued: stage free
                ++kb;
            };
            while (kb0 < kblocks || kb1 < kblocks) {
                bool one = kb1 >= kb0;  // the lagging half first (ties: half 0)
                if (nh > 1) {
                    // the lagging half's accumulator is still draining: run the other one ahead if it can
                    // go now (within the stage ring, its own accumulator free)
                    if (one && fresh0 && !mbar_test(&tempty[0], par0) && kb1 < kblocks &&
                        kb1 <= kb0 + Cfg::kStages - 1 && (!fresh1 || mbar_test(&tempty[1], par1)))
                        one = false;
                    else if (!one && fresh1 && !mbar_test(&tempty[1], par1) && kb0 < kblocks &&
                             kb0 <= kb1 + Cfg::kStages - 1 && (!fresh0 || mbar_test(&tempty[0], par0)))
                        one = true;
                }
                if (one) issue(0, kb0, beg0, end0, par0, fresh0, kb1);
                else issue(1, kb1, beg1, end1, par1, fresh1, kb0);
            }
        }
        __syncwarp();
    } else if (warp == Cfg::kMma) {
        // ================= MMA issuer (the pair's leader only) =================
        if (!PAIR || rank == 0) {
            const uint32_t idesc = AT ? idesc_f16_at(Cfg::kACols, nb_pad) : idesc_f16_mn(Cfg::kACols, nb_pad);
            Ring mr;
            for (int chunk = 0; chunk < nchunks; ++chunk) {
                const uint32_t acc = chunk % Cfg::kAcc;
                const uint32_t d_tmem = tmem_base + acc * 256;
                TN_TIMED_WAIT(w_b, mbar_wait(&tempty[acc], ((chunk / Cfg::kAcc) & 1) ^ 1));
                tc_fence_after();
                const int kb_end = min(kblocks, (chunk + 1) * Cfg::kChunk);
                for (int kb = chunk * Cfg::kChunk; kb < kb_end; ++kb, mr.next(Cfg::kStages)) {
                    TN_TIMED_WAIT(w_a, mbar_wait(&full[mr.idx], mr.phase));
                    tc_fence_after();
                    if (lane == 0) {
                        const uint8_t* st = smem + mr.idx * Cfg::kStage;
                        const uint32_t ahi = smem_u32(st), alo = smem_u32(st + kTnATile);
                        const uint32_t bhi = smem_u32(st + kBOff), blo = smem_u32(st + kBOff + Cfg::kBTile);
#pragma unroll
                        for (int k = 0; k < kTnBK / 16; ++k) {
                            const uint32_t adv = k * 2 * kTnSbo;  // 16 rows = 2 K groups
                            const uint64_t dbh = desc_mn_sw128(bhi + adv, kTnLbo, kTnSbo);
                            const uint64_t dbl = desc_mn_sw128(blo + adv, kTnLbo, kTnSbo);
                            const uint32_t first = (kb == chunk * Cfg::kChunk && k == 0) ? 0u : 1u;
                            if constexpr (AT) {  // 16 k = 8 TMEM columns; lo plane 16 columns after hi
                                const uint32_t tah = tmem_base + 256 + mr.idx * 32 + k * 8;
                                mma_f16_ts_pair(d_tmem, tah, dbh, idesc, first);
                                mma_f16_ts_pair(d_tmem, tah, dbl, idesc, 1u);
                                mma_f16_ts_pair(d_tmem, tah + 16, dbh, idesc, 1u);
                            } else {
                                const uint64_t dah = desc_mn_sw128(ahi + adv, kTnLbo, kTnSbo);
                                const uint64_t dal = desc_mn_sw128(alo + adv, kTnLbo, kTnSbo);
                                mma_f16_g<PAIR>(d_tmem, dah, dbh, idesc, first);
                                mma_f16_g<PAIR>(d_tmem, dah, dbl, idesc, 1u);
                                mma_f16_g<PAIR>(d_tmem, dal, dbh, idesc, 1u);
                            }
                        }
                        mma_commit_g<PAIR>(&empty[mr.idx]);
                        if (kb == kb_end - 1) mma_commit_g<PAIR>(&tfull[acc]);
                    }
                    __syncwarp();
                }
            }
        }
    } else if (AT) {
        // ================= epilogue (A' in TMEM): drain each half's run into the fp32 partial ws[split] =========
        // Runs complete in order of their last k-block (half 0 first on ties); each drain covers the half's
        // TMEM columns (128 with two halves, else nb_pad), mapped back to the tile's B' columns: half h's
        // 32-column block j0 of the MMA's N = 128 came from CTA 0's local columns 64h + j0 (j0 < 64) or
        // CTA 1's 64h + j0 - 64 (tile columns 128 + ...). The first run of a half stores, later runs add
        // (fire-and-forget reductions at L2; one owner per element, program order: deterministic).
        const int ew = warp & 3;
        const int32_t m0w = n10 + ew * 32;  // first output row (N1 index) of this warp
        const int rows_here = max(0, min(32, p.N1 - m0w));
        const float unscale = ldexpf(1.f, -(ka + kbx));
        float* outw = p.ws + (int64_t(split) * p.N1 + m0w) * p.N2 + n20;
        float* orow = outw + int64_t(lane) * p.N2;
        const bool vec = (p.N2 & 3) == 0;
        const uint64_t pol_ws = l2_evict_last();
        float* tbuf = reinterpret_cast<float*>(smem + Cfg::kEpiOff) + ew * 32 * Cfg::kEpiPitch;
        if (p.ws_tma && nh == 1) {
            // TMA drain: each 32-column block of the run goes TMEM -> registers -> (unscaled) SW128 smem box
            // -> one bulk store (first run) or bulk reduce-add (later runs) into ws[split]; the tensor map
            // clips rows >= N1 / columns >= N2. The previous run's bulk groups are complete before the
            // next run's are issued, so every element's additions keep the run order (deterministic, the
            // same adds as the reduction path). The accumulator goes back to the MMAs once the TMEM loads
            // and box hand-offs are done, not after the L2 reductions.
            uint8_t* box = smem + Cfg::kEpiOff + ew * 4096;
            int endr = tn_run_end(0, 0, kblocks, 1, stag);
            uint32_t run = 0;
            while (kblocks > 0 && endr <= kblocks) {
                TN_TIMED_WAIT(w_a, mbar_wait(&tfull[0], run & 1));
                tc_fence_after();
                if (lane == 0) bulk_wait_all();
                __syncwarp();
                for (int j0 = 0; j0 < nb_pad; j0 += 32) {
                    uint32_t r[32];
                    tmem_ld32(tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + j0, r);
                    if (j0 >= nb || rows_here == 0) continue;  // warp-uniform
                    if (lane == 0) bulk_wait_read<0>();         // the previous box has been read
                    __syncwarp();
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        *reinterpret_cast<float4*>(box + lane * 128 + ((j ^ (lane & 7)) << 4)) =
                            make_float4(__uint_as_float(r[4 * j]) * unscale, __uint_as_float(r[4 * j + 1]) * unscale,
                                        __uint_as_float(r[4 * j + 2]) * unscale, __uint_as_float(r[4 * j + 3]) * unscale);
                    fence_proxy_async();
                    __syncwarp();
                    if (lane == 0) {
                        if (run == 0) tma_store_3d(&p.tm_ws, box, n20 + j0, m0w, split, pol_ws);
                        else tma_reduce_add_3d(&p.tm_ws, box, n20 + j0, m0w, split, pol_ws);
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(tempty_l);
                ++run;
                endr = endr < kblocks ? tn_run_end(0, endr, kblocks, 1, stag) : kblocks + 1;
            }
            if (lane == 0) bulk_wait_all();
            if (kblocks == 0)
                for (int rr = 0; rr < rows_here; ++rr)
                    for (int c = lane; c < nb; c += 32) outw[int64_t(rr) * p.N2 + c] = 0.f;
        } else {
        const int hw = nb_pad / nh;  // TMEM columns per half
        int endh[2] = {tn_run_end(0, 0, kblocks, nh, stag), nh > 1 ? tn_run_end(1, 0, kblocks, nh, stag) : kblocks + 1};
        uint32_t runh[2] = {0, 0};
        while (endh[0] <= kblocks || (nh > 1 && endh[1] <= kblocks)) {
            if (kblocks == 0) break;
            const int h = (nh > 1 && endh[1] < endh[0]) ? 1 : 0;
            TN_TIMED_WAIT(w_a, mbar_wait(&tfull[h], runh[h] & 1));
            tc_fence_after();
            for (int j0 = 0; j0 < hw; j0 += 32) {
                uint32_t r[32];
                tmem_ld32(tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + h * 128 + j0, r);
                const int c0 = nh > 1 ? (j0 < 64 ? 64 * h + j0 : 128 + 64 * h + (j0 - 64)) : j0;  // tile column
                if (c0 >= nb) continue;  // warp-uniform
                if (vec && c0 + 32 <= nb) {
#pragma unroll
                    for (int q = 0; q < 32; ++q) tbuf[lane * Cfg::kEpiPitch + q] = __uint_as_float(r[q]) * unscale;
                    __syncwarp();
#pragma unroll
                    for (int rr = 0; rr < 8; ++rr) {
                        const int row = 4 * rr + (lane >> 3), c = (lane & 7) * 4;
                        const float* t = tbuf + row * Cfg::kEpiPitch + c;
                        float* o = outw + int64_t(row) * p.N2 + c0 + c;
                        if (row < rows_here) {
                            if (runh[h] == 0) st_v4_l2hint(o, t[0], t[1], t[2], t[3], pol_ws);
                            else red_add_v4_l2hint(o, t[0], t[1], t[2], t[3], pol_ws);
                        }
                    }
                    __syncwarp();
                } else if (lane < rows_here) {
                    float* o = orow + c0;
                    const int nv = min(32, nb - c0);
#pragma unroll
                    for (int q = 0; q < 32; ++q) {
                        if (q >= nv) break;
                        const float x = __uint_as_float(r[q]) * unscale;
                        if (runh[h] == 0) st_l2hint(o + q, x, pol_ws);
                        else red_add_l2hint(o + q, x, pol_ws);
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(tempty_l + h * 8);
            ++runh[h];
            endh[h] = endh[h] < kblocks ? tn_run_end(h, endh[h], kblocks, nh, stag) : kblocks + 1;
        }
        if (kblocks == 0)
            for (int rr = 0; rr < rows_here; ++rr)
                for (int c = lane; c < nb; c += 32) outw[int64_t(rr) * p.N2 + c] = 0.f;
        }
    } else {
        // ================= epilogue: drain each chunk into the fp32 partial ws[split] =================
        // Lane = output row (TMEM lane). The first chunk stores, later chunks add with fire-and-forget
        // vector reductions performed in L2 (red.global.add.v4.f32). Every partial element is owned
        // by one thread, and same-address operations of a thread stay in program order, so the sum
        // over chunks is evaluated in a fixed order (deterministic).
        const int ew = warp & 3;
        const int32_t m0w = n10 + ew * 32;  // first output row (N1 index) of this warp
        const int rows_here = max(0, min(32, p.N1 - m0w));
        const float unscale = ldexpf(1.f, -(ka + kbx));
        float* outw = p.ws + (int64_t(split) * p.N1 + m0w) * p.N2 + n20;
        float* orow = outw + int64_t(lane) * p.N2;
        const bool vec = (p.N2 & 3) == 0;  // 16-byte aligned partial rows
        const uint64_t pol_ws = l2_evict_last();  // the partials stay in L2 while operands stream past
        float* tbuf = reinterpret_cast<float*>(smem + Cfg::kEpiOff) + ew * 32 * Cfg::kEpiPitch;
        for (int chunk = 0; chunk < nchunks; ++chunk) {
            const uint32_t acc = chunk % Cfg::kAcc;
            TN_TIMED_WAIT(w_a, mbar_wait(&tfull[acc], (chunk / Cfg::kAcc) & 1));
            tc_fence_after();
            for (int c0 = 0; c0 < nb_pad; c0 += 32) {
                uint32_t r[32];
                tmem_ld32(tmem_base + acc * 256 + (static_cast<uint32_t>(ew * 32) << 16) + c0, r);
                if (c0 >= nb) continue;  // warp-uniform
                if (vec && c0 + 32 <= nb) {
                    // Transpose the warp's 32 x 32 block through shared memory so each vector
                    // reduction covers 4 row segments of 128 contiguous bytes instead of 32
                    // scattered 16-byte pieces (8x fewer L2 transactions per drain).
#pragma unroll
                    for (int q = 0; q < 32; ++q) tbuf[lane * Cfg::kEpiPitch + q] = __uint_as_float(r[q]) * unscale;
                    __syncwarp();
#pragma unroll
                    for (int rr = 0; rr < 8; ++rr) {
                        const int row = 4 * rr + (lane >> 3), c = (lane & 7) * 4;
                        const float* t = tbuf + row * Cfg::kEpiPitch + c;
                        float* o = outw + int64_t(row) * p.N2 + c0 + c;
                        if (row < rows_here) {
                            if (chunk == 0) st_v4_l2hint(o, t[0], t[1], t[2], t[3], pol_ws);
                            else red_add_v4_l2hint(o, t[0], t[1], t[2], t[3], pol_ws);
                        }
                    }
                    __syncwarp();
                } else if (lane < rows_here) {
                    float* o = orow + c0;
                    const int nv = min(32, nb - c0);
#pragma unroll
                    for (int q = 0; q < 32; ++q) {
                        if (q >= nv) break;
                        const float x = __uint_as_float(r[q]) * unscale;
                        if (chunk == 0) st_l2hint(o + q, x, pol_ws);
                        else red_add_l2hint(o + q, x, pol_ws);
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if constexpr (PAIR) mbar_arrive_cluster(tempty_l + acc * 8);
                else mbar_arrive(&tempty[acc]);
            }
        }
        if (nchunks == 0)
            for (int rr = 0; rr < rows_here; ++rr)
                for (int c = lane; c < nb; c += 32) outw[int64_t(rr) * p.N2 + c] = 0.f;
    }
#ifdef SC_TN_TRACE_BUILD
    if (p.trace && lane == 0) {  // roles: 0 converters, 1 epilogue, 2 MMA, 3 loader
        const int role = warp < Cfg::kCW ? 0 : warp < Cfg::kCW + 4 ? 1 : warp == Cfg::kMma ? 2 : 3;
        if (role != 2 || !PAIR || rank == 0) {
            atomicAdd(p.trace + 4 * role + 0, w_a);
            atomicAdd(p.trace + 4 * role + 1, w_b);
            atomicAdd(p.trace + 4 * role + 2, static_cast<unsigned long long>(clock64() - t_start));
            atomicAdd(p.trace + 4 * role + 3, 1ull);
        }
    }
#endif
    tc_fence_before();
    if constexpr (PAIR) cluster_sync();
    else __syncthreads();
    if (warp == Cfg::kMma) {
        tc_fence_after();
        tmem_dealloc_g<PAIR>(tmem_base);
    }
}

// Dual launch: rows [0, n1a) of the split sum -> C1 (all N2 columns), rows [n1a, N1) -> C2
// (columns [n2a, N2) only: the A2 x B1 block is never computed).
__global__ void tn_reduce_dual_kernel(int32_t S, int32_t N1, int32_t N2, int32_t n1a, int32_t n2a, const float* ws,
                                      float* C1, int64_t ldc1, float* C2, int64_t ldc2) {
    const int64_t total = int64_t(N1) * N2;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = i / N2, c = i % N2;
        if (r >= n1a && c < n2a) continue;
        float acc = 0.f;
        for (int32_t s = 0; s < S; ++s) acc += ws[int64_t(s) * total + i];
        if (r < n1a) C1[r * ldc1 + c] = acc;
        else C2[(r - n1a) * ldc2 + (c - n2a)] = acc;
    }
}

__global__ void tn_reduce_kernel(int32_t S, int32_t N1, int32_t N2, const float* ws, float* C, int64_t ldc) {
    const int64_t total = int64_t(N1) * N2;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
        float acc = 0.f;
        for (int32_t s = 0; s < S; ++s) acc += ws[int64_t(s) * total + i];
        C[(i / N2) * ldc + (i % N2)] = acc;
    }
}

}  // namespace tc

// ---- host side -------------------------------------------------------------------

namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        SC_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
        if (!f || q != cudaDriverEntryPointSuccess) throw CudaError("cuTensorMapEncodeTiled unavailable");
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }();
    return fn;
}
// 2D fp32 map over a row-major [rows x cols] matrix with row stride ld, box {box_c, box_r}.
void encode_2d(CUtensorMap* map, const float* base, int64_t rows, int64_t cols, int64_t ld, uint32_t box_c,
               uint32_t box_r, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
    const cuuint64_t gdim[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    const cuuint64_t gstride[1] = {static_cast<cuuint64_t>(ld) * sizeof(float)};
    const cuuint32_t box[2] = {box_c, box_r};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), gdim, gstride,
                                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
}
// 2D map over a pre-split weight image viewed as [rows x 32 fp16] (64 B rows, already
// in SW64 order, copied verbatim), box = `box_rows` rows.
void encode_img(CUtensorMap* map, const uint8_t* img, int64_t rows, uint32_t box_rows) {
    const cuuint64_t gdim[2] = {32, static_cast<cuuint64_t>(rows)};
    const cuuint64_t gstride[1] = {64};
    const cuuint32_t box[2] = {32, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<uint8_t*>(img), gdim, gstride,
                                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (image) failed (" + std::to_string(int(r)) + ")");
}
// Which NT GEMMs run on the A'-in-TMEM kernel, SC_NT_TM bit mask (default 0: none): 1 one source,
// N <= 128 (one pass; the unfused head was 0.6 ms faster on it, but the projected top layer's 48-wide
// P / Q GEMMs are 0.85 ms per epoch faster on the general kernel, profiles/r02_toggles_ab.txt); 2 one
// source, N = 256 as two passes, K <= 256 (msg, dmean: slower, profiles/r02_nt_tm_ab.txt); 4 two
// sources, N <= 128 (the composed head: 0.6 ms slower).
int nt_tm_mode() {
    static const int mode = [] {
        const char* e = std::getenv("SC_NT_TM");
        return e ? std::atoi(e) : 0;
    }();
    return mode;
}
// NT GEMMs run on CTA pairs (cta_group::2) unless SC_NT_PAIR=0.
bool nt_pair_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("SC_NT_PAIR");
        return !(e && e[0] == '0');
    }();
    return on;
}
}  // namespace

namespace {
// Weight-gradient GEMMs with more than 128 A' columns run on CTA pairs unless SC_TN_PAIR=0.
bool tn_use_pair(int32_t N1) {
    static const bool on = [] {
        const char* e = std::getenv("SC_TN_PAIR");
        return !(e && e[0] == '0');
    }();
    return on && N1 > tc::kBM;
}
}  // namespace

int32_t tn_f16x3_splits(int32_t N1, int32_t N2, int64_t M) {
    const bool pair = tn_use_pair(N1);
    const int32_t acols = pair ? 2 * tc::kBM : tc::kBM;
    const int32_t units = ((N1 + acols - 1) / acols) * ((N2 + tc::kMaxN - 1) / tc::kMaxN);
    const int32_t slots = pair ? std::max(1, num_sms() / 2) : num_sms();  // CTAs (pairs) resident at once
    int64_t s = std::max<int64_t>(1, slots / units);  // one wave of persistent-sized CTAs
    s = std::min<int64_t>(s, (M + 4095) / 4096);       // >= 4096 rows per split
    return static_cast<int32_t>(std::max<int64_t>(s, 1));
}

namespace {
// TMA drains of the A'-in-TMEM TN kernel into ws [S][N1][N2] (SC_TN_TMA_DRAIN=0: L2 reductions)
void encode_ws(tc::TnParams& p, int32_t S, int32_t N1, int32_t N2) {
    static const bool on = [] {
        const char* e = std::getenv("SC_TN_TMA_DRAIN");
        return !(e && e[0] == '0');
    }();
    p.ws_tma = 0;
    if (!on || N2 % 4 != 0 || (reinterpret_cast<uintptr_t>(p.ws) & 15) != 0) return;
    const cuuint64_t gdim[3] = {static_cast<cuuint64_t>(N2), static_cast<cuuint64_t>(N1), static_cast<cuuint64_t>(S)};
    const cuuint64_t gstride[2] = {static_cast<cuuint64_t>(N2) * sizeof(float),
                                   static_cast<cuuint64_t>(N1) * N2 * sizeof(float)};
    const cuuint32_t box[3] = {32, 32, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = encode_fn()(&p.tm_ws, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, p.ws, gdim, gstride, box, estr,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (ws) failed (" + std::to_string(int(r)) + ")");
    p.ws_tma = 1;
}

// Split-K launch of the TN kernel over p's tile list, S splits; ws holds [S][N1][N2] partials.
void tn_launch(tc::TnParams& p, bool pair, int32_t S, cudaStream_t s) {
    static const bool trace = [] {
        const char* e = std::getenv("SC_TN_TRACE");
        return e && std::atoi(e) != 0;
    }();
    static DevBuf<unsigned long long> trace_buf;
    if (trace) {
        trace_buf.ensure(16);
        SC_CUDA(cudaMemsetAsync(trace_buf.get(), 0, 16 * sizeof(unsigned long long), s));
        p.trace = trace_buf.get();
    }
    static const int split_acc = [] {
        const char* e = std::getenv("SC_TN_SPLIT");
        return e ? std::atoi(e) : 0;
    }();
    p.split_acc = split_acc;
    static const int stagger = [] {
        const char* e = std::getenv("SC_TN_STAGGER");
        return e ? std::atoi(e) : 1;
    }();
    p.stagger = stagger;
    static const int pf_dist = [] {
        const char* e = std::getenv("SC_TN_PF");
        return e ? std::atoi(e) : 0;
    }();
    p.pf_dist = pf_dist;
    const int64_t units = int64_t(S) * p.ntiles;
    auto launch = [&](auto kernel, int smem_bytes, int threads) {
        SC_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes));
        cudaLaunchConfig_t cfg{};
        cudaLaunchAttribute attr[1];
        cfg.gridDim = dim3(static_cast<unsigned>(pair ? 2 * units : units));
        cfg.blockDim = dim3(threads);
        cfg.dynamicSmemBytes = static_cast<size_t>(smem_bytes);
        cfg.stream = s;
        if (pair) {
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = 2;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
        }
        SC_CUDA(cudaLaunchKernelEx(&cfg, kernel, p));
    };
    static const bool a_tmem = [] {
        const char* e = std::getenv("SC_TN_ATMEM");
        return e ? std::atoi(e) != 0 : true;
    }();
    if (pair && a_tmem)
        launch(tc::gemm_tn_f16x3_kernel<true, true>, tc::TnCfg<true, true>::kSmem, tc::TnCfg<true, true>::kThr);
    else if (pair)
        launch(tc::gemm_tn_f16x3_kernel<true, false>, tc::TnCfg<true, false>::kSmem, tc::TnCfg<true, false>::kThr);
    else
        launch(tc::gemm_tn_f16x3_kernel<false, false>, tc::TnCfg<false, false>::kSmem, tc::TnCfg<false, false>::kThr);
    SC_LAUNCH_CHECK();
    if (trace) {  // per role: mean over warps of (wait A, wait B, total) cycles
        unsigned long long h[16];
        SC_CUDA(cudaMemcpyAsync(h, trace_buf.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
        SC_CUDA(cudaStreamSynchronize(s));
        const char* names[4] = {"conv(empty,sfull)", "epi(tfull,-)", "mma(full,tempty)", "load(sempty,-)"};
        std::fprintf(stderr, "TN trace M=%lld N1=%d N2=%d:", static_cast<long long>(p.M), p.N1, p.N2);
        for (int r = 0; r < 4; ++r) {
            const double c = h[4 * r + 3] ? double(h[4 * r + 3]) : 1.0;
            std::fprintf(stderr, " %s %.0f/%.0f of %.0f;", names[r], h[4 * r] / c, h[4 * r + 1] / c, h[4 * r + 2] / c);
        }
        std::fprintf(stderr, "\n");
    }
}

// Common TN parameters: A (N1 columns as one source), B1 | B2, M rows, S splits.
int32_t tn_fill(tc::TnParams& p, const MatT& a, const float* amax_a, const MatT& b1, const float* amax_b1,
                const MatT* b2, const float* amax_b2, int32_t N1, int64_t M, bool pair) {
    const int32_t N2 = b1.cols + (b2 ? b2->cols : 0);
    p.a = a.ptr;
    p.lda = a.ld;
    p.N1 = N1;
    p.amax_a = amax_a;
    p.amax_a2 = amax_a;
    p.n1a = N1;
    p.b[0] = tc::TnB{b1.ptr, b1.ld, b1.rows, b1.cols, amax_b1};
    encode_2d(&p.tm_a, a.ptr, M, a.cols, a.ld, 32, tc::kTnBK);
    p.tm_a2 = p.tm_a;
    encode_2d(&p.tm_b1, b1.ptr, M, b1.cols, b1.ld, 32, tc::kTnBK);
    if (b2) encode_2d(&p.tm_b2, b2->ptr, M, b2->cols, b2->ld, 32, tc::kTnBK);
    p.nb = b2 ? 2 : 1;
    if (b2) p.b[1] = tc::TnB{b2->ptr, b2->ld, b2->rows, b2->cols, amax_b2};
    p.n2a = b1.cols;
    p.N2 = N2;
    p.M = M;
    const int32_t acols = pair ? 2 * tc::kBM : tc::kBM;
    p.tiles1 = (N1 + acols - 1) / acols;
    p.tiles2 = (N2 + tc::kMaxN - 1) / tc::kMaxN;
    return N2;
}
}  // namespace

void gemm_tn_f16x3(const MatT& a, const float* amax_a, const MatT& b1, const float* amax_b1, const MatT* b2,
                   const float* amax_b2, int64_t M, float* C, int64_t ldc, float* ws, int64_t ws_floats,
                   cudaStream_t s) {
    const int32_t N1 = a.cols, N2 = b1.cols + (b2 ? b2->cols : 0);
    if (N1 <= 0 || N2 <= 0) return;
    if (M <= 0) {
        for (int32_t r = 0; r < N1; ++r) SC_CUDA(cudaMemsetAsync(C + int64_t(r) * ldc, 0, sizeof(float) * N2, s));
        return;
    }
    const bool pair = tn_use_pair(N1);
    tc::TnParams p{};
    tn_fill(p, a, amax_a, b1, amax_b1, b2, amax_b2, N1, M, pair);
    if (p.tiles1 * p.tiles2 > 8) throw std::logic_error("gemm_tn_f16x3: too many tiles");
    p.ntiles = 0;
    for (int t1 = 0; t1 < p.tiles1; ++t1)
        for (int t2 = 0; t2 < p.tiles2; ++t2) {
            p.tile_a[p.ntiles] = static_cast<int8_t>(t1);
            p.tile_b[p.ntiles] = static_cast<int8_t>(t2);
            ++p.ntiles;
        }
    const int32_t S = tn_f16x3_splits(N1, N2, M);
    if (int64_t(S) * N1 * N2 > ws_floats) throw std::logic_error("gemm_tn_f16x3: workspace too small");
    p.rows_per_split = ((M + S - 1) / S + tc::kTnBK - 1) / tc::kTnBK * tc::kTnBK;
    p.ws = ws;
    encode_ws(p, S, N1, N2);
    tn_launch(p, pair, S, s);
    tc::tn_reduce_kernel<<<grid_for(int64_t(N1) * N2, 256), 256, 0, s>>>(S, N1, N2, ws, C, ldc);
    SC_LAUNCH_CHECK();
    count_launch(2);
}

bool tn_dual_supported(const MatT& a1, const MatT& a2, const MatT& b1, const MatT& b2) {
    const int32_t tile = 2 * tc::kBM;
    return tn_use_pair(a1.cols + a2.cols) && tn_supported(a1, b1, &b2) && tn_supported(a2, b2, nullptr) &&
           a1.cols % tile == 0 && b1.cols % tc::kMaxN == 0 && (a1.cols + a2.cols + tile - 1) / tile *
           ((b1.cols + b2.cols + tc::kMaxN - 1) / tc::kMaxN) <= 8;
}

void gemm_tn_f16x3_dual(const MatT& a1, const float* amax_a1, const MatT& a2, const float* amax_a2, const MatT& b1,
                        const float* amax_b1, const MatT& b2, const float* amax_b2, int64_t M, float* C1,
                        int64_t ldc1, float* C2, int64_t ldc2, float* ws, int64_t ws_floats, cudaStream_t s) {
    if (!tn_dual_supported(a1, a2, b1, b2)) throw std::logic_error("gemm_tn_f16x3_dual: unsupported shapes");
    const int32_t N1 = a1.cols + a2.cols;
    if (M <= 0) {
        for (int32_t r = 0; r < a1.cols; ++r)
            SC_CUDA(cudaMemsetAsync(C1 + int64_t(r) * ldc1, 0, sizeof(float) * (b1.cols + b2.cols), s));
        for (int32_t r = 0; r < a2.cols; ++r) SC_CUDA(cudaMemsetAsync(C2 + int64_t(r) * ldc2, 0, sizeof(float) * b2.cols, s));
        return;
    }
    tc::TnParams p{};
    const int32_t N2 = tn_fill(p, a1, amax_a1, b1, amax_b1, &b2, amax_b2, N1, M, true);
    encode_2d(&p.tm_a2, a2.ptr, M, a2.cols, a2.ld, 32, tc::kTnBK);
    p.amax_a2 = amax_a2;
    p.n1a = a1.cols;
    p.ntiles = 0;
    const int32_t tile = 2 * tc::kBM;
    for (int t1 = 0; t1 < p.tiles1; ++t1)
        for (int t2 = 0; t2 < p.tiles2; ++t2) {
            if (t1 * tile >= p.n1a && (t2 + 1) * tc::kMaxN <= p.n2a) continue;  // A2 x B1: not needed
            p.tile_a[p.ntiles] = static_cast<int8_t>(t1);
            p.tile_b[p.ntiles] = static_cast<int8_t>(t2);
            ++p.ntiles;
        }
    // splits sized for the tiles actually computed
    const int32_t slots = std::max(1, num_sms() / 2);
    int64_t S = std::max<int64_t>(1, slots / p.ntiles);
    S = std::max<int64_t>(1, std::min<int64_t>(S, (M + 4095) / 4096));
    if (S * N1 * N2 > ws_floats) throw std::logic_error("gemm_tn_f16x3_dual: workspace too small");
    p.rows_per_split = ((M + S - 1) / S + tc::kTnBK - 1) / tc::kTnBK * tc::kTnBK;
    p.ws = ws;
    tn_launch(p, true, static_cast<int32_t>(S), s);
    tc::tn_reduce_dual_kernel<<<grid_for(int64_t(N1) * N2, 256), 256, 0, s>>>(static_cast<int32_t>(S), N1, N2, p.n1a,
                                                                             p.n2a, ws, C1, ldc1, C2, ldc2);
    SC_LAUNCH_CHECK();
    count_launch(2);
}

bool tc_supported(const MatA& a1, const MatA* a2, int32_t N) {
    // rows are fetched in whole 16 B units by bulk copies: 16 B aligned rows (ld % 4 == 0)
    // operands stream through 2D TMA (no row gathers): 16 B aligned rows
    auto ok = [](const MatA& a) {
        return !a.rows && (a.ld % 4) == 0 && (reinterpret_cast<uintptr_t>(a.ptr) % 16) == 0 && a.K >= 1 &&
               a.ld >= a.K;
    };
    return N >= 1 && N <= tc::kMaxN && ok(a1) && (!a2 || ok(*a2));
}

bool tc_out_supported(const float* C, int64_t ldc) {
    // C is written by 2D TMA stores: 16 B aligned base and rows
    return (reinterpret_cast<uintptr_t>(C) % 16) == 0 && (ldc % 4) == 0;
}

bool tn_supported(const MatT& a, const MatT& b1, const MatT* b2) {
    auto ok = [](const MatT& x) {
        return !x.rows && (x.ld % 4) == 0 && (reinterpret_cast<uintptr_t>(x.ptr) % 16) == 0 && x.ld >= x.cols;
    };
    // B' boxes are 32 columns wide and come from one source each
    return ok(a) && ok(b1) && (!b2 || (ok(*b2) && b1.cols % 32 == 0));
}

void prep_bimage(BImage& im, const MatB& b, int32_t N, int32_t K, cudaStream_t s) {
    im.N = N;
    im.K = K;
    im.n_pad = (N + 31) / 32 * 32;  // whole 32-column TMEM chunks in the epilogue
    im.kblocks = (K + tc::kNtBK - 1) / tc::kNtBK;
    im.img.ensure(static_cast<size_t>(im.kblocks) * 2 * im.n_pad * 64);
    im.bexp.ensure(1);
    im.amax.ensure(1);
    SC_CUDA(cudaMemsetAsync(im.amax.get(), 0, sizeof(float), s));
    const int64_t nk = int64_t(N) * K;
    tc::prep_b_amax_kernel<<<grid_for(nk, 256, 64), 256, 0, s>>>(b.ptr, b.ld, b.nn ? 1 : 0, N, K, im.amax.get());
    SC_LAUNCH_CHECK();
    const int64_t chunks = int64_t(im.kblocks) * im.n_pad * 4;
    tc::prep_b_split_kernel<<<grid_for(chunks, 256), 256, 0, s>>>(b.ptr, b.ld, b.nn ? 1 : 0, N, K, im.n_pad,
                                                                  im.kblocks, im.amax.get(), im.img.get(),
                                                                  im.bexp.get());
    SC_LAUNCH_CHECK();
    count_launch(2);
}


void gemm_f16x3(const MatA& a1, const float* amax1, const BImage& b1, const MatA* a2, const float* amax2,
                const BImage* b2, float* C, int64_t ldc, int64_t M, int32_t N, int epi, const float* row_scale,
                float* amax_out, cudaStream_t s, uint32_t* relu_pos, const float* mask_msg,
                const uint32_t* mask_pos) {
    if (M <= 0 || N <= 0) return;
    if (!tc_supported(a1, a2, N) || !tc_out_supported(C, ldc))
        throw std::logic_error("gemm_f16x3: unsupported operand layout");
    tc::Params p{};
    p.nsrc = a2 ? 2 : 1;
    const MatA* as[2] = {&a1, a2};
    const BImage* bs[2] = {&b1, b2};
    const float* am[2] = {amax1, amax2};
    for (int i = 0; i < p.nsrc; ++i) {
        if (bs[i]->N != N || bs[i]->K != as[i]->K) throw std::logic_error("gemm_f16x3: B image shape mismatch");
        tc::Src& S = p.src[i];
        S.a = as[i]->ptr;
        S.lda = as[i]->ld;
        S.K = as[i]->K;
        S.kblocks = bs[i]->kblocks;
        S.bimg = bs[i]->img.get();
        S.amax_a = am[i];
        S.bexp = bs[i]->bexp.get();
        encode_2d(&S.tmap, S.a, M, S.K, S.lda, tc::kNtBK, tc::kBM);
    }
    encode_2d(&p.tmap_c, C, M, N, ldc, 32, 32);
    p.M = M;
    p.N = N;
    p.n_pad = b1.n_pad;
    p.C = C;
    p.ldc = ldc;
    p.epi = epi;
    p.row_scale = row_scale;
    p.amax_out = amax_out;
    p.relu_pos = epi == kEpiRelu ? relu_pos : nullptr;
    p.mask_msg = mask_msg;
    p.mask_pos = mask_pos;
    if (epi == kEpiMask && !mask_msg && !mask_pos) throw std::logic_error("gemm_f16x3: mask epilogue without a mask");
    static const bool trace = [] {
        const char* e = std::getenv("SC_TN_TRACE");
        return e && std::atoi(e) != 0;
    }();
    static DevBuf<unsigned long long> trace_buf;
    if (trace) {
        trace_buf.ensure(16);
        SC_CUDA(cudaMemsetAsync(trace_buf.get(), 0, 16 * sizeof(unsigned long long), s));
        p.trace = trace_buf.get();
    }
    static const int nt_pf = [] {
        const char* e = std::getenv("SC_NT_PF");
        return e ? std::atoi(e) : 0;
    }();
    p.prefetch = nt_pf;
    const bool pair = nt_pair_enabled();
    // single source, K <= 256: the A'-in-TMEM kernel with the weight image resident in shared memory
    // one pass (N <= 128): A' streams through an 8-stage TMEM ring, both sources, the weight images
    // resident in shared memory if they fit; two passes (N = 256, SC_NT_TM=2): one source, K <= 256.
    const int tm_mode = nt_tm_mode();
    const int kb_all = b1.kblocks + (p.nsrc > 1 ? bs[1]->kblocks : 0);
    const bool tm1 = (tm_mode & (p.nsrc == 1 ? 1 : 4)) && b1.n_pad <= tc::kBM &&
                     int64_t(kb_all) * b1.n_pad * 64 <= tc::NtTmCfg::kBBytes;
    const bool tm2 = (tm_mode & 2) && p.nsrc == 1 && b1.kblocks <= tc::NtTmCfg::kMaxKb && b1.n_pad % 64 == 0;
    const bool tm = pair && (tm1 || tm2) && epi != kEpiMask;  // (the A'-in-TMEM epilogue has no mask)
    if (tm) {
        const int np = b1.n_pad > tc::kBM ? 2 : 1;
        for (int i = 0; i < p.nsrc; ++i)
            encode_img(&p.src[i].tmap_b, bs[i]->img.get(), int64_t(bs[i]->kblocks) * 2 * bs[i]->n_pad,
                       bs[i]->n_pad / np / 2);
    } else if (pair) {
        for (int i = 0; i < p.nsrc; ++i)
            encode_img(&p.src[i].tmap_b, bs[i]->img.get(), int64_t(bs[i]->kblocks) * 2 * bs[i]->n_pad, bs[i]->n_pad / 2);
    }
    const int64_t rows_per_tile = pair ? 2 * tc::kBM : tc::kBM;
    p.tiles = (M + rows_per_tile - 1) / rows_per_tile;
    auto launch = [&](auto kernel, int smem_bytes) {
        SC_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes));
        cudaLaunchConfig_t cfg{};
        cudaLaunchAttribute attr[1];
        cfg.blockDim = dim3(tm ? tc::NtTmCfg::kThr : pair ? tc::NtCfg<true>::kThr : tc::NtCfg<false>::kThr);
        cfg.dynamicSmemBytes = static_cast<size_t>(smem_bytes);
        cfg.stream = s;
        if (pair) {
            const int64_t pairs = std::min<int64_t>(p.tiles, std::max(1, num_sms() / 2));
            cfg.gridDim = dim3(static_cast<unsigned>(2 * pairs));
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = 2;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
        } else {
            cfg.gridDim = dim3(static_cast<unsigned>(std::min<int64_t>(p.tiles, num_sms())));
        }
        SC_CUDA(cudaLaunchKernelEx(&cfg, kernel, p));
    };
    auto dispatch = [&](auto epi_tag, auto amax_tag) {
        constexpr int E = decltype(epi_tag)::value;
        constexpr bool A = decltype(amax_tag)::value;
        if (tm) launch(tc::gemm_nt_tm_kernel<E, A>, tc::NtTmCfg::kSmem);
        else if (pair) launch(tc::gemm_f16x3_kernel<E, A, true>, tc::NtCfg<true>::kSmem);
        else launch(tc::gemm_f16x3_kernel<E, A, false>, tc::NtCfg<false>::kSmem);
    };
    using T = std::true_type;
    using F = std::false_type;
    const bool amax = amax_out != nullptr;
    switch (epi) {
        case kEpiNone:
            amax ? dispatch(std::integral_constant<int, kEpiNone>{}, T{})
                 : dispatch(std::integral_constant<int, kEpiNone>{}, F{});
            break;
        case kEpiRelu:
            amax ? dispatch(std::integral_constant<int, kEpiRelu>{}, T{})
                 : dispatch(std::integral_constant<int, kEpiRelu>{}, F{});
            break;
        case kEpiRowScale:
            amax ? dispatch(std::integral_constant<int, kEpiRowScale>{}, T{})
                 : dispatch(std::integral_constant<int, kEpiRowScale>{}, F{});
            break;
        case kEpiMask:
            amax ? dispatch(std::integral_constant<int, kEpiMask>{}, T{})
                 : dispatch(std::integral_constant<int, kEpiMask>{}, F{});
            break;
        default: throw std::logic_error("gemm_f16x3: bad epilogue");
    }
    SC_LAUNCH_CHECK();
    count_launch();
    if (trace) {
        unsigned long long h[16];
        SC_CUDA(cudaMemcpyAsync(h, trace_buf.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
        SC_CUDA(cudaStreamSynchronize(s));
        const char* names[4] = {"conv(empty,sfull)", "epi(tfull,boxwait)", "mma(full,tempty)", "load(sempty,-)"};
        std::fprintf(stderr, "NT trace M=%lld N=%d K=%d+%d:", static_cast<long long>(M), N, a1.K, a2 ? a2->K : 0);
        for (int r = 0; r < 4; ++r) {
            const double c = h[4 * r + 3] ? double(h[4 * r + 3]) : 1.0;
            std::fprintf(stderr, " %s %.0f/%.0f of %.0f;", names[r], h[4 * r] / c, h[4 * r + 1] / c, h[4 * r + 2] / c);
        }
        std::fprintf(stderr, "\n");
    }
}

void TcGemm::init(sc_trainer* t) {
    enabled = t->gemm_mode == 0;
    // One launch for a layer's dU and dW measured ~1 % slower than two (profiles/r02_tn_ab.txt): opt-in.
    const char* e = std::getenv("SC_TN_DUAL");
    dual = e && e[0] == '1';
}

const BImage& TcGemm::image(const MatB& b, int32_t N, int32_t K, cudaStream_t s) {
    const Key key{b.ptr, b.ld, b.nn, N, K};
    auto& e = cache[key];
    if (e.version != version) {
        prep_bimage(e.im, b, N, K, s);
        e.version = version;
    }
    return e.im;
}

void TcGemm::nt(sc_trainer* t, const MatA& a1, const float* amax1, const MatB& b1, const MatA* a2,
                const float* amax2, const MatB* b2, float* C, int64_t ldc, int64_t M, int32_t N, int epi,
                const float* row_scale, float* amax_out, uint32_t* relu_pos, const float* mask_msg,
                const uint32_t* mask_pos) {
    cudaStream_t s = t->ctx->stream;
    if (enabled && tc_supported(a1, a2, N) && tc_out_supported(C, ldc)) {
        const BImage& i1 = image(b1, N, a1.K, s);
        const BImage* i2 = a2 ? &image(*b2, N, a2->K, s) : nullptr;
        gemm_f16x3(a1, amax1, i1, a2, amax2, i2, C, ldc, M, N, epi, row_scale, amax_out, s, relu_pos, mask_msg,
                   mask_pos);
    } else {
        if (enabled) ++simt_fallbacks;
        gemm_nt(a1, b1, a2, b2, C, ldc, M, N, epi, row_scale, s, amax_out, mask_msg, mask_pos);
        if (epi == kEpiRelu && relu_pos) relu_sign_bits(M, N, C, ldc, relu_pos, s);
    }
}

bool TcGemm::tn_dual(sc_trainer* t, const MatT& a1, const float* amax_a1, const MatT& a2, const float* amax_a2,
                     const MatT& b1, const float* amax_b1, const MatT& b2, const float* amax_b2, int64_t M, float* C1,
                     int64_t ldc1, float* C2, int64_t ldc2) {
    if (!dual || !enabled || !tn_dual_supported(a1, a2, b1, b2)) return false;
    gemm_tn_f16x3_dual(a1, amax_a1, a2, amax_a2, b1, amax_b1, b2, amax_b2, M, C1, ldc1, C2, ldc2, t->ws.get(),
                       t->ws_floats, t->ctx->stream);
    return true;
}

void TcGemm::tn(sc_trainer* t, const MatT& a, const float* amax_a, const MatT& b1, const float* amax_b1,
                const MatT* b2, const float* amax_b2, int64_t M, float* C, int64_t ldc, cudaStream_t s, float* ws) {
    if (!s) s = t->ctx->stream;
    if (!ws) ws = t->ws.get();
    if (enabled && tn_supported(a, b1, b2))
        gemm_tn_f16x3(a, amax_a, b1, amax_b1, b2, amax_b2, M, C, ldc, ws, t->ws_floats, s);
    else {
        if (enabled) ++simt_fallbacks;
        gemm_tn(a, b1, b2, M, C, ldc, ws, t->ws_floats, s);
    }
}

}  // namespace sc
