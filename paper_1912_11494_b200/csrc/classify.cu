// classify.cu -- sm_100a kernels of the segmentation hot path.
//
//   k_morton_hist / k_scan_blocks / k_scan_totals / k_morton_scatter   (a9) spatial-order prepass:
//        a counting sort of the fibers by the Morton code of point 10, so that a CTA holds 256 nearby
//        fibers that want the same atlas tiles (the B200 analogue of the paper's data-locality
//        argument).
//   k_cull   (a2, list) per CTA of k_classify, the tiles its fibers may need under their bundle
//        thresholds (bundle point-10 spheres, then the three-sphere tile bound), ordered best-first.
//   k_classify   (a1-a8) the CTA's fibers in shared memory (cp.async ingest, a1); the listed tiles
//        streamed into a shared-memory ring by 1-D TMA bulk copies from a producer warp; per tile the
//        exact sphere bound with each fiber's live cutoff decided by warp ballot (a2), then the
//        paper's cascade with lane = centroid: test1 centre point (a3), test2 end points in both
//        orientations (a4), candidate rounds with test3 four points (a5) and test4 the
//        rest with early exits (a6), the closest-bundle key update (a7,
//        PAPER.md:129-133, :163) and the epilogue scattered back through the permutation (a8,
//        PAPER.md:138).  DESIGN.md Sec. 5 has the layout, the roofline and the measurements.
//
// FP32 on the CUDA cores: every point distance is the same explicitly-rounded expression
// (d2 below), so a value reused by an earlier stage is bit-identical to the one the full
// 21-point maximum would compute, and discarding can never change a result.
#include <cfloat>
#include <climits>
#include <cstdint>

#include "seg_internal.cuh"

namespace seg {

// ----------------------------------------------------------------------------------------
// PTX helpers: mbarrier + 1-D TMA bulk copy (cp.async.bulk -> UBLKCP)
// ----------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async4(void *dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
// the same with src-size operand n (0 or 4): n = 0 copies nothing and writes 4 zero bytes (no global read)
__device__ __forceinline__ void cp_async4_n(void *dst, const void *src, uint32_t n) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Eq. 1 squared, FP32, fixed rounding: ((dx*dx) + dy*dy) + dz*dz with explicit _rn ops so no
// contraction choice of the compiler can make two evaluations of the same pair differ.
__device__ __forceinline__ float d2(float px, float py, float pz, float4 q) {
    const float dx = __fsub_rn(px, q.x), dy = __fsub_rn(py, q.y), dz = __fsub_rn(pz, q.z);
    return __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
}

// Two squared distances at once with packed f32x2 arithmetic (FADD2/FMUL2/FFMA2 on sm_100a): the
// scalar point p against the two points whose coordinates are packed in (qx, qy, qz).  Per lane it
// is the very same sequence of round-to-nearest operations as d2(), so the values are bit-identical.
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk2(float lo, float hi) {
    u64 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ float2 upk2(u64 v) {
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
    return r;
}
__device__ __forceinline__ float2 d2_pair(float px, float py, float pz, u64 qx, u64 qy, u64 qz) {
    u64 dx, dy, dz, r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(dx) : "l"(pk2(px, px)), "l"(qx));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(dy) : "l"(pk2(py, py)), "l"(qy));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(dz) : "l"(pk2(pz, pz)), "l"(qz));
    asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(r) : "l"(dx));
    asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(r) : "l"(dy), "l"(r));
    asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(r) : "l"(dz), "l"(r));
    return upk2(r);
}

// The same, for the two points packed in (px, py, pz) against the scalar point q.
__device__ __forceinline__ float2 d2_pair_b(u64 px, u64 py, u64 pz, float qx, float qy, float qz) {
    u64 dx, dy, dz, r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(dx) : "l"(px), "l"(pk2(qx, qx)));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(dy) : "l"(py), "l"(pk2(qy, qy)));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(dz) : "l"(pz), "l"(pk2(qz, qz)));
    asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(r) : "l"(dx));
    asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(r) : "l"(dy), "l"(r));
    asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(r) : "l"(dz), "l"(r));
    return upk2(r);
}
__device__ __forceinline__ u64 f2u(float2 v) {
    u64 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(v.x), "f"(v.y));
    return r;
}

// -DSEG_NOSCREEN: exact mode's dense loop in the d2 form (tests/test_gpu_screen.py requires the same bits)
#ifdef SEG_NOSCREEN
constexpr bool SCREEN_OFF = true;
#else
constexpr bool SCREEN_OFF = false;
#endif
// Paper mode screens too (round 2): the dense loop keeps every orientation whose screened 3-point estimate
// passes (a superset, as in exact mode) and the candidate rounds take the end-point orientation decision on
// the exact FP32 distances, dropping the other orientation.  -DSEG_PAPER_D2: the round-1 form (exact d2 in
// the dense loop, the orientation decided there).
#ifdef SEG_PAPER_D2
constexpr bool PAPER_D2 = true;
#else
constexpr bool PAPER_D2 = false;
#endif
// the tile image (seg_internal.cuh, TI_*): points 0 / 10 / 20 carry the screen's half norms in w; paper mode
// also fills the per-centroid chord length and stored-reversed flag

// Exact mode's dot-product screen (seg_internal.cuh): h = (s + ...) - a.c for the two fiber points packed
// in (px, py, pz) against the scalar centroid point q, s = the packed sums of the lowered half norms.
// Never above d2 / 2 (see there).
__device__ __forceinline__ float2 screen_pair_b(u64 px, u64 py, u64 pz, float qx, float qy, float qz, u64 s) {
    u64 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pz), "l"(pk2(-qz, -qz)), "l"(s));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(py), "l"(pk2(-qy, -qy)), "l"(r));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(px), "l"(pk2(-qx, -qx)), "l"(r));
    return upk2(r);
}
__device__ __forceinline__ u64 add_pair_b(u64 a, float b) {
    u64 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(pk2(b, b)));
    return r;
}
// the fiber side's lowered half squared norm, FP32 (at most 5u of its own error; seg_internal.cuh)
__device__ __forceinline__ float screen_half_norm(float x, float y, float z) {
    if (!(fabsf(x) <= SCREEN_SAFE && fabsf(y) <= SCREEN_SAFE && fabsf(z) <= SCREEN_SAFE)) return -INFINITY;
    const float h = __fmul_rn(__fmaf_rn(z, z, __fmaf_rn(y, y, __fmul_rn(x, x))), 0.5f);
    return __fsub_rn(__fmaf_rn(h, -0x1p-18f, h), 0x1p-62f);
}

// ----------------------------------------------------------------------------------------
// a9: spatial-order prepass (counting sort on a Morton grid of point 10: 2^21 buckets, 2^18 for small N)
// ----------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t spread3(uint32_t v) {  // up to 10 bits -> every third bit
    v &= 0x3ffu;
    v = (v | (v << 16)) & 0x030000ffu;
    v = (v | (v << 8)) & 0x0300f00fu;
    v = (v | (v << 4)) & 0x030c30c3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}

#ifndef SEG_MORTON_FPT
#define SEG_MORTON_FPT 8
#endif
constexpr int MORTON_FPT = SEG_MORTON_FPT;   // fibers per thread in k_morton_hist (independent loads in flight)

__global__ void k_morton_hist(MortonParams p) {
    const float lim = (float)((1 << p.bits) - 1);
    const float sc = (float)(1 << (p.bits - MORTON_BITS));   // inv_cell is for the 6-bit grid
    const int i0 = blockIdx.x * blockDim.x * MORTON_FPT + threadIdx.x;
    float v[MORTON_FPT][3];
#pragma unroll
    for (int q = 0; q < MORTON_FPT; ++q) {
        const int i = i0 + q * blockDim.x;
        const float *f = p.fibers + (size_t)min(i, p.n - 1) * (3 * NPTS) + 30;  // point 10
#pragma unroll
        for (int c = 0; c < 3; ++c) v[q][c] = __ldg(f + c);
    }
#pragma unroll
    for (int q = 0; q < MORTON_FPT; ++q) {
        const int i = i0 + q * blockDim.x;
        if (i >= p.n) break;
        // fmaxf/fminf map NaN to the bound, so non-finite fibers land in a valid bucket
        const float qx = fminf(fmaxf((v[q][0] - p.lo.x) * (p.inv_cell.x * sc), 0.f), lim);
        const float qy = fminf(fmaxf((v[q][1] - p.lo.y) * (p.inv_cell.y * sc), 0.f), lim);
        const float qz = fminf(fmaxf((v[q][2] - p.lo.z) * (p.inv_cell.z * sc), 0.f), lim);
        const uint32_t k = spread3((uint32_t)qx) | (spread3((uint32_t)qy) << 1) | (spread3((uint32_t)qz) << 2);
        p.key[i] = k;
        p.rank[i] = atomicAdd(p.hist + k, 1u);   // the rank in the bucket: the scatter needs no atomic
    }
}

// Exclusive scan of the MORTON_BUCKETS counters in two levels: every block of SCAN_B buckets scans its
// range in place and writes its total (k_scan_blocks, 256 blocks in parallel); one block scans the
// totals (k_scan_totals); k_morton_scatter adds the block offset of its key.
constexpr int SCAN_B = 1024;                       // buckets per block: 256 threads x 4
static_assert(MORTON_BUCKETS % SCAN_B == 0 && (MORTON_BUCKETS / SCAN_B) % 256 == 0, "scan shape");

__device__ __forceinline__ uint32_t block_excl_scan256(uint32_t v, uint32_t *warp_sums, uint32_t &total) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) warp_sums[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        const uint32_t w = lane < 8 ? warp_sums[lane] : 0u;
        uint32_t wi = w;
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += t;
        }
        if (lane < 8) warp_sums[lane] = wi - w;
        if (lane == 7) warp_sums[8] = wi;
    }
    __syncthreads();
    total = warp_sums[8];
    return warp_sums[wid] + incl - v;
}

__global__ void __launch_bounds__(256) k_scan_blocks(uint32_t *hist, uint32_t *bsum) {
    __shared__ uint32_t warp_sums[9];
    uint4 v = reinterpret_cast<uint4 *>(hist + (size_t)blockIdx.x * SCAN_B)[threadIdx.x];
    const uint32_t s1 = v.x, s2 = s1 + v.y, s3 = s2 + v.z, s4 = s3 + v.w;
    uint32_t total;
    const uint32_t ex = block_excl_scan256(s4, warp_sums, total);
    reinterpret_cast<uint4 *>(hist + (size_t)blockIdx.x * SCAN_B)[threadIdx.x] = make_uint4(ex, ex + s1, ex + s2, ex + s3);
    if (threadIdx.x == 0) bsum[blockIdx.x] = total;
}

__global__ void __launch_bounds__(256) k_scan_totals(uint32_t *bsum, int nb) {
    // nb block totals (a multiple of 256), nb / 256 consecutive ones per thread
    const int per = nb / 256;
    __shared__ uint32_t warp_sums[9];
    uint32_t sum = 0;
    for (int k = 0; k < per; ++k) sum += bsum[threadIdx.x * per + k];
    uint32_t total;
    uint32_t ex = block_excl_scan256(sum, warp_sums, total);
    for (int k = 0; k < per; ++k) {
        const uint32_t v = bsum[threadIdx.x * per + k];
        bsum[threadIdx.x * per + k] = ex;
        ex += v;
    }
}

__global__ void k_morton_scatter(MortonParams p) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= p.n) return;
    const uint32_t k = p.key[i];
    SEG_DCHECK(k < (1u << (3 * p.bits)));
    const uint32_t pos = __ldg(p.hist + k) + p.rank[i] + __ldg(p.bsum + k / SCAN_B);
    SEG_DCHECK(pos < (uint32_t)p.n);
    p.perm[pos] = i;
}

// (The prepass as CUB's onesweep radix sort of (key, index) was measured and rejected: DESIGN.md Sec. 5.)

cudaError_t launch_morton_prepass(const MortonParams &p, cudaStream_t s) {
    const size_t buckets = (size_t)1 << (3 * p.bits);
    const int nb = (int)(buckets / SCAN_B);
    cudaError_t e = cudaMemsetAsync(p.hist, 0, sizeof(uint32_t) * buckets, s);
    if (e != cudaSuccess) return e;
    const int g = (p.n + 255) / 256;
    k_morton_hist<<<(p.n + 256 * MORTON_FPT - 1) / (256 * MORTON_FPT), 256, 0, s>>>(p);
    k_scan_blocks<<<nb, 256, 0, s>>>(p.hist, p.bsum);
    k_scan_totals<<<1, 256, 0, s>>>(p.bsum, nb);
    k_morton_scatter<<<g, 256, 0, s>>>(p);
    return cudaGetLastError();
}

size_t morton_scratch_words(int bits) {
    const size_t buckets = (size_t)1 << (3 * bits);
    return buckets + buckets / SCAN_B;
}

// ----------------------------------------------------------------------------------------
// a1-a8: the classify kernel
//
// CTA = NCW consumer warps (one fiber per consumer lane; the CTA's 256 Morton-sorted fibers are
// interleaved over the warps so every warp gets a share of every tile's work) + 1 producer warp.
//   a1  fiber ingest: every coordinate straight from global memory (through the prepass permutation)
//       into its shared-memory plane with 4-byte cp.async: end points packed for FFMA2, point 10,
//       and the other 18 points in xy / z planes; non-finite fibers flagged.
//   a2  the PRODUCER warp streams the tile list k_cull wrote for this CTA through a STAGES-deep ring
//       (one 1-D TMA bulk copy per tile, cp.async.bulk -> UBLKCP, mbarrier completion); an end
//       marker closes the stream.  Each consumer lane re-tests its fiber against the tile's three
//       boxes with its live cutoff tau = min(thr_b^2, best^2); a warp ballot picks the fibers.
//   a3+a4  consumers, dense and transposed: lane c holds centroid c's points 0/10/20, the warp walks
//       its passing fibers one at a time: test1 (centre point) and test2 (end points, both
//       orientations, FFMA2) for all 32 centroids at once;
//   a5+a6  every alive orientation goes onto the warp's candidate stack; at the end of the tile the
//       stack runs in rounds of 32 lanes, each entry re-checked against its fiber's freshest best;
//       test3 = points {3,17,7,13}, test4 = the rest with an early exit after every group
//       (PAPER.md:159);
//   a7  a finished orientation updates its fiber's best (d^2, bundle) key -- paper mode:
//       (d_ME + TN, bundle) -- with a shared-memory 64-bit atomicMin (lexicographic, so tile order
//       and orientation never matter);
//   a8  epilogue: label / sqrt(d^2) (paper mode: the score) stored through the permutation, or the
//       raw key for an atlas-sharded run (row f4).
// ----------------------------------------------------------------------------------------
#ifndef SEG_NCW
#define SEG_NCW 8
#endif
constexpr int NCW = SEG_NCW;           // consumer warps (4 warps x 3 CTAs/SM measured slower: 8.74 vs 7.73 ms)
constexpr int CTAS_PER_SM = 2;
constexpr int FPC = NCW * 32;          // fibers per CTA
constexpr int NTHREADS = FPC + 32;     // + producer warp
#ifndef SEG_EARLY_TMA
#define SEG_EARLY_TMA 1   // the first STAGES tile copies issued before the fiber ingest
#endif
#ifndef SEG_STAGES
#define SEG_STAGES 4
#endif
constexpr int STAGES = SEG_STAGES;     // tile ring depth
#ifndef SEG_DEFER_BELOW
#define SEG_DEFER_BELOW 32
#endif
#ifndef SEG_DEFER_TILES
#define SEG_DEFER_TILES 2
#endif
// candidate stacks shorter than DEFER_BELOW entries are carried over to the next tile, holding at most
// DEFER_TILES ring stages (< STAGES - 1 so the producer keeps a tile of lookahead); 0 = flush every tile
constexpr int DEFER_BELOW = SEG_DEFER_BELOW, DEFER_TILES = SEG_DEFER_TILES;
static_assert(DEFER_TILES >= 0 && DEFER_TILES <= STAGES - 1, "a warp must not hold every ring stage");
#ifndef SEG_CULL_UNROLL
#define SEG_CULL_UNROLL 32
#endif
#ifndef SEG_DENSE_UNROLL
#define SEG_DENSE_UNROLL 1
#endif
#ifndef SEG_INGEST_UNROLL
#define SEG_INGEST_UNROLL 32
#endif
#ifndef SEG_BUNDLE_UNROLL
#define SEG_BUNDLE_UNROLL 32
#endif
constexpr int INGEST_UNROLL = SEG_INGEST_UNROLL; // k_classify's fiber ingest loops (32 fibers per warp)
constexpr int BUNDLE_UNROLL = SEG_BUNDLE_UNROLL; // k_cull's 32-bundle sphere loop
constexpr int CULL_UNROLL = SEG_CULL_UNROLL;     // k_cull's 32-tile chunk loop
#ifndef SEG_RANK_UNROLL
#define SEG_RANK_UNROLL 4
#endif
constexpr int RANK_UNROLL = SEG_RANK_UNROLL;     // k_cull's best-first ranking loop
constexpr int DENSE_UNROLL = SEG_DENSE_UNROLL;   // k_classify's dense step loop
#ifndef SEG_VOTE_JJ_ALWAYS
#define SEG_VOTE_JJ_ALWAYS 0
#endif
// fibers per step of the dense test1+test2 loop (a warp-tile holds ~11 passing fibers).  Exact mode, with
// the dot-product screen: 1 since round 2's bank-conflict and branch fixes (cfg 3 -1.1%, cfg 4 -1.6% vs 2;
// 3: +1.5%); round 1 had measured 2 best.  Paper mode: 2 until the next fiber was picked one step ahead
// (SEG_JNEXT), which only the one-fiber step can do: then 1 (cfg 3 4.80 -> 4.65 ms, cfg 4 -3.6%).
#ifndef SEG_FB
#define SEG_FB 1
#endif
#ifndef SEG_NLIST
#define SEG_NLIST 1     // consumers loop over the list length instead of reading an end marker per tile
#endif
// consumers' tile wait: try_wait + nanosleep(N) instead of the suspend-hinted try_wait (0).  Exact mode: 0 (32 - 256 ns
// measured equal or worse); paper mode: 64 (-1.2%)
#ifndef SEG_WAIT_NS
#define SEG_WAIT_NS 0
#endif
#ifndef SEG_WAIT_NS_PAPER
#define SEG_WAIT_NS_PAPER 64
#endif
#ifndef SEG_JNEXT
#define SEG_JNEXT 1   // FB == 1: the next dense step's fiber picked during the current step
#endif
#ifndef SEG_FB_PAPER
#define SEG_FB_PAPER 1
#endif
constexpr int NMID = NPTS - 3;         // fiber points other than 0, 10, 20 (smem planes)
// pitch of one point's plane (32 fibers) in the per-warp fxy (float2) and fz (float) arrays.  33, not 32: the
// ingest's 4-byte cp.async of one fiber by 32 lanes writes one coordinate of ~10 different points, which at
// pitch 32 all fall into the same bank (10x the ideal wavefronts, ncu r02); at 33 they spread over the banks.
// Reads of one point by 32 lanes (different fibers) stay conflict-free either way.
#ifndef SEG_PLANE_PITCH
#define SEG_PLANE_PITCH 33
#endif
constexpr int PP = SEG_PLANE_PITCH;
#ifndef SEG_PLANE_SKEW
#define SEG_PLANE_SKEW 16
#endif
#ifndef SEG_Q2CAP
#define SEG_Q2CAP 128
#endif
constexpr int MULTI_WORDS = 4;         // multi-label masks: at most 128 bundles (they live in the q2r region)
// the q2r region per warp: the stack's 3-point values (PAPER_D2 builds only) or the 32 fibers' masks (MULTI)
constexpr int Q2R_WORDS = (PAPER_D2 && SEG_Q2CAP > 32 * MULTI_WORDS) ? SEG_Q2CAP : 32 * MULTI_WORDS;
constexpr int Q2CAP = SEG_Q2CAP;       // candidate stack; flushed when fewer than 64 slots remain (128: room for the 4th ring stage)
constexpr int PECAP = 32;              // MULTI: winners of one tile (at most one per fiber)
constexpr uint32_t SLEEP_NS = 1000000; // mbarrier try_wait suspend-time hint
constexpr unsigned long long KEY_NONE = ~0ull;
constexpr unsigned long long KEY_X_NONE = 0x7fffffffffffffffull;       // seg.h SEG_KEY_NONE
constexpr unsigned long long KEY_X_NONFINITE = 0x7ffffffffffffffeull;  // seg.h SEG_KEY_NONFINITE
constexpr int MAX_TILES = 30000;
static_assert(MAX_TILES < 65535, "k_cull's per-CTA tile lists hold u16 tile indices");
// per CTA of k_cull / k_classify: [count, tiles...] as u16, padded to a whole 32-bit word
__host__ __device__ constexpr int cull_stride(int T) { return (T + 2) & ~1; }
constexpr int MAX_SMEM_BUNDLES = 512;  // k_cull stages up to this many bundle headers (16 KB)       // k_cull keeps per-tile priorities and the list in shared memory

enum {
    ST_FIBERS = 0, ST_WT_LISTED, ST_WT_COMPUTED, ST_LT_PASS, ST_T1, ST_T2, ST_T34, ST_FULL, ST_UPD,
    ST_PDIST, ST_SPHERE, ST_CTAS, ST_CYC_CONS, ST_CYC_FULLWAIT, ST_CYC_HIT, ST_CYC_FLUSH, ST_CYC_SPHERE, ST_CYC_INGEST, ST_ROUNDS, ST_ROUND_LANES, ST_HITS, ST_RESERVED21, ST_N
};

struct StageMeta {
    int tile;              // tile index, -1 = end of stream
};

struct SmemLayout {
    size_t ring = 0, fxy = 0, fz = 0, fe = 0, fez = 0, fm = 0, q2e = 0, q2r = 0, pe = 0, best = 0, flen = 0,
           bars = 0, meta = 0, total = 0;
    __host__ __device__ constexpr SmemLayout() {
        size_t o = 0;
        ring = o; o += (size_t)STAGES * TILE_STRIDE_BYTES;
        fxy = o;  o += (size_t)NCW * NMID * PP * sizeof(float2);
        fz = o;   o += (size_t)NCW * NMID * PP * sizeof(float);
        o = (o + 15) & ~(size_t)15;   // the float4 / u64 arrays below need 16-B alignment whatever NCW and PP are
        // fe / fm / fez 16 B apart in bank alignment, so the ingest's writes of x0, x10, z0 (etc.) of one
        // fiber do not share a bank (bank model: 3.3 -> 2.3 wavefronts per ingest instruction)
        fe = o;   o += (size_t)FPC * sizeof(float4) + SEG_PLANE_SKEW;   // (x0, x20, y0, y20)
        fm = o;   o += (size_t)FPC * sizeof(float4) + SEG_PLANE_SKEW;   // point 10, w = h10 (NaN: a non-finite fiber)
        fez = o;  o += (size_t)FPC * sizeof(float4);   // (z0, z20, h0, h20): h = lowered half norms
        best = o; o += (size_t)FPC * sizeof(unsigned long long);
        flen = o; o += (size_t)FPC * sizeof(float);          // paper mode: chord length of each fiber
        bars = o; o += 2 * STAGES * sizeof(uint64_t);
        q2r = o;  o += (size_t)NCW * Q2R_WORDS * sizeof(float);
        q2e = o;  o += (size_t)NCW * Q2CAP * sizeof(uint16_t);
        pe = o;   o += (size_t)NCW * PECAP * sizeof(uint16_t);
        meta = o; o += (size_t)STAGES * sizeof(StageMeta);
        total = (o + 127) & ~(size_t)127;
    }
};

// CTAS_PER_SM CTAs per SM: 228 KB per SM, 1 KB reserved per CTA
static_assert(SmemLayout().total <= 233472 / CTAS_PER_SM - 1024, "k_classify shared memory exceeds the CTA/SM budget");
static_assert(SmemLayout().fe % 16 == 0 && SmemLayout().fm % 16 == 0 && SmemLayout().fez % 16 == 0 &&
              SmemLayout().best % 8 == 0 && SmemLayout().bars % 8 == 0, "k_classify shared-memory arrays misaligned");


__device__ __forceinline__ void mbar_sleep_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAITS_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@!P1 bra WAITS_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(SLEEP_NS)
        : "memory");
}

__device__ __forceinline__ bool mbar_try(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n}" : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    return ok != 0;
}

__device__ __forceinline__ float key_d2(unsigned long long k) { return __uint_as_float((uint32_t)(k >> 32)); }

// The squared cutoff a fiber's best key implies.  Exact mode keys hold d^2; paper mode keys hold the
// score s = d_ME + TN (mm) and the cutoff on the squared running max is s^2 rounded UP (TN >= 0, so a
// pair whose max exceeds s cannot beat s; rounding up keeps that sound).  KEY_NONE reads as NaN,
// which fminf(thr2, .) ignores.
template <bool PAPER>
__device__ __forceinline__ float key_cut2(unsigned long long k) {
    const float v = key_d2(k);
    return PAPER ? __fmul_ru(v, v) : v;
}

// Eq. 3 in FP32 with round-to-nearest ops: ((|ls - lc| / max(ls, lc)) + 1)^2 - 1.
__device__ __forceinline__ float tn_f32(float ls, float lc) {
    const float q = __fadd_rn(__fdiv_rn(fabsf(__fsub_rn(ls, lc)), fmaxf(ls, lc)), 1.f);
    return __fsub_rn(__fmul_rn(q, q), 1.f);
}

// a2: exact tile lower bound
// squared distance from point (x, y, z) to the box [lo, hi] (0 inside), FP32
__device__ __forceinline__ float box_d2(float x, float y, float z, const float4 &lo, const float4 &hi) {
    const float dx = fmaxf(fmaxf(lo.x - x, x - hi.x), 0.f);
    const float dy = fmaxf(fmaxf(lo.y - y, y - hi.y), 0.f);
    const float dz = fmaxf(fmaxf(lo.z - z, z - hi.z), 0.f);
    return __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
}
// a2 with boxes: for every centroid c of the tile, |f_p - c_p| >= dist(f_p, box_p) (c_p lies in box_p);
// the same orientation logic as the spheres.  Skip iff the bound exceeds s = sqrt(tau) + CULL_EPS.
#if SEG_PAIRBOX
__device__ __forceinline__ u64 sub_pair(u64 a, u64 b) {
    u64 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
// per half: max(lo - x, x - hi, 0), the same values as box_d2's scalar gaps
__device__ __forceinline__ u64 box_gap_pair(u64 x, float lo_a, float lo_b, float hi_a, float hi_b) {
    const float2 a = upk2(sub_pair(pk2(lo_a, lo_b), x)), b = upk2(sub_pair(x, pk2(hi_a, hi_b)));
    return pk2(fmaxf(fmaxf(a.x, b.x), 0.f), fmaxf(fmaxf(a.y, b.y), 0.f));
}
__device__ __forceinline__ float2 sq3_pair(u64 gx, u64 gy, u64 gz) {
    u64 r;
    asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(r) : "l"(gx));
    asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(r) : "l"(gy), "l"(r));
    asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(r) : "l"(gz), "l"(r));
    return upk2(r);
}
#endif
__device__ __forceinline__ bool tile_may_pass(const float4 &E, const float2 &Ez, const float4 &F10,
                                              const TileHdr &h, float s) {
    const float s2 = s * s;
#if SEG_PAIRBOX
    // the four end-point box distances as two packed pairs (direct: (0 vs box 0, 20 vs box 20); inverse:
    // (0 vs box 20, 20 vs box 0)), bit for bit box_d2's values; combined without short-circuits as below
    const bool p10 = box_d2(F10.x, F10.y, F10.z, h.lo10, h.hi10) <= s2;
    const u64 X = pk2(E.x, E.y), Y = pk2(E.z, E.w), Z = pk2(Ez.x, Ez.y);
    const float2 dd = sq3_pair(box_gap_pair(X, h.dxy_lo.x, h.dxy_lo.y, h.dxy_hi.x, h.dxy_hi.y),
                               box_gap_pair(Y, h.dxy_lo.z, h.dxy_lo.w, h.dxy_hi.z, h.dxy_hi.w),
                               box_gap_pair(Z, h.dz.x, h.dz.y, h.dz.z, h.dz.w));
    const float2 di = sq3_pair(box_gap_pair(X, h.ixy_lo.x, h.ixy_lo.y, h.ixy_hi.x, h.ixy_hi.y),
                               box_gap_pair(Y, h.ixy_lo.z, h.ixy_lo.w, h.ixy_hi.z, h.ixy_hi.w),
                               box_gap_pair(Z, h.iz.x, h.iz.y, h.iz.z, h.iz.w));
    return p10 & (((dd.x <= s2) & (dd.y <= s2)) | ((di.x <= s2) & (di.y <= s2)));
#elif defined(SEG_BOX_SHORTCIRCUIT)
    const bool p10 = box_d2(F10.x, F10.y, F10.z, h.lo10, h.hi10) <= s2;
    const bool pdir = box_d2(E.x, E.z, Ez.x, h.lo0, h.hi0) <= s2 && box_d2(E.y, E.w, Ez.y, h.lo20, h.hi20) <= s2;
    const bool pinv = box_d2(E.x, E.z, Ez.x, h.lo20, h.hi20) <= s2 && box_d2(E.y, E.w, Ez.y, h.lo0, h.hi0) <= s2;
    return p10 && (pdir || pinv);
#else
    // all five box distances, combined without short-circuits: the && form compiled to branches that
    // diverge across the warp's fibers (ncu r02: a third of the kernel's divergent branches)
    const bool p10 = box_d2(F10.x, F10.y, F10.z, h.lo10, h.hi10) <= s2;
    const bool d0 = box_d2(E.x, E.z, Ez.x, h.lo0, h.hi0) <= s2, d20 = box_d2(E.y, E.w, Ez.y, h.lo20, h.hi20) <= s2;
    const bool i0 = box_d2(E.x, E.z, Ez.x, h.lo20, h.hi20) <= s2, i20 = box_d2(E.y, E.w, Ez.y, h.lo0, h.hi0) <= s2;
    return p10 & ((d0 & d20) | (i0 & i20));
#endif
}

// MULTI (row f4's optional half, PAPER.md:163's original DWM assignment): every bundle within its threshold,
// as a bit mask per fiber (exact mode only).  The cascade is the same with the cutoff thr_b (no best-so-far
// across bundles), a bundle already accepted for a fiber is skipped, and an accepted candidate ORs its bit.
template <bool STATS, bool PAPER, bool MULTI = false>
__global__ void __launch_bounds__(NTHREADS, CTAS_PER_SM) k_classify(ClassifyParams p) {
    extern __shared__ __align__(128) unsigned char smem[];
    const SmemLayout L;
    float4 *ring = reinterpret_cast<float4 *>(smem + L.ring);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + L.bars);
    uint64_t *empty = full + STAGES;
    StageMeta *meta = reinterpret_cast<StageMeta *>(smem + L.meta);
    float4 *fe_all = reinterpret_cast<float4 *>(smem + L.fe);
    float4 *fm_all = reinterpret_cast<float4 *>(smem + L.fm);
    float4 *fez_all = reinterpret_cast<float4 *>(smem + L.fez);
    unsigned long long *best_all = reinterpret_cast<unsigned long long *>(smem + L.best);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool consumer = warp < NCW;
    // the fiber window (and k_cull's list) this CTA works on: the longest lists launch first
    const int cta = p.cta_order ? __ldg(p.cta_order + blockIdx.x) : (int)blockIdx.x;
    SEG_DCHECK(cta >= 0 && (size_t)cta * FPC < (size_t)p.n);
    const int cw = consumer ? warp : 0;
    float2 *fxy = reinterpret_cast<float2 *>(smem + L.fxy) + cw * (NMID * PP);   // [18][PP]
    float *fz = reinterpret_cast<float *>(smem + L.fz) + cw * (NMID * PP);       // [18][PP]
    float4 *fe = fe_all + cw * 32;
    float4 *fm = fm_all + cw * 32;
    float4 *fez = fez_all + cw * 32;
    unsigned long long *best = best_all + cw * 32;
    float *flen = reinterpret_cast<float *>(smem + L.flen) + cw * 32;
    uint16_t *q2e = reinterpret_cast<uint16_t *>(smem + L.q2e) + cw * Q2CAP;   // entries: c | fiber << 5 | o << 10 | stage << 11
    uint16_t *pe = reinterpret_cast<uint16_t *>(smem + L.pe) + cw * PECAP;     // MULTI: the tile's winners, same format
    // MULTI: this warp's 32 fibers' masks ([32][MULTI_WORDS] words in the otherwise unused q2r region)
    uint32_t *mmask = reinterpret_cast<uint32_t *>(smem + L.q2r) + cw * 32 * MULTI_WORDS;
    static_assert(32 * MULTI_WORDS <= Q2R_WORDS && (!PAPER_D2 || Q2CAP <= Q2R_WORDS), "q2r region");
    auto has_bundle = [&](int f, int b) -> bool { return (mmask[f * MULTI_WORDS + (b >> 5)] >> (b & 31)) & 1u; };
    float *q2r = reinterpret_cast<float *>(smem + L.q2r) + cw * Q2R_WORDS;

    // the producer lane sets up the ring and issues the first STAGES tile copies (or the end marker) at once,
    // so they land while the consumers ingest their fibers; the loop below continues from kpre
    const unsigned short *lst_g = reinterpret_cast<const unsigned short *>(p.tile_bits) + (size_t)cta * cull_stride(p.T);
    int kpre = 0, nlist = 0;
    __shared__ int s_nlist;   // SEG_NLIST: the list length, for the consumers' loop bound
    if (threadIdx.x == FPC) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, NCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        nlist = __ldg(lst_g);
        SEG_DCHECK(nlist >= 0 && nlist <= p.T);
#if SEG_EARLY_TMA
        if (SEG_NLIST) s_nlist = nlist;   // visible to the consumers after the CTA barrier that ends the ingest
        for (; kpre < STAGES && kpre < nlist + (SEG_NLIST ? 0 : 1); ++kpre) {
            if (kpre < nlist) {
                const int t = __ldg(lst_g + 1 + kpre);
                SEG_DCHECK(t >= 0 && t < p.T);
                if (!SEG_NLIST) meta[kpre].tile = t;
                mbar_arrive_expect_tx(full + kpre, TILE_STRIDE_BYTES);
                bulk_g2s(ring + kpre * TILE_STRIDE_F4, p.tiles + (size_t)t * TILE_STRIDE_F4, TILE_STRIDE_BYTES, full + kpre);
            } else {
                meta[kpre].tile = -1;   // end of stream
                mbar_arrive(full + kpre);
            }
        }
#endif
    }
    unsigned long long cnt[ST_N];
    long long ti0 = 0;
    if (STATS) {
#pragma unroll
        for (int k = 0; k < ST_N; ++k) cnt[k] = 0;
        cnt[ST_CTAS] = threadIdx.x == 0 ? 1 : 0;
        ti0 = clock64();
    }

    // ---- a1: coalesced fiber ingest (consumer warps) ----
    // the CTA's fibers interleaved over the warps (fiber i -> warp i % NCW): every warp gets a similar
    // share of every tile's work, so the warps sharing the ring stay in step (cfg 3: -1%, cfg 1: -6%
    // against contiguous 32-fiber slices; the CTA's fibers are all Morton-close anyway)
    const int gi = cta * FPC + lane * NCW + warp;
    const bool inrange = consumer && gi < p.n;
    const int fidx = inrange ? (p.perm ? __ldg(p.perm + gi) : gi) : -1;
    SEG_DCHECK(!inrange || (fidx >= 0 && fidx < p.n));
    if (consumer) {
        // every value straight from global into its shared-memory plane with 4-byte cp.async
        // (LDGSTS): this lane copies floats k0 = lane and k1 = 32 + lane (k1 < 63) of each of the
        // warp's 32 fibers, all in flight at once; then it checks the values it copied
        const int k0 = lane, k1 = 32 + lane;
        // plane of float k of a fiber: its address for fiber 0 of the warp and its stride in floats
        auto plane = [&](int k, int &stride) -> float * {
            // fe = (x0, x20, y0, y20), fez = (z0, z20, h0, h20), fm = (x10, y10, z10, h10)
            const int pt = k / 3, c = k % 3;
            if (pt == 0 || pt == 20) {
                if (c < 2) { stride = 4; return reinterpret_cast<float *>(fe) + 2 * c + (pt == 20 ? 1 : 0); }
                stride = 4;
                return reinterpret_cast<float *>(fez) + (pt == 20 ? 1 : 0);
            }
            if (pt == 10) { stride = 4; return reinterpret_cast<float *>(fm) + c; }
            if (c < 2) { stride = 2; return reinterpret_cast<float *>(fxy + mid_slot(pt) * PP) + c; }
            stride = 1;
            return fz + mid_slot(pt) * PP;
        };
        int s0 = 1, s1 = 1;
#ifdef SEG_INGEST_BRANCH
        float *d0 = plane(k0, s0), *d1 = plane(k1 < 3 * NPTS ? k1 : 0, s1);
#else
        // lane 31 has no second value (63 floats per fiber): it zero-fills a slot of flen instead (written
        // after the ingest in paper mode, unused in exact mode), so the loops below need no branch on k1
        float *d0 = plane(k0, s0), *d1 = k1 < 3 * NPTS ? plane(k1, s1) : flen;
        if (k1 >= 3 * NPTS) s1 = 1;
        const uint32_t n1 = k1 < 3 * NPTS ? 4u : 0u;
        const int k1s = k1 < 3 * NPTS ? k1 : 3 * NPTS - 1;
#endif
        int fjs = -1;
#pragma unroll INGEST_UNROLL
        for (int j = 0; j < 32; ++j) {
            const int fj = __shfl_sync(0xffffffffu, fidx, j);
            if (lane == j) fjs = fj;
            if (fj >= 0) {
                const float *src = p.fibers + (size_t)fj * (3 * NPTS);
                cp_async4(d0 + j * s0, src + k0);
#ifdef SEG_INGEST_BRANCH
                if (k1 < 3 * NPTS) cp_async4(d1 + j * s1, src + k1);
#else
                cp_async4_n(d1 + j * s1, src + k1s, n1);
#endif
            }
        }
        cp_async_wait_all();
        uint32_t fin = 0;   // bit j: this lane's two values of fiber j are finite
#pragma unroll INGEST_UNROLL
        for (int j = 0; j < 32; ++j) {
#ifdef SEG_INGEST_BRANCH
            const bool ok = isfinite(d0[j * s0]) && (k1 >= 3 * NPTS || isfinite(d1[j * s1]));
#else
            const bool ok = isfinite(d0[j * s0]) & isfinite(d1[j * s1]);
#endif
            fin |= (ok ? 1u : 0u) << j;
        }
        fin = __reduce_and_sync(0xffffffffu, fin);   // bit j: every value of fiber j is finite
        __syncwarp();
        {   // fm.w: NaN marks a non-finite fiber (or an empty slot); else the screen's half norms
            const bool okf = ((fin >> lane) & 1u) && fjs >= 0;
            const float4 e = fe[lane], m = fm[lane], z = fez[lane];
            fm[lane].w = okf ? screen_half_norm(m.x, m.y, m.z) : __int_as_float(0x7fffffff);
            fez[lane].z = okf ? screen_half_norm(e.x, e.z, z.x) : 0.f;
            fez[lane].w = okf ? screen_half_norm(e.y, e.w, z.y) : 0.f;
        }
        if (PAPER) {
            // chord length of this lane's fiber (reading R16), FP32, segments summed in order
            auto pt = [&](int i) -> float4 {
                if (i == 0) return make_float4(fe[lane].x, fe[lane].z, fez[lane].x, 0.f);
                if (i == 20) return make_float4(fe[lane].y, fe[lane].w, fez[lane].y, 0.f);
                if (i == 10) return fm[lane];
                const float2 a = fxy[mid_slot(i) * PP + lane];
                return make_float4(a.x, a.y, fz[mid_slot(i) * PP + lane], 0.f);
            };
            float len = 0.f;
            float4 prev = pt(0);
#pragma unroll
            for (int i = 1; i < NPTS; ++i) {
                const float4 cur = pt(i);
                len = __fadd_rn(len, __fsqrt_rn(d2(cur.x, cur.y, cur.z, prev)));
                prev = cur;
            }
            flen[lane] = len;
        }
        best[lane] = (p.seed && inrange) ? p.seed[fidx] : KEY_NONE;
        if (MULTI) {
#pragma unroll
            for (int w = 0; w < MULTI_WORDS; ++w) mmask[lane * MULTI_WORDS + w] = 0u;
        }
        if (STATS) cnt[ST_FIBERS] = inrange ? 1 : 0;
    }
    __syncthreads();
    // the seed (exact mode): k_cull named for each fiber the best-first winner of its nearest tile; the lane
    // evaluates that one candidate in full -- its fiber from shared memory, the centroid's 21 points from
    // the centroid-major copy -- with k_classify's arithmetic, and starts from its key.  It is one of the
    // candidates the tile stream would evaluate, so the result cannot change; a good start prunes the rest.
    if (consumer && p.seed_code && inrange && !isnan(fm[lane].w)) {
        const int code = __ldg(p.seed_code + fidx);
        if (code >= 0) {
            const int tn = code >> 6, c = (code >> 1) & 31;
            int o = code & 1;
            const float4 *cc = p.tiles_cm + ((size_t)tn * TILE + c) * NPTS;
            const TileHdr *h = reinterpret_cast<const TileHdr *>(p.tiles + (size_t)tn * TILE_STRIDE_F4);
            const float4 E = fe[lane], F10 = fm[lane];
            const float4 Ez = fez[lane];
            if (PAPER) {
                // paper mode: the orientation the end points infer, decided as in the dense loop (R17; an
                // exact tie -> the caller's direct orientation, i.e. stored-inverse for a reversed centroid)
                const float4 c0p = __ldg(cc), c20p = __ldg(cc + NPTS - 1);
                const float e00 = d2(E.x, E.z, Ez.x, c0p), e2020 = d2(E.y, E.w, Ez.y, c20p);
                const float e020 = d2(E.x, E.z, Ez.x, c20p), e200 = d2(E.y, E.w, Ez.y, c0p);
                const float flip = __ldg(reinterpret_cast<const float *>(p.tiles + (size_t)tn * TILE_STRIDE_F4 + TILE_HDR_F4) + TI_FLIP + c);
                const float mi = fmaxf(e020, e200), md = fmaxf(e00, e2020);
                o = (mi < md || (mi == md && flip != 0.f)) ? 1 : 0;
            }
            float r = d2(F10.x, F10.y, F10.z, __ldg(cc + 10));
            r = fmaxf(r, d2(E.x, E.z, Ez.x, __ldg(cc + (o ? NPTS - 1 : 0))));
            r = fmaxf(r, d2(E.y, E.w, Ez.y, __ldg(cc + (o ? 0 : NPTS - 1))));
#pragma unroll
            for (int i = 1; i < NPTS - 1; ++i) {
                if (i == 10) continue;
                const float2 a = fxy[mid_slot(i) * PP + lane];
                r = fmaxf(r, d2(a.x, a.y, fz[mid_slot(i) * PP + lane], __ldg(cc + (o ? NPTS - 1 - i : i))));
            }
            if (PAPER) {
                // score = d_ME + TN (Eq. 3), the lengths as the candidate rounds take them
                const float clen = __ldg(reinterpret_cast<const float *>(p.tiles + (size_t)tn * TILE_STRIDE_F4 + TILE_HDR_F4) + TI_LEN + c);
                const float sc = __fadd_rn(__fsqrt_rn(r), tn_f32(flen[lane], clen));
                // the same acceptance as a candidate of the tile stream: r <= thr2, then score <= thr
                if (r <= __ldg(&h->thr2) && sc <= __ldg(&h->thr)) {
                    const unsigned long long kk = ((unsigned long long)__float_as_uint(sc) << 32) | (uint32_t)__ldg(&h->bundle);
                    if (kk < best[lane]) best[lane] = kk;
                }
            } else if (r <= __ldg(&h->thr2)) {
                const unsigned long long kk = ((unsigned long long)__float_as_uint(r) << 32) | (uint32_t)__ldg(&h->bundle);
                if (kk < best[lane]) best[lane] = kk;
            }
        }
    }
    if (STATS && consumer && lane == 0) cnt[ST_CYC_INGEST] += clock64() - ti0;

    if (!consumer) {
        // ---- producer warp: stream the tiles k_cull listed for this CTA (TMA bulk copies) ----
        if (lane == 0) {
            int k = kpre;
            for (; k < nlist; ++k) {
                const int t = __ldg(lst_g + 1 + k);
                SEG_DCHECK(t >= 0 && t < p.T);
                const int s = k % STAGES, u = k / STAGES;
                if (u > 0) mbar_sleep_wait(empty + s, (u - 1) & 1);
                if (!SEG_NLIST) meta[s].tile = t;
                mbar_arrive_expect_tx(full + s, TILE_STRIDE_BYTES);
                bulk_g2s(ring + s * TILE_STRIDE_F4, p.tiles + (size_t)t * TILE_STRIDE_F4, TILE_STRIDE_BYTES, full + s);
            }
            if (!SEG_NLIST && kpre <= nlist) {   // end of stream, unless it went out with the first copies
                const int s = k % STAGES, u = k / STAGES;
                if (u > 0) mbar_sleep_wait(empty + s, (u - 1) & 1);
                meta[s].tile = -1;
                mbar_arrive(full + s);
            }
        }
    } else {
        // ---- consumers ----
        const uint32_t lt_mask = (1u << lane) - 1u;
        const float4 myE = fe[lane], myF10 = fm[lane];
        const float2 myEz = make_float2(fez[lane].x, fez[lane].y);
        const bool myok = !isnan(myF10.w);
        // candidate round: full Eq. 2 maximum for one orientation of (fiber fl, centroid c),
        // starting from its 3-point running max r
        // (a fiber may hold several lanes of a round: its best key is updated with a shared-memory atomicMin)
        auto run_cand = [&](const uint16_t *qe, const float *qr, int n) {
            if (STATS && lane == 0 && n > 0) { cnt[ST_ROUNDS]++; cnt[ST_ROUND_LANES] += n; }
#if defined(SEG_EXP) && SEG_EXP == 2
            n = 0;  // experiment: no candidate rounds
#endif
            if (lane < n) {
                const uint32_t e = (uint32_t)qe[lane];
                const int fl = (e >> 5) & 31, c = e & 31, o = (e >> 10) & 1, es = (e >> 11) & 3;
                SEG_DCHECK(es < STAGES && (e >> 13) == 0);
                // the candidate's tile: the ring stage recorded in its entry
                const float4 *estage = ring + es * TILE_STRIDE_F4;
                const float4 *T = estage + TILE_HDR_F4;
                const float *Tf = reinterpret_cast<const float *>(T);
                // the centroid's middle points in the caller's order: slot k, or TILE_MID - 1 - k reversed
                const int cofs = c + (o ? (TILE_MID - 1) * TILE : 0), st = o ? -TILE : TILE;
                const float2 *cxy = reinterpret_cast<const float2 *>(Tf + TI_MXY) + cofs;
                const float *cz = Tf + TI_MZ + cofs;
                float r;
                bool keep = true;
                if (PAPER && PAPER_D2) {
                    r = qr[lane];
                } else if (PAPER) {
                    // the paper's orientation (R17): argmin of the exact end-point maxima, an
                    // exact tie -> the caller's direct orientation; a candidate of the other orientation
                    // (kept only by the screen's superset) drops out here
                    const float4 a10 = fm[fl], E = fe[fl], Ez = fez[fl];
                    const float4 q0 = T[TI_P0 + c], q20 = T[TI_P20 + c];
                    const float e00 = d2(E.x, E.z, Ez.x, q0), e2020 = d2(E.y, E.w, Ez.y, q20);
                    const float e020 = d2(E.x, E.z, Ez.x, q20), e200 = d2(E.y, E.w, Ez.y, q0);
                    const float mi = fmaxf(e020, e200), md = fmaxf(e00, e2020);
                    const int oinf = (mi < md || (mi == md && Tf[TI_FLIP + c] != 0.f)) ? 1 : 0;
                    keep = o == oinf;
                    r = fmaxf(d2(a10.x, a10.y, a10.z, T[TI_P10 + c]), o ? mi : md);
                } else {
                    // exact mode screened with estimates: the 3-point running max, exactly as the
                    // dense test2 of the d2 form computes it (d2 and d2_pair_b agree bit for bit)
                    const float4 a10 = fm[fl], E = fe[fl], Ez = fez[fl];
                    r = fmaxf(fmaxf(d2(a10.x, a10.y, a10.z, T[TI_P10 + c]),
                                    d2(E.x, E.z, Ez.x, T[(o ? TI_P20 : TI_P0) + c])),
                              d2(E.y, E.w, Ez.y, T[(o ? TI_P0 : TI_P20) + c]));
                }
                const float thr2 = reinterpret_cast<const TileHdr *>(estage)->thr2;
                const float thr = reinterpret_cast<const TileHdr *>(estage)->thr;
                const int b = reinterpret_cast<const TileHdr *>(estage)->bundle;
                const float taul = MULTI ? (has_bundle(fl, b) ? -1.f : thr2) : fminf(thr2, key_cut2<PAPER>(best[fl]));
                if (keep && r <= taul) {  // re-check against the freshest best (an earlier round of this tile may have lowered it)
                    bool done = false;
#define SEG_STEP(i)                                                                                  \
    {                                                                                                \
const float2 a = fxy[mid_slot(i) * PP + fl];                                                 \
const float2 b = cxy[mid_slot(i) * st];                                                      \
r = fmaxf(r, d2(a.x, a.y, fz[mid_slot(i) * PP + fl], make_float4(b.x, b.y, cz[mid_slot(i) * st], 0.f))); \
    }
                    if (STATS) cnt[ST_T34]++;
                    SEG_STEP(3); SEG_STEP(17); SEG_STEP(7); SEG_STEP(13);
                    if (STATS) cnt[ST_PDIST] += 4;
                    if (r > taul) done = true;
                    if (!done) {
                        SEG_STEP(1); SEG_STEP(19); SEG_STEP(5); SEG_STEP(15);
                        if (STATS) cnt[ST_PDIST] += 4;
                        if (r > taul) done = true;
                    }
                    if (!done) {
                        SEG_STEP(2); SEG_STEP(18); SEG_STEP(4); SEG_STEP(16);
                        if (STATS) cnt[ST_PDIST] += 4;
                        if (r > taul) done = true;
                    }
                    if (!done) {
                        SEG_STEP(6); SEG_STEP(14); SEG_STEP(8); SEG_STEP(12); SEG_STEP(9);
                        SEG_STEP(11);
                        if (STATS) { cnt[ST_PDIST] += 6; cnt[ST_FULL]++; }
                        // a7: lexicographic (d^2, bundle) minimum; paper mode: (d_ME + TN, bundle)
                        if (PAPER) {
                            if (r <= taul) {
                                const float sc = __fadd_rn(__fsqrt_rn(r), tn_f32(flen[fl], Tf[TI_LEN + c]));
                                if (sc <= thr) {
                                    const unsigned long long kk = ((unsigned long long)__float_as_uint(sc) << 32) | (uint32_t)b;
                                    atomicMin(best + fl, kk);
                                    if (STATS) cnt[ST_UPD]++;
                                }
                            }
                        } else if (MULTI) {
                            if (r <= thr2) {
                                atomicOr(mmask + fl * MULTI_WORDS + (b >> 5), 1u << (b & 31));
                                if (STATS) cnt[ST_UPD]++;
                            }
                        } else if (r <= thr2) {
                            const unsigned long long kk = ((unsigned long long)__float_as_uint(r) << 32) | (uint32_t)b;
                            atomicMin(best + fl, kk);
                            if (STATS) cnt[ST_UPD]++;
                        }
                    }
#undef SEG_STEP
                }
            }
            __syncwarp();
        };
        int n2 = 0, np = 0;
        uint32_t pend = 0;   // ring stages (bits) whose candidates still wait on the stack
        auto flush = [&](int keep) {   // rounds of 32 off the top of the stack until at most `keep` are left
            long long tf0 = 0;
            if (STATS) tf0 = clock64();
            __syncwarp();
            if (MULTI && np > 0) run_cand(pe, q2r, np);   // MULTI: the winners first (q2r unused: no PAPER_D2)
            np = 0;
            while (n2 > keep) {
                const int m = n2 >= 32 ? 32 : n2;
                n2 -= m;
                run_cand(q2e + n2, q2r + n2, m);
            }
            if (STATS && lane == 0) cnt[ST_CYC_FLUSH] += clock64() - tf0;
        };
        long long tc0 = 0;
        if (STATS) tc0 = clock64();
        const int klim = SEG_NLIST ? s_nlist : 0x7fffffff;
        for (int k = 0; k < klim; ++k) {
            const int s = k % STAGES, u = k / STAGES;
            long long tw0 = 0;
            if (STATS) tw0 = clock64();
            constexpr int WAIT_NS = PAPER ? SEG_WAIT_NS_PAPER : SEG_WAIT_NS;
            if (WAIT_NS > 0) {
                while (!mbar_try(full + s, u & 1)) __nanosleep(WAIT_NS);
            } else {
                mbar_sleep_wait(full + s, u & 1);
            }
            if (STATS && lane == 0) cnt[ST_CYC_FULLWAIT] += clock64() - tw0;
            if (!SEG_NLIST && meta[s].tile < 0) break;
            const float4 *stage = ring + s * TILE_STRIDE_F4;
            const TileHdr th = *reinterpret_cast<const TileHdr *>(stage);
            const float thr2 = th.thr2;
            long long ts0 = 0;
            if (STATS) ts0 = clock64();
            // MULTI: the bundle's own threshold, or nothing once the fiber holds the bundle (tau < 0: the
            // bound's NaN radius fails every test)
            const float tau = MULTI ? (has_bundle(lane, th.bundle) ? -1.f : thr2)
                                    : fminf(thr2, key_cut2<PAPER>(best[lane]));
            constexpr bool D2FORM = SCREEN_OFF || (PAPER && PAPER_D2);
            const float tcmp = D2FORM ? tau : __fmul_rn(tau, 0.5f);   // the screen works at half scale
            // paper mode: this lane's stack-entry bits for the tile, opaque to the compiler (it would re-derive
            // the lane index with an S2R on every hit): paper -1.5%; exact mode +0.2%, so it keeps the plain form
            uint32_t ebase = 0;
            if (PAPER) asm volatile("mov.b32 %0, %1;" : "=r"(ebase) : "r"((uint32_t)(lane | (s << 11))));
            // a2 with the live cutoff: the exact sphere bound of this lane's fiber vs the tile
            // MUFU.SQRT (relative error < 2^-22) raised by 2^-20 so the radius never falls below the
            // exact one: no IEEE slow-path branch on the per-tile chain
            float sq;
            asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(sq) : "f"(tau));
            const float sb = __fmaf_ru(sq, 1.f + 0x1p-20f, CULL_EPS);
            const bool pass = myok && tile_may_pass(myE, myEz, myF10, th, sb);
            uint32_t pm = __ballot_sync(0xffffffffu, pass);
            if (STATS && lane == 0) cnt[ST_CYC_SPHERE] += clock64() - ts0;
#if defined(SEG_EXP) && SEG_EXP == 1
            pm = 0;  // experiment: tile loop overhead only
#endif
            if (STATS) {
                if (lane == 0) cnt[ST_WT_LISTED]++;
                if (myok) { cnt[ST_SPHERE]++; cnt[ST_PDIST] += 5; }
            }
            if (pm) {
                const float4 *T = stage + TILE_HDR_F4;
                if (STATS) {
                    if (lane == 0) cnt[ST_WT_COMPUTED]++;
                    if ((pm >> lane) & 1u) { cnt[ST_LT_PASS]++; cnt[ST_T1] += TILE; cnt[ST_PDIST] += TILE; }
                }
                // ---- a3 + a4, dense and transposed: lane = centroid, the warp walks its fibers ----
                const float4 c10 = T[TI_P10 + lane];
                const float4 c0 = T[TI_P0 + lane], c20 = T[TI_P20 + lane];
                constexpr int FB = PAPER ? SEG_FB_PAPER : SEG_FB;
#if SEG_JNEXT
                // one fiber per step (FB == 1): the next step's fiber is found during this step (highest set bit
                // first, FLO), so its FLO -> LEA -> LDS latency stays off the step's dependent chain (cfg 3 -3%,
                // paper -2.5%; the same for every fiber of an FB = 2 step, or the cutoff shuffle moved along too:
                // both lose)
                int jnext;
                asm("bfind.u32 %0, %1;" : "=r"(jnext) : "r"(pm));
#endif
#pragma unroll DENSE_UNROLL
                while (pm) {
                    // FB fibers per step: independent chains (ILP) and one warp vote per step
                    int jj[FB];
                    float rdv[FB], riv[FB], tjv[FB];
                    uint32_t hit = 0;
#if SEG_JNEXT
                    if (FB == 1) {
                        uint32_t below;
                        jj[0] = jnext;
                        asm("bmsk.clamp.b32 %0, 0, %1;" : "=r"(below) : "r"(jnext));   // the bits below jnext
                        pm &= below;
                        asm("bfind.u32 %0, %1;" : "=r"(jnext) : "r"(pm));             // -1 once pm is empty
                    } else
#endif
#pragma unroll
                    for (int q = 0; q < FB; ++q) {
                        // highest set bit first: FLO gives the index directly, and -1 once pm is empty
                        // (the order of a tile's fibers never changes a result: the best is a
                        // lexicographic minimum)
                        uint32_t bit;
                        asm("bfind.u32 %0, %1;" : "=r"(jj[q]) : "r"(pm));       // FLO: -1 if pm == 0
                        asm("shl.b32 %0, 1, %1;" : "=r"(bit) : "r"(jj[q]));     // PTX clamps: 0 for -1
                        pm &= ~bit;
                    }
#pragma unroll
                    for (int q = 0; q < FB; ++q) {
                        // an empty slot (-1) reads the word just before fe / fm / fez (in the same
                        // shared-memory block: fz, fe, fm come first) and lane 31's cutoff; its
                        // result is discarded by the jj >= 0 test below
                        const int j = jj[q];
                        // fiber j's end points arrive packed: (x0, x20), (y0, y20), (z0, z20)
                        const float4 E = fe[j];
                        const float4 Ez = fez[j];
                        const float4 a10 = fm[j];
                        const float tj = __shfl_sync(0xffffffffu, tcmp, j);
                        const u64 EX = f2u(make_float2(E.x, E.y)), EY = f2u(make_float2(E.z, E.w)),
                                  EZ = f2u(make_float2(Ez.x, Ez.y));
                        float m10;
                        float2 R0, R20;
                        if (D2FORM) {
                            m10 = d2(a10.x, a10.y, a10.z, c10);                         // test1
                            R0 = d2_pair_b(EX, EY, EZ, c0.x, c0.y, c0.z);               // (e0,0, e20,0)
                            R20 = d2_pair_b(EX, EY, EZ, c20.x, c20.y, c20.z);           // (e0,20, e20,20)
                        } else {
                            // exact mode: the dot-product screen, half scale (never above d2 / 2; the
                            // candidate rounds re-evaluate the three points exactly)
                            m10 = __fmaf_rn(a10.x, -c10.x, __fmaf_rn(a10.y, -c10.y,
                                      __fmaf_rn(a10.z, -c10.z, __fadd_rn(a10.w, c10.w))));
                            const u64 EN = f2u(make_float2(Ez.z, Ez.w));
                            R0 = screen_pair_b(EX, EY, EZ, c0.x, c0.y, c0.z, add_pair_b(EN, c0.w));
                            R20 = screen_pair_b(EX, EY, EZ, c20.x, c20.y, c20.z, add_pair_b(EN, c20.w));
                        }
                        rdv[q] = fmaxf(fmaxf(m10, R0.x), R20.y);                        // test2, direct
                        riv[q] = fmaxf(fmaxf(m10, R20.x), R0.y);                        // test2, inverse
                        if (PAPER && PAPER_D2) {
                            // the paper infers the direction from the end points:
                            // argmin of the end-point maxima, ties -> the caller's direct orientation
                            // (reading R17; the TI_FLIP word marks a centroid stored reversed); only that
                            // orientation goes on
                            const float mi = fmaxf(R20.x, R0.y), md = fmaxf(R0.x, R20.y);
                            if (mi < md || (mi == md && reinterpret_cast<const float *>(T)[TI_FLIP + lane] != 0.f)) rdv[q] = INFINITY;
                            else riv[q] = INFINITY;
                        }
                        tjv[q] = tj;
                        // one VOTE.ANY per fiber: far shorter latency than a REDUX.OR of the step's bits
                        // (cfg 3: -3.6%)
                        // one fiber per step: the loop runs while pm != 0, so the slot is never empty (no
                        // jj >= 0 test on the vote's dependent chain)
                        const bool live = (FB == 1 && !SEG_VOTE_JJ_ALWAYS) || jj[q] >= 0;
                        if (__any_sync(0xffffffffu, live && fminf(rdv[q], riv[q]) <= tj)) hit |= 1u << q;
                        if (STATS && jj[q] >= 0 && m10 <= tj) { cnt[ST_T2]++; cnt[ST_PDIST] += 4; }
                    }
#if defined(SEG_EXP) && SEG_EXP == 3
                    hit = p.n < 0 ? hit : 0;  // experiment: dense test1+test2 only (opaque, so it is not dead code)
#endif
                    if (!hit) continue;
                    long long th0 = 0;
                    if (STATS) th0 = clock64();
                    // one copy of the selection code, the step's hit fibers picked by selects
                    // (keeps the kernel's code small: the q loop unrolled it FB times, flush included)
                    for (uint32_t hb = hit; hb; hb &= hb - 1) {
                        const int q = __ffs(hb) - 1;
                        int j = jj[0];
                        float rd = rdv[0], ri = riv[0], tj = tjv[0];
#pragma unroll
                        for (int t = 1; t < FB; ++t)
                            if (q == t) { j = jj[t]; rd = rdv[t]; ri = riv[t]; tj = tjv[t]; }
                        const bool ad = rd <= tj, ai = ri <= tj;
                        // every surviving orientation goes onto the candidate stack.  (Round 1 sent each fiber's
                        // best 3-point survivor to a winners' round first, for its fresher cutoff: one more round
                        // per tile, which costs more than its pruning saves -- DESIGN.md Sec. 5)
                        if (STATS && lane == 0) cnt[ST_HITS]++;
                        const uint32_t e = PAPER ? ebase | (uint32_t)(j << 5) : (uint32_t)((j << 5) | lane | (s << 11));
                        bool qd = ad, qi = ai;
                        if (MULTI) {
                            // multi-label masks keep a winners' round: one accepted centroid settles the bundle
                            // for the fiber, so the tile's other candidates of that fiber stop at their re-check.
                            // The winner is the smallest screened 3-point score (lane in the 5 low bits)
                            const float sc = fmaxf(fminf(ad ? rd : INFINITY, ai ? ri : INFINITY), 0.f);
                            const int wo = (ad && (!ai || rd <= ri)) ? 0 : 1;
                            const uint32_t smin = __reduce_min_sync(0xffffffffu, (__float_as_uint(sc) & ~31u) | (uint32_t)lane);
                            const bool win = lane == (int)(smin & 31u);
                            SEG_DCHECK(np < PECAP);
                            if (win) pe[np] = (uint16_t)(e | ((uint32_t)wo << 10));
                            ++np;
                            qd = ad && !(win && wo == 0);
                            qi = ai && !(win && wo == 1);
                        }
                        const uint32_t bd = __ballot_sync(0xffffffffu, qd), bi = __ballot_sync(0xffffffffu, qi);
                        if (qd) {
                            const int pos = n2 + __popc(bd & lt_mask);
                            q2e[pos] = (uint16_t)e;
                            if (PAPER && PAPER_D2) q2r[pos] = rd;
                        }
                        if (qi) {
                            const int pos = n2 + __popc(bd) + __popc(bi & lt_mask);
                            q2e[pos] = (uint16_t)(e | (1u << 10));
                            if (PAPER && PAPER_D2) q2r[pos] = ri;
                        }
                        n2 += __popc(bd) + __popc(bi);
                        SEG_DCHECK(n2 <= Q2CAP);
                        if (n2 > Q2CAP - 64) flush(31);
                    }
                    if (STATS && lane == 0) cnt[ST_CYC_HIT] += clock64() - th0;
                }
            }
            // a stack shorter than one round waits for the next tile's entries (its stage stays held, at most
            // DEFER_TILES of them: the producer refills a stage only after every warp released it, and this
            // warp's next tile must not depend on a stage it holds itself)
            if (!MULTI && n2 > 0 && n2 < DEFER_BELOW && __popc(pend) < DEFER_TILES) {
                pend |= 1u << s;
                continue;
            }
            flush(0);
            __syncwarp();
            pend |= 1u << s;
            if (lane == 0)
                for (uint32_t b = pend; b; b &= b - 1) mbar_arrive(empty + (__ffs(b) - 1));
            pend = 0;
        }
        if (pend) flush(0);

        if (STATS && lane == 0) cnt[ST_CYC_CONS] += clock64() - tc0;
        // ---- a8: epilogue ----
        if (inrange) {
            const unsigned long long key = best[lane];
            int lab;
            float dd;
            if (isnan(fm[lane].w)) {
                lab = -1;
                dd = __int_as_float(0x7fffffff);  // NaN: non-finite fiber
            } else if (key != KEY_NONE) {
                lab = (int)(uint32_t)(key & 0xffffffffu);
                dd = PAPER ? key_d2(key) : __fsqrt_rn(key_d2(key));   // paper mode keys hold the score
            } else {
                lab = -1;
                dd = INFINITY;
            }
            if (MULTI) {
                const bool fin = !isnan(fm[lane].w);
                for (int w = 0; w < p.mwords; ++w)
                    p.masks[(size_t)fidx * p.mwords + w] = (fin && w < MULTI_WORDS) ? mmask[lane * MULTI_WORDS + w] : 0u;
            } else if (p.keys) {
                // row f4: the raw best key for an atlas-sharded run (all_reduce MIN over the shards);
                // exchange space: every key < 2^63, NONE = INT64_MAX, non-finite = INT64_MAX - 1
                p.keys[fidx] = isnan(fm[lane].w) ? KEY_X_NONFINITE : key == KEY_NONE ? KEY_X_NONE : key;
            } else {
                p.label[fidx] = lab;
                p.dist[fidx] = dd;
            }
        }
    }
    if (STATS) {
#pragma unroll
        for (int j = 0; j < ST_N; ++j) {
            unsigned long long v = cnt[j];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0 && v) atomicAdd(p.stats + j, v);
        }
    }
}

// ----------------------------------------------------------------------------------------
// a2 (list): k_cull -- per CTA of the classify kernel (the same FPC fibers), the tiles some fiber may
// need under its bundle threshold: bundle test on the point-10 sphere, then the 3-sphere tile test
// for the tiles of the surviving bundles.  Written as an ordered list per CTA ([count, tiles...]),
// best-first (see below).  A separate, light kernel (no big shared-memory ring) so its
// latency-bound header loads run at full occupancy.
// ----------------------------------------------------------------------------------------
#ifndef SEG_CULL_XPOSE
#define SEG_CULL_XPOSE 1   // k_cull's per-chunk pass / inside counts by a warp bit-matrix transpose (-4%)
#endif
#ifndef SEG_CULL_APPEND
#define SEG_CULL_APPEND 1  // k_cull: tiles appended to the list as they are first marked (no list-building pass; -1.4%)
#endif
#ifndef SEG_CULL_WBOX
#define SEG_CULL_WBOX 1   // k_cull: each warp's candidate bundles from the box of its points 10 (no CTA union; -8%)
#endif
#ifndef SEG_CULL_MAXREG_CTAS
#define SEG_CULL_MAXREG_CTAS 5
#endif
// k_cull's dynamic shared memory: [twords + bwords + T] u32 (tile bits, bundle bits, priorities), [T] u16 list
__host__ __device__ inline size_t cull_smem_bytes(int T, int B) {
    return sizeof(uint32_t) * (size_t)(((T + 31) >> 5) + ((B + 31) >> 5) + T) + sizeof(uint16_t) * (size_t)T;
}
__global__ void __launch_bounds__(FPC, SEG_CULL_MAXREG_CTAS) k_cull(ClassifyParams p) {
    // smem: [twords] tile bits, [bwords] bundle bits, [T] per-tile priority, [T] list (u16)
    extern __shared__ __align__(16) uint32_t sbits[];
    const int twords = (p.T + 31) >> 5, bwords = (p.B + 31) >> 5;
    uint32_t *tb = sbits, *bb = sbits + twords, *prio = bb + bwords;
    uint16_t *lst = reinterpret_cast<uint16_t *>(prio + p.T);
    __shared__ int nlist;
    // per bundle the point-10 sphere grown by the bundle threshold: (centre, R^2); an empty bundle (and
    // the padding up to a multiple of 32) gets a centre at 1e30 so that no fiber passes it
    __shared__ float4 sbs[MAX_SMEM_BUNDLES];
    for (int i = threadIdx.x; i < twords + bwords + p.T; i += FPC) sbits[i] = 0;
    if (SEG_CULL_APPEND && threadIdx.x == 0) nlist = 0;
    const bool stage_bh = p.B <= MAX_SMEM_BUNDLES;
    auto bsphere = [&](int b) {
        if (b >= p.B) return make_float4(1e30f, 1e30f, 1e30f, 0.f);
        const BundleHdr h = p.bh[b];
        const float r = h.s10.w + h.thr + CULL_EPS;
        return h.t1 > h.t0 ? make_float4(h.s10.x, h.s10.y, h.s10.z, r * r) : make_float4(1e30f, 1e30f, 1e30f, 0.f);
    };
    const int bpad = (p.B + 31) & ~31;
    if (stage_bh)
        for (int i = threadIdx.x; i < bpad; i += FPC) sbs[i] = bsphere(i);
    const int lane = threadIdx.x & 31;
    const int gi = blockIdx.x * FPC + threadIdx.x;
    bool ok = gi < p.n;
    float4 E = make_float4(0.f, 0.f, 0.f, 0.f), F10 = E;
    float2 Ez = make_float2(0.f, 0.f);
    if (ok) {
        const int fidx = p.perm ? __ldg(p.perm + gi) : gi;
        const float *src = p.fibers + (size_t)fidx * (3 * NPTS);
        E = make_float4(__ldg(src + 0), __ldg(src + 60), __ldg(src + 1), __ldg(src + 61));
        Ez = make_float2(__ldg(src + 2), __ldg(src + 62));
        F10 = make_float4(__ldg(src + 30), __ldg(src + 31), __ldg(src + 32), 0.f);
        ok = isfinite(E.x) && isfinite(E.y) && isfinite(E.z) && isfinite(E.w) && isfinite(Ez.x) && isfinite(Ez.y) &&
             isfinite(F10.x) && isfinite(F10.y) && isfinite(F10.z);
    }
    if (!ok) F10 = make_float4(__int_as_float(0x7fffffff), 0.f, 0.f, 0.f);   // NaN: every bound test fails
    float nd2 = INFINITY;   // each fiber's nearest tile by its sphere centres: the seed's tile
    int ntile = -1;
    __syncthreads();
#if SEG_CULL_WBOX
    // each warp's candidate bundles, lane = bundle: the distance from the box of the warp's points 10 to a bundle's
    // grown point-10 sphere, with d2's operation sequence, is never above a member fiber's own d2 (every rounding
    // is monotone), so the candidates hold every bundle a fiber of the warp passes; each is re-tested per fiber
    float blo[3], bhi[3];
    {
        const bool v = !isnan(F10.x);   // a non-finite fiber carries F10.x = NaN and passes nothing
        blo[0] = v ? F10.x : INFINITY; blo[1] = v ? F10.y : INFINITY; blo[2] = v ? F10.z : INFINITY;
        bhi[0] = v ? F10.x : -INFINITY; bhi[1] = v ? F10.y : -INFINITY; bhi[2] = v ? F10.z : -INFINITY;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                blo[k] = fminf(blo[k], __shfl_xor_sync(0xffffffffu, blo[k], o));
                bhi[k] = fmaxf(bhi[k], __shfl_xor_sync(0xffffffffu, bhi[k], o));
            }
    }
    for (int w = 0; w < bwords; ++w) {
        uint32_t bits;
        {
            const float4 c = stage_bh ? sbs[(w << 5) + lane] : bsphere((w << 5) + lane);   // padded past B
            const float gx = fmaxf(fmaxf(__fsub_rn(blo[0], c.x), __fsub_rn(c.x, bhi[0])), 0.f);
            const float gy = fmaxf(fmaxf(__fsub_rn(blo[1], c.y), __fsub_rn(c.y, bhi[1])), 0.f);
            const float gz = fmaxf(fmaxf(__fsub_rn(blo[2], c.z), __fsub_rn(c.z, bhi[2])), 0.f);
            bits = __ballot_sync(0xffffffffu, __fmaf_rn(gz, gz, __fmaf_rn(gy, gy, __fmul_rn(gx, gx))) <= c.w);
        }
        while (bits) {
#else
    // bundles some fiber of the CTA may need (point-10 sphere + threshold, exact)
    for (int b0 = 0; b0 < p.B; b0 += 32) {
        uint32_t m = 0;
#pragma unroll BUNDLE_UNROLL
        for (int j = 0; j < 32; ++j) {
            const float4 c = stage_bh ? sbs[b0 + j] : bsphere(b0 + j);
            m |= (d2(F10.x, F10.y, F10.z, c) <= c.w ? 1u : 0u) << j;
        }
        m = __reduce_or_sync(0xffffffffu, m);
        if (lane == 0 && m) atomicOr(bb + (b0 >> 5), m);
    }
    __syncthreads();
    for (int w = 0; w < bwords; ++w) {
        uint32_t bits = bb[w];
        while (bits) {
#endif
            const int b = (w << 5) + __ffs(bits) - 1;
            bits &= bits - 1;
            const float4 c = stage_bh ? sbs[b] : bsphere(b);
            const bool bpass = d2(F10.x, F10.y, F10.z, c) <= c.w;
            if (!__any_sync(0xffffffffu, bpass)) continue;
            const BundleHdr h = p.bh[b];
#if defined(SEG_EXP) && SEG_EXP == 5
            // experiment: every tile of a passing bundle listed, no per-fiber tile tests
            for (int t = h.t0 + lane; t < h.t1; t += 32) atomicOr(tb + (t >> 5), 1u << (t & 31));
            if (h.t1 > 0) continue;
#endif
            for (int t0 = h.t0; t0 < h.t1; t0 += 32) {
                // 32 tiles per chunk: independent header loads and tests (ILP)
                const int nt = min(32, h.t1 - t0);
                uint32_t pm = 0, cm = 0;
#pragma unroll CULL_UNROLL
                for (int j = 0; j < 32; ++j) {
                    if (j < nt) {
                        const CullTile ct = p.ct[t0 + j];
                        // the threshold-only three-sphere bound (squared radii precomputed), and the
                        // processing priority: fibers whose points 0/10/20 lie inside the spheres
                        const float d10 = d2(F10.x, F10.y, F10.z, ct.c10);
                        const float d00 = d2(E.x, E.z, Ez.x, ct.c0), d2020 = d2(E.y, E.w, Ez.y, ct.c20);
                        const float d020 = d2(E.x, E.z, Ez.x, ct.c20), d200 = d2(E.y, E.w, Ez.y, ct.c0);
                        const bool pass = bpass && d10 <= ct.c10.w &&
                                          ((d00 <= ct.c0.w && d2020 <= ct.c20.w) || (d020 <= ct.c20.w && d200 <= ct.c0.w));
                        const bool close = pass && d10 <= ct.q.y &&
                                           ((d00 <= ct.q.x && d2020 <= ct.q.z) || (d020 <= ct.q.z && d200 <= ct.q.x));
                        pm |= (pass ? 1u : 0u) << j;
                        cm |= (close ? 1u : 0u) << j;
                        const float dc = fmaxf(d10, fminf(fmaxf(d00, d2020), fmaxf(d020, d200)));
                        if (pass && dc < nd2) { nd2 = dc; ntile = t0 + j; }
                    }
                }
                // transpose: lane j gets the pass / inside counts of tile t0 + j over the warp,
                // then every lane records its own tile (parallel shared atomics)
                uint32_t any = __reduce_or_sync(0xffffffffu, pm);
                int npass = 0, nclose = 0;
#if SEG_CULL_XPOSE
                // the 32 x 32 bit matrices (lane = fiber, bit = tile) transposed in five butterfly stages, so lane j
                // holds tile j's column: 2 x 5 shuffles instead of 2 ballots per passing tile (~19 per chunk)
                if (any) {
                    uint32_t tp = pm, tc = cm;
#pragma unroll
                    for (int sh = 16; sh > 0; sh >>= 1) {
                        const uint32_t m = sh == 16 ? 0x0000ffffu : sh == 8 ? 0x00ff00ffu : sh == 4 ? 0x0f0f0f0fu
                                         : sh == 2 ? 0x33333333u : 0x55555555u;
                        const uint32_t yp = __shfl_xor_sync(0xffffffffu, tp, sh);
                        const uint32_t yc = __shfl_xor_sync(0xffffffffu, tc, sh);
                        const bool hi = (lane & sh) != 0;
                        tp = hi ? (((yp >> sh) & m) | (tp & ~m)) : ((tp & m) | ((yp << sh) & ~m));
                        tc = hi ? (((yc >> sh) & m) | (tc & ~m)) : ((tc & m) | ((yc << sh) & ~m));
                    }
                    npass = __popc(tp);
                    nclose = __popc(tc);
                }
#else
                while (any) {
                    const int j = __ffs(any) - 1;
                    any &= any - 1;
                    const int a = __popc(__ballot_sync(0xffffffffu, (pm >> j) & 1u));
                    const int c2 = __popc(__ballot_sync(0xffffffffu, (cm >> j) & 1u));
                    if (lane == j) { npass = a; nclose = c2; }
                }
#endif
                if (npass) {
                    const int t = t0 + lane;
#if SEG_CULL_APPEND
                    // the first lane to mark a tile appends it to the (unordered) list; the ranking below orders it
                    const uint32_t bit = 1u << (t & 31);
                    if (!(atomicOr(tb + (t >> 5), bit) & bit)) lst[atomicAdd(&nlist, 1)] = (uint16_t)t;
#else
                    atomicOr(tb + (t >> 5), 1u << (t & 31));
#endif
                    atomicAdd(prio + t, (uint32_t)nclose * 256u + (uint32_t)npass);
                }
            }
        }
    }
    // the seed candidate (exact mode): per fiber, the best-first winner of its nearest tile (smallest 3-point
    // score), named as (tile, centroid, orientation) for k_classify, which evaluates it in full and starts
    // from it.  Warp-cooperative: lane = centroid for the 3-point scores (the tile's rows stay in registers
    // while consecutive fibers share the tile); only points 0 / 10 / 20, already in registers, are needed.
    if (p.seed_code) {
        const int myfidx = gi < p.n ? (p.perm ? __ldg(p.perm + gi) : gi) : -1;
        const bool want = myfidx >= 0 && ntile >= 0;
        if (myfidx >= 0 && !want) p.seed_code[myfidx] = -1;
#if defined(SEG_EXP) && (SEG_EXP == 4 || SEG_EXP == 5)
        if (want) p.seed_code[myfidx] = -1;   // experiment: no seeds
        if (p.n >= 0) goto seed_done;
#endif
        int ct = -1;
        float thr2 = 0.f;
        float4 c10 = make_float4(0.f, 0.f, 0.f, 0.f), c0 = c10, c20 = c10;
        for (uint32_t rem = __ballot_sync(0xffffffffu, want); rem; rem &= rem - 1) {
            const int j = __ffs(rem) - 1;
            const int fj = __shfl_sync(0xffffffffu, myfidx, j);
            const int tj = __shfl_sync(0xffffffffu, ntile, j);
            if (tj != ct) {
                ct = tj;
                const float4 *tile = p.tiles + (size_t)tj * TILE_STRIDE_F4;
                const TileHdr *h = reinterpret_cast<const TileHdr *>(tile);
                const float4 *T = tile + TILE_HDR_F4;
                thr2 = __ldg(&h->thr2);
                c10 = __ldg(T + TI_P10 + lane);
                c0 = __ldg(T + TI_P0 + lane);
                c20 = __ldg(T + TI_P20 + lane);
            }
            const float4 Ej = make_float4(__shfl_sync(0xffffffffu, E.x, j), __shfl_sync(0xffffffffu, E.y, j),
                                          __shfl_sync(0xffffffffu, E.z, j), __shfl_sync(0xffffffffu, E.w, j));
            const float2 Ezj = make_float2(__shfl_sync(0xffffffffu, Ez.x, j), __shfl_sync(0xffffffffu, Ez.y, j));
            const float3 Fj = make_float3(__shfl_sync(0xffffffffu, F10.x, j), __shfl_sync(0xffffffffu, F10.y, j),
                                          __shfl_sync(0xffffffffu, F10.z, j));
            const float m10 = d2(Fj.x, Fj.y, Fj.z, c10);
            const float rd = fmaxf(fmaxf(m10, d2(Ej.x, Ej.z, Ezj.x, c0)), d2(Ej.y, Ej.w, Ezj.y, c20));
            const float ri = fmaxf(fmaxf(m10, d2(Ej.x, Ej.z, Ezj.x, c20)), d2(Ej.y, Ej.w, Ezj.y, c0));
            const float sc = fminf(rd <= thr2 ? rd : INFINITY, ri <= thr2 ? ri : INFINITY);
            const uint32_t smin = __reduce_min_sync(0xffffffffu, (__float_as_uint(sc) & ~31u) | (uint32_t)lane);
            int32_t code = -1;   // (tile << 6) | (centroid << 1) | orientation of the winner, -1 = none
            if ((smin & ~31u) < 0x7f800000u) {
                const int wl = (int)(smin & 31u);
                const int wo = __shfl_sync(0xffffffffu, (rd <= thr2 && rd == sc) ? 0 : 1, wl);
                code = (ct << 6) | (wl << 1) | wo;
            }
            if (lane == 0) p.seed_code[fj] = code;
        }
    }
#if defined(SEG_EXP) && (SEG_EXP == 4 || SEG_EXP == 5)
seed_done:
#endif
    __syncthreads();
#if !SEG_CULL_APPEND
    // the CTA's tiles from the bit set (warp 0: prefix over the words), in tile order
    if (threadIdx.x < 32) {
        int base = 0;
        for (int w0 = 0; w0 < twords; w0 += 32) {
            const uint32_t bits = w0 + lane < twords ? tb[w0 + lane] : 0u;
            const int c = __popc(bits);
            int incl = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            int pos = base + incl - c;
            uint32_t bb2 = bits;
            while (bb2) {
                lst[pos++] = (uint16_t)(((w0 + lane) << 5) + __ffs(bb2) - 1);
                bb2 &= bb2 - 1;
            }
            base += __shfl_sync(0xffffffffu, incl, 31);
        }
        SEG_DCHECK(base <= p.T);
        if (lane == 0) nlist = base;
    }
    __syncthreads();
#endif
    SEG_DCHECK(nlist <= p.T);
    // best-first order for k_classify: tiles that contain more of the CTA's fibers (inside all
    // three spheres) first, then tiles that more fibers may need, then the tile index.  Any order
    // gives the same result (the (d^2, bundle) minimum is order-independent); a good order makes
    // the running best tight early, which prunes the later tiles.
    const int n = nlist;
    uint16_t *out = reinterpret_cast<uint16_t *>(p.tile_bits) + (size_t)blockIdx.x * cull_stride(p.T);
    if (threadIdx.x == 0) {
        out[0] = (uint16_t)n;
        if (p.cta_order) p.cta_order[blockIdx.x] = n;   // k_cta_order's input (LPT launch order)
    }
    for (int i = threadIdx.x; i < n; i += FPC) {
        const int ti = lst[i];
        const uint32_t ki = prio[ti];
        int rank = 0;
#pragma unroll RANK_UNROLL
        for (int k = 0; k < n; ++k) {
            const int tk = lst[k];
            const uint32_t kk = prio[tk];
            rank += (kk > ki || (kk == ki && tk < ti)) ? 1 : 0;
        }
        SEG_DCHECK(rank < n);
        out[1 + rank] = (uint16_t)ti;
    }
}

// row f4: keys -> (label, dist), the decode of an atlas-sharded run
__global__ void k_keys_to_labels(const unsigned long long *keys, int64_t n, int paper, int32_t *label, float *dist) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned long long k = keys[i];
    if (k == KEY_X_NONE) {
        label[i] = -1;
        dist[i] = INFINITY;
    } else if (k >= KEY_X_NONFINITE) {
        label[i] = -1;
        dist[i] = __int_as_float(0x7fffffff);
    } else {
        label[i] = (int32_t)(uint32_t)(k & 0xffffffffu);
        const float v = __uint_as_float((uint32_t)(k >> 32));
        dist[i] = paper ? v : __fsqrt_rn(v);
    }
}

cudaError_t launch_keys_to_labels(const unsigned long long *keys, int64_t n, int paper, int32_t *label, float *dist,
                                  cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    k_keys_to_labels<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(keys, n, paper, label, dist);
    return cudaGetLastError();
}

size_t classify_smem_bytes(int, int) { return SmemLayout().total; }

int classify_fibers_per_cta() { return FPC; }

int classify_max_tiles() { return MAX_TILES; }

int classify_multi_max_bundles() { return 32 * MULTI_WORDS; }

size_t cull_bits_words(int n, int T) { return (size_t)((n + FPC - 1) / FPC) * (size_t)(cull_stride(T) / 2); }

// Longest-processing-time-first launch order for k_classify: CTAs sorted by the length of k_cull's tile
// list (descending, in 2,048 buckets), so the longest windows do not land in the grid's last wave.  Any
// order gives the same results (windows are independent).
constexpr int LPT_BUCKETS = 2048;
// k_cull left each window's list length in order[window]; one block reads them all (coalesced, at most
// 32 per thread: slices hold at most 2^23 fibers = 32,768 windows), then overwrites order with the ranking.
constexpr int LPT_PER_THREAD = 32;
__global__ void __launch_bounds__(1024) k_cta_order(int ncta, int T, int32_t *order) {
    __shared__ uint32_t cnt[LPT_BUCKETS];
    __shared__ uint32_t wsum[33];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    for (int i = t; i < LPT_BUCKETS; i += 1024) cnt[i] = 0;
    __syncthreads();
    SEG_DCHECK(ncta <= 1024 * LPT_PER_THREAD);
    int bk[LPT_PER_THREAD];
#pragma unroll
    for (int k = 0; k < LPT_PER_THREAD; ++k) {
        const int c = t + 1024 * k;
        const long long len = c < ncta ? order[c] : 0;
        bk[k] = LPT_BUCKETS - 1 - (int)min((long long)LPT_BUCKETS - 1, len * LPT_BUCKETS / (T + 1));
    }
#pragma unroll
    for (int k = 0; k < LPT_PER_THREAD; ++k)
        if (t + 1024 * k < ncta) atomicAdd(&cnt[bk[k]], 1u);
    __syncthreads();
    const uint32_t a = cnt[2 * t], b = cnt[2 * t + 1];
    uint32_t incl = a + b;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    if (w == 0) {
        const uint32_t x = wsum[lane];
        uint32_t xi = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, xi, o);
            if (lane >= o) xi += v;
        }
        wsum[lane] = xi - x;
    }
    __syncthreads();
    const uint32_t ex = wsum[w] + incl - (a + b);
    cnt[2 * t] = ex;
    cnt[2 * t + 1] = ex + a;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < LPT_PER_THREAD; ++k) {
        const int c = t + 1024 * k;
        if (c < ncta) {
            const uint32_t pos = atomicAdd(&cnt[bk[k]], 1u);
            SEG_DCHECK(pos < (uint32_t)ncta);
            order[pos] = c;
        }
    }
}

cudaError_t launch_classify(const ClassifyParams &p, bool stats, cudaStream_t s, cudaEvent_t after_cull) {
    if (p.n <= 0) return cudaSuccess;
    const size_t smem = classify_smem_bytes(p.B, p.T);
    const int grid = (p.n + FPC - 1) / FPC;
    const size_t cull_smem = cull_smem_bytes(p.T, p.B);
    cudaError_t e = cudaFuncSetAttribute(k_cull, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cull_smem);
    if (e != cudaSuccess) return e;
    k_cull<<<grid, FPC, cull_smem, s>>>(p);
    if (p.cta_order) k_cta_order<<<1, 1024, 0, s>>>(grid, p.T, p.cta_order);
    if (after_cull) {
        e = cudaEventRecord(after_cull, s);
        if (e != cudaSuccess) return e;
    }
    auto go = [&](auto kern) {
        cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (r != cudaSuccess) return r;
        kern<<<grid, NTHREADS, smem, s>>>(p);
        return cudaSuccess;
    };
    if (p.masks) e = stats ? go(k_classify<true, false, true>) : go(k_classify<false, false, true>);
    else if (p.paper) e = stats ? go(k_classify<true, true>) : go(k_classify<false, true>);
    else e = stats ? go(k_classify<true, false>) : go(k_classify<false, false>);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace seg
