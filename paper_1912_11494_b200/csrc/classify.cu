// classify.cu -- sm_100a kernels of the segmentation hot path.
//
//   k_morton_hist / k_scan_exclusive / k_morton_scatter   (a9) spatial-order prepass: a counting
//        sort of the fibers by the Morton code of point 10, so that a warp holds 32 nearby fibers
//        and its lanes want the same atlas tiles (the B200 analogue of the paper's data-locality
//        argument).
//   k_classify                                             (a1-a8) one fiber per thread, its 63
//        coordinates in registers (a1); atlas tiles of 32 centroids streamed into shared memory by
//        1-D TMA bulk copies through an mbarrier ring fed by a producer warp; per tile an exact
//        sphere lower bound (a2) decided by warp ballot, then the paper's cascade per centroid:
//        test1 centre point (a3), test2 end points with sound orientation pruning (a4), test3 four
//        points (a5), test4 all 21 points with early exit (a6), the
//        closest-bundle update kept in registers (a7) and a coalesced
//        epilogue scattered back through the permutation (a8).
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

// ----------------------------------------------------------------------------------------
// a9: spatial-order prepass (counting sort on a 2^18-bucket Morton grid of point 10)
// ----------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t spread3(uint32_t v) {  // 6 bits -> every third bit
    v &= 0x3f;
    v = (v | (v << 8)) & 0x0000f00fu;
    v = (v | (v << 4)) & 0x000c30c3u;
    v = (v | (v << 2)) & 0x00249249u;
    return v;
}

__global__ void k_morton_hist(MortonParams p) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= p.n) return;
    const float *f = p.fibers + (size_t)i * (3 * NPTS) + 30;  // point 10
    const float lim = (float)((1 << MORTON_BITS) - 1);
    // fmaxf/fminf map NaN to the bound, so non-finite fibers land in a valid bucket
    const float qx = fminf(fmaxf((__ldg(f + 0) - p.lo.x) * p.inv_cell.x, 0.f), lim);
    const float qy = fminf(fmaxf((__ldg(f + 1) - p.lo.y) * p.inv_cell.y, 0.f), lim);
    const float qz = fminf(fmaxf((__ldg(f + 2) - p.lo.z) * p.inv_cell.z, 0.f), lim);
    const uint32_t k = spread3((uint32_t)qx) | (spread3((uint32_t)qy) << 1) | (spread3((uint32_t)qz) << 2);
    p.key[i] = k;
    atomicAdd(p.hist + k, 1u);
}

// In-place exclusive scan of MORTON_BUCKETS counters by one CTA of 1024 threads, 4 per thread per
// round (uint4 loads), carry propagated across rounds.
__global__ void __launch_bounds__(1024) k_scan_exclusive(uint32_t *hist) {
    __shared__ uint32_t warp_sums[32];
    __shared__ uint32_t carry_s;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid == 0) carry_s = 0;
    __syncthreads();
    for (int base = 0; base < MORTON_BUCKETS; base += 4096) {
        uint4 v = reinterpret_cast<uint4 *>(hist + base)[tid];
        const uint32_t s1 = v.x, s2 = s1 + v.y, s3 = s2 + v.z, s4 = s3 + v.w;
        uint32_t incl = s4;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) warp_sums[wid] = incl;
        __syncthreads();
        if (wid == 0) {
            uint32_t w = warp_sums[lane], wi = w;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, wi, o);
                if (lane >= o) wi += t;
            }
            warp_sums[lane] = wi - w;  // exclusive prefix of warp totals
        }
        __syncthreads();
        const uint32_t carry = carry_s;
        const uint32_t excl = carry + warp_sums[wid] + (incl - s4);
        reinterpret_cast<uint4 *>(hist + base)[tid] = make_uint4(excl, excl + s1, excl + s2, excl + s3);
        __syncthreads();
        if (tid == 1023) carry_s = excl + s4;
        __syncthreads();
    }
}

__global__ void k_morton_scatter(MortonParams p) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= p.n) return;
    const uint32_t pos = atomicAdd(p.hist + p.key[i], 1u);
    p.perm[pos] = i;
}

cudaError_t launch_morton_prepass(const MortonParams &p, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(p.hist, 0, sizeof(uint32_t) * MORTON_BUCKETS, s);
    if (e != cudaSuccess) return e;
    const int g = (p.n + 255) / 256;
    k_morton_hist<<<g, 256, 0, s>>>(p);
    k_scan_exclusive<<<1, 1024, 0, s>>>(p.hist);
    k_morton_scatter<<<g, 256, 0, s>>>(p);
    return cudaGetLastError();
}

// ----------------------------------------------------------------------------------------
// a1-a8: the classify kernel
//
// CTA = NCW consumer warps (one fiber per lane) + 1 producer warp that streams the CTA's listed
// atlas tiles (64-B header + [21][32] float4 points) through a STAGES-deep shared-memory ring
// with 1-D TMA bulk copies (cp.async.bulk -> UBLKCP), completion on mbarriers.
// Per listed tile and consumer warp:
//   a2  exact sphere lower bound per lane (points 0/10/20 vs the tile's spheres), warp ballot;
//   a3  test1, dense and transposed: lane c holds centroid c's point 10 and the warp walks its
//       passing fibers; one ballot per fiber gives that fiber's survivors against its cutoff
//       tau = min(thr_b^2, best^2), pushed straight into a small queue q1;
//   a4  test2, compacted: q1 is processed 32 entries at a time with every lane busy: end points
//       in both orientations; each orientation still under tau goes to queue q2 with its max;
//   a5/a6 test3 + test4, compacted: q2 entries are processed 32 at a time: points {3,17,7,13},
//       then the rest with an early exit after every group;
//   a7  a finished orientation updates its fiber's best (d^2, bundle) key with a shared-memory
//       64-bit atomicMin (lexicographic, so tile order and orientation never matter).
// Fiber coordinates live in shared memory (per warp: xy plane float2 [21][32] + z plane float
// [21][32]) so any lane can process any lane's candidate; points 0/10/20 also stay in registers.
// ----------------------------------------------------------------------------------------
constexpr int NCW = 4;                 // consumer warps
constexpr int FPC = NCW * 32;          // fibers per CTA
constexpr int NTHREADS = FPC + 32;     // + producer warp
constexpr int STAGES = 3;              // tile ring depth
constexpr int FB = 4;                  // fibers per step of the transposed test1 loop
constexpr int Q1CAP = 32 + FB * 32;    // < 32 carried + up to 32 pushed per fiber of a step
constexpr int Q2CAP = 96;              // < 32 carried + up to 64 pushed per q1 round
constexpr uint32_t SLEEP_NS = 1000000; // mbarrier try_wait suspend-time hint
constexpr unsigned long long KEY_NONE = ~0ull;

enum {
    ST_FIBERS = 0, ST_WT_LISTED, ST_WT_COMPUTED, ST_LT_PASS, ST_T1, ST_T2, ST_T34, ST_FULL, ST_UPD,
    ST_PDIST, ST_SPHERE, ST_CTAS, ST_N
};

struct SmemLayout {
    size_t ring, fxy, fz, q1, q2e, q2r, best, bars, tbits, bbits, total;
    __host__ __device__ SmemLayout(int B, int T) {
        size_t o = 0;
        ring = o; o += (size_t)STAGES * TILE_STRIDE_BYTES;
        fxy = o;  o += (size_t)NCW * NPTS * 32 * sizeof(float2);
        fz = o;   o += (size_t)NCW * NPTS * 32 * sizeof(float);
        best = o; o += (size_t)NCW * 32 * sizeof(unsigned long long);
        bars = o; o += 2 * STAGES * sizeof(uint64_t);
        q2e = o;  o += (size_t)NCW * Q2CAP * sizeof(uint32_t);
        q2r = o;  o += (size_t)NCW * Q2CAP * sizeof(float);
        q1 = o;   o += (size_t)NCW * Q1CAP * sizeof(uint16_t);
        tbits = o; o += sizeof(uint32_t) * (size_t)((T + 31) >> 5);
        bbits = o; o += sizeof(uint32_t) * (size_t)((B + 31) >> 5);
        total = (o + 127) & ~(size_t)127;
    }
};

__device__ __forceinline__ void mbar_sleep_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAITS_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@!P1 bra WAITS_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(SLEEP_NS)
        : "memory");
}

__device__ __forceinline__ float key_d2(unsigned long long k) { return __uint_as_float((uint32_t)(k >> 32)); }

// a2: exact tile lower bound: for every centroid c of the tile,
// d_ME >= |f10 - c10| >= |f10 - C10| - R10 and d_ME >= min over orientations of the end-point
// maximum, each term bounded the same way.  Skip iff the bound exceeds s = sqrt(tau) + CULL_EPS.
__device__ __forceinline__ bool tile_may_pass(const float3 &f0, const float3 &f10, const float3 &f20,
                                              const TileHdr &h, float s) {
    const float r0 = h.s0.w + s, r10 = h.s10.w + s, r20 = h.s20.w + s;
    const float a0 = r0 * r0, a10 = r10 * r10, a20 = r20 * r20;
    const bool p10 = d2(f10.x, f10.y, f10.z, h.s10) <= a10;
    const bool pdir = d2(f0.x, f0.y, f0.z, h.s0) <= a0 && d2(f20.x, f20.y, f20.z, h.s20) <= a20;
    const bool pinv = d2(f0.x, f0.y, f0.z, h.s20) <= a20 && d2(f20.x, f20.y, f20.z, h.s0) <= a0;
    return p10 && (pdir || pinv);
}

template <bool STATS>
__global__ void __launch_bounds__(NTHREADS, 3) k_classify(ClassifyParams p) {
    extern __shared__ __align__(128) unsigned char smem[];
    const SmemLayout L(p.B, p.T);
    float4 *ring = reinterpret_cast<float4 *>(smem + L.ring);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + L.bars);
    uint64_t *empty = full + STAGES;
    uint32_t *tbits = reinterpret_cast<uint32_t *>(smem + L.tbits);
    uint32_t *bbits = reinterpret_cast<uint32_t *>(smem + L.bbits);
    const int twords = (p.T + 31) >> 5;
    const int bwords = (p.B + 31) >> 5;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool consumer = warp < NCW;
    const int cw = consumer ? warp : 0;
    float2 *fxy = reinterpret_cast<float2 *>(smem + L.fxy) + cw * (NPTS * 32);   // [21][32]
    float *fz = reinterpret_cast<float *>(smem + L.fz) + cw * (NPTS * 32);       // [21][32]
    unsigned long long *best = reinterpret_cast<unsigned long long *>(smem + L.best) + cw * 32;
    uint16_t *q1 = reinterpret_cast<uint16_t *>(smem + L.q1) + cw * Q1CAP;
    uint32_t *q2e = reinterpret_cast<uint32_t *>(smem + L.q2e) + cw * Q2CAP;
    float *q2r = reinterpret_cast<float *>(smem + L.q2r) + cw * Q2CAP;

    for (int i = threadIdx.x; i < twords + bwords; i += NTHREADS) tbits[i] = 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, NCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }

    // ---- a1: fiber ingest: 63 floats -> smem planes; points 0/10/20 kept in registers ----
    const int gi = blockIdx.x * FPC + warp * 32 + lane;
    const bool inrange = consumer && gi < p.n;
    const int fidx = inrange ? (p.perm ? __ldg(p.perm + gi) : gi) : 0;
    bool finite = inrange;
    float3 f0 = make_float3(0.f, 0.f, 0.f), f10 = f0, f20 = f0;
    if (consumer) {
        const float *src = p.fibers + (size_t)fidx * (3 * NPTS);
#pragma unroll
        for (int i = 0; i < NPTS; ++i) {
            float x = 0.f, y = 0.f, z = 0.f;
            if (inrange) {
                x = __ldg(src + 3 * i);
                y = __ldg(src + 3 * i + 1);
                z = __ldg(src + 3 * i + 2);
            }
            finite = finite && isfinite(x) && isfinite(y) && isfinite(z);
            fxy[i * 32 + lane] = make_float2(x, y);
            fz[i * 32 + lane] = z;
            if (i == 0) f0 = make_float3(x, y, z);
            if (i == 10) f10 = make_float3(x, y, z);
            if (i == 20) f20 = make_float3(x, y, z);
        }
        best[lane] = (p.seed && inrange) ? p.seed[fidx] : KEY_NONE;
    }
    unsigned long long cnt[ST_N];
    if (STATS) {
#pragma unroll
        for (int k = 0; k < ST_N; ++k) cnt[k] = 0;
        cnt[ST_FIBERS] = inrange ? 1 : 0;
        cnt[ST_CTAS] = threadIdx.x == 0 ? 1 : 0;
    }
    __syncthreads();

    // ---- a2 (pre-pass): CTA candidate list from the threshold-only bound ----
    if (consumer) {
        for (int b0 = 0; b0 < p.B; b0 += 32) {
            uint32_t m = 0;
#pragma unroll 4
            for (int j = 0; j < 32; ++j) {
                const int b = b0 + j;
                if (b < p.B) {
                    const BundleHdr h = p.bh[b];
                    const float r = h.s10.w + h.thr + CULL_EPS;
                    const bool pass = h.t1 > h.t0 && finite && d2(f10.x, f10.y, f10.z, h.s10) <= r * r;
                    m |= (pass ? 1u : 0u) << j;
                }
            }
            if (STATS && finite) { cnt[ST_SPHERE] += min(32, p.B - b0); cnt[ST_PDIST] += min(32, p.B - b0); }
            m = __reduce_or_sync(0xffffffffu, m);
            if (lane == 0 && m) atomicOr(bbits + (b0 >> 5), m);
        }
    }
    __syncthreads();
    if (consumer) {
        for (int w = 0; w < bwords; ++w) {
            uint32_t bits = bbits[w];
            while (bits) {
                const int b = (w << 5) + __ffs(bits) - 1;
                bits &= bits - 1;
                const BundleHdr h = p.bh[b];
                const float s = h.thr + CULL_EPS;
                const float r = h.s10.w + s;
                const bool bpass = finite && d2(f10.x, f10.y, f10.z, h.s10) <= r * r;
                if (!__any_sync(0xffffffffu, bpass)) continue;
                for (int t0 = h.t0; t0 < h.t1; t0 += 32) {
                    uint32_t m = 0;
                    const int nt = min(32, h.t1 - t0);
#pragma unroll 4
                    for (int j = 0; j < 32; ++j) {
                        if (j < nt) {
                            const TileHdr th = p.th[t0 + j];
                            m |= (bpass && tile_may_pass(f0, f10, f20, th, s) ? 1u : 0u) << j;
                        }
                    }
                    if (STATS && bpass) { cnt[ST_SPHERE] += nt; cnt[ST_PDIST] += 5 * nt; }
                    m = __reduce_or_sync(0xffffffffu, m);
                    if (lane == 0 && m) {
                        // tiles t0..t0+nt-1 -> bit positions; may straddle two words
                        const int w0 = t0 >> 5, sh = t0 & 31;
                        atomicOr(tbits + w0, m << sh);
                        if (sh && (m >> (32 - sh))) atomicOr(tbits + w0 + 1, m >> (32 - sh));
                    }
                }
            }
        }
    }
    __syncthreads();

    if (!consumer) {
        // ---- producer warp: TMA bulk copies of the listed tiles into the ring ----
        if (lane == 0) {
            int k = 0;
            for (int w = 0; w < twords; ++w) {
                uint32_t bits = tbits[w];
                while (bits) {
                    const int t = (w << 5) + __ffs(bits) - 1;
                    bits &= bits - 1;
                    const int s = k % STAGES, u = k / STAGES;
                    if (u > 0) mbar_sleep_wait(empty + s, (u - 1) & 1);
                    mbar_arrive_expect_tx(full + s, TILE_STRIDE_BYTES);
                    bulk_g2s(ring + s * TILE_STRIDE_F4, p.tiles + (size_t)t * TILE_STRIDE_F4, TILE_STRIDE_BYTES,
                             full + s);
                    ++k;
                }
            }
        }
        return;
    }

    const uint32_t lt_mask = (1u << lane) - 1u;
    int k = 0;
    for (int w = 0; w < twords; ++w) {
        uint32_t bits = tbits[w];
        while (bits) {
            bits &= bits - 1;
            const int s = k % STAGES, u = k / STAGES;
            ++k;
            mbar_sleep_wait(full + s, u & 1);
            const float4 *stage = ring + s * TILE_STRIDE_F4;
            const TileHdr th = *reinterpret_cast<const TileHdr *>(stage);
            const float4 *T = stage + TILE_HDR_F4;
            const float thr2 = th.thr2;
            const int b = th.bundle;
            const float tau = fminf(thr2, key_d2(best[lane]));
            const bool pass = finite && tile_may_pass(f0, f10, f20, th, sqrtf(tau) + CULL_EPS);
            if (STATS) {
                if (lane == 0) cnt[ST_WT_LISTED]++;
                if (finite) { cnt[ST_SPHERE]++; cnt[ST_PDIST] += 5; }
            }
            if (__any_sync(0xffffffffu, pass)) {
                if (STATS) {
                    if (lane == 0) cnt[ST_WT_COMPUTED]++;
                    if (pass) { cnt[ST_LT_PASS]++; cnt[ST_T1] += TILE; cnt[ST_PDIST] += TILE; }
                }
                // ---- q2 round: test3 + test4 on entries [base, base + cnt2) ----
                auto run_q2 = [&](int base, int cnt2) {
                    if (lane < cnt2) {
                        const uint32_t e = q2e[base + lane];
                        float r = q2r[base + lane];
                        const int fl = (e >> 5) & 31, c = e & 31, o = (e >> 10) & 1;
                        const float taul = fminf(thr2, key_d2(best[fl]));
                        const float4 *cb = T + c + (o ? 20 * TILE : 0);
                        const int st = o ? -TILE : TILE;
                        bool done = false;
#define SEG_STEP(i)                                                             \
    {                                                                           \
        const float2 a = fxy[(i) * 32 + fl];                                    \
        r = fmaxf(r, d2(a.x, a.y, fz[(i) * 32 + fl], cb[(i) * st]));            \
    }
                        if (STATS) cnt[ST_T34]++;
                        SEG_STEP(3); SEG_STEP(17); SEG_STEP(7); SEG_STEP(13);
                        if (STATS) cnt[ST_PDIST] += 4;
                        if (r > taul) done = true;
                        if (!done) {
                            SEG_STEP(10); SEG_STEP(1); SEG_STEP(19); SEG_STEP(2);
                            if (STATS) cnt[ST_PDIST] += 4;
                            if (r > taul) done = true;
                        }
                        if (!done) {
                            SEG_STEP(18); SEG_STEP(4); SEG_STEP(16); SEG_STEP(5);
                            if (STATS) cnt[ST_PDIST] += 4;
                            if (r > taul) done = true;
                        }
                        if (!done) {
                            SEG_STEP(15); SEG_STEP(6); SEG_STEP(14); SEG_STEP(8); SEG_STEP(12);
                            SEG_STEP(9); SEG_STEP(11);
                            if (STATS) { cnt[ST_PDIST] += 7; cnt[ST_FULL]++; }
                            // a7: lexicographic (d^2, bundle) minimum
                            if (r <= thr2) {
                                atomicMin(best + fl, ((unsigned long long)__float_as_uint(r) << 32) | (uint32_t)b);
                                if (STATS) cnt[ST_UPD]++;
                            }
                        }
#undef SEG_STEP
                    }
                    __syncwarp();
                };

                // ---- q1 round: test2 on entries [base, base + cnt1), survivors pushed to q2 ----
                int n2 = 0;
                auto run_q1 = [&](int base, int cnt1) {
                    bool ad = false, ai = false;
                    uint32_t e = 0;
                    float rd = 0.f, ri = 0.f;
                    if (lane < cnt1) {
                        e = q1[base + lane];
                        const int fl = e >> 5, c = e & 31;
                        const float taul = fminf(thr2, key_d2(best[fl]));
                        const float2 a0 = fxy[fl], a20 = fxy[20 * 32 + fl];
                        const float z0 = fz[fl], z20 = fz[20 * 32 + fl];
                        const float4 c0 = T[c], c20 = T[20 * TILE + c];
                        const float e00 = d2(a0.x, a0.y, z0, c0), e2020 = d2(a20.x, a20.y, z20, c20);
                        const float e020 = d2(a0.x, a0.y, z0, c20), e200 = d2(a20.x, a20.y, z20, c0);
                        rd = fmaxf(e00, e2020);
                        ri = fmaxf(e020, e200);
                        ad = rd <= taul;
                        ai = ri <= taul;
                        if (STATS) { cnt[ST_T2]++; cnt[ST_PDIST] += 4; }
                    }
                    const uint32_t bd = __ballot_sync(0xffffffffu, ad), bi = __ballot_sync(0xffffffffu, ai);
                    if (ad) {
                        const int pos = n2 + __popc(bd & lt_mask);
                        q2e[pos] = e;
                        q2r[pos] = rd;
                    }
                    if (ai) {
                        const int pos = n2 + __popc(bd) + __popc(bi & lt_mask);
                        q2e[pos] = e | (1u << 10);
                        q2r[pos] = ri;
                    }
                    n2 += __popc(bd) + __popc(bi);
                    __syncwarp();
                    while (n2 >= 32) {
                        n2 -= 32;
                        run_q2(n2, 32);
                    }
                };

                // ---- a3, test1 (dense, transposed): lane c holds centroid c's point 10; the warp
                // walks its passing fibers j (broadcast point 10 from smem) and one ballot per
                // fiber yields that fiber's survivor set, pushed straight into q1 ----
                const float4 cc10 = T[10 * TILE + lane];
                uint32_t pm = __ballot_sync(0xffffffffu, pass);
                int n1 = 0;
                while (pm) {
                    // up to FB fibers per step: independent distance chains for ILP
                    int jj[FB];
                    bool ok[FB];
#pragma unroll
                    for (int q = 0; q < FB; ++q) {
                        jj[q] = pm ? __ffs(pm) - 1 : -1;
                        pm &= pm - 1;
                    }
#pragma unroll
                    for (int q = 0; q < FB; ++q) {
                        const int j = jj[q] < 0 ? 0 : jj[q];
                        const float2 a = fxy[10 * 32 + j];
                        const float m10 = d2(a.x, a.y, fz[10 * 32 + j], cc10);
                        ok[q] = jj[q] >= 0 && m10 <= __shfl_sync(0xffffffffu, tau, j);
                    }
#pragma unroll
                    for (int q = 0; q < FB; ++q) {
                        const uint32_t bal = __ballot_sync(0xffffffffu, ok[q]);
                        if (ok[q]) q1[n1 + __popc(bal & lt_mask)] = (uint16_t)((jj[q] << 5) | lane);
                        n1 += __popc(bal);
                    }
                    __syncwarp();
                    while (n1 >= 32) {
                        n1 -= 32;
                        run_q1(n1, 32);
                    }
                }
                __syncwarp();
                if (n1 > 0) run_q1(0, n1);
                if (n2 > 0) run_q2(0, n2);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + s);
        }
    }

    // ---- a8: epilogue ----
    if (inrange) {
        const unsigned long long key = best[lane];
        int lab;
        float dd;
        if (!finite) {
            lab = -1;
            dd = __int_as_float(0x7fffffff);  // NaN
        } else if (key != KEY_NONE) {
            lab = (int)(uint32_t)(key & 0xffffffffu);
            dd = __fsqrt_rn(key_d2(key));
        } else {
            lab = -1;
            dd = INFINITY;
        }
        p.label[fidx] = lab;
        p.dist[fidx] = dd;
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

size_t classify_smem_bytes(int B, int T) { return SmemLayout(B, T).total; }

int classify_fibers_per_cta() { return FPC; }

cudaError_t launch_classify(const ClassifyParams &p, bool stats, cudaStream_t s) {
    if (p.n <= 0) return cudaSuccess;
    const size_t smem = classify_smem_bytes(p.B, p.T);
    const int grid = (p.n + FPC - 1) / FPC;
    cudaError_t e;
    if (stats) {
        e = cudaFuncSetAttribute(k_classify<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        k_classify<true><<<grid, NTHREADS, smem, s>>>(p);
    } else {
        e = cudaFuncSetAttribute(k_classify<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        k_classify<false><<<grid, NTHREADS, smem, s>>>(p);
    }
    return cudaGetLastError();
}

}  // namespace seg
