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
// ----------------------------------------------------------------------------------------
constexpr int NCW = 4;                 // consumer warps (one fiber per lane)
constexpr int FPC = NCW * 32;          // fibers per CTA
constexpr int NTHREADS = FPC + 32;     // + one producer warp (TMA issue)
constexpr int STAGES = 4;              // smem ring depth (4 x 10.5 KB)

enum {
    ST_FIBERS = 0, ST_WT_LISTED, ST_WT_COMPUTED, ST_LT_PASS, ST_T1, ST_T2, ST_T34, ST_FULL, ST_UPD,
    ST_PDIST, ST_SPHERE, ST_CTAS, ST_N
};

// Tile lower bound (a2).  For every centroid c of a tile, d_ME(f, c) >= |f10 - c10| and
// d_ME(f, c) >= min over orientations of the end-point maximum; each |f_p - c_q| is bounded
// below by |f_p - C_q| - R_q with (C_q, R_q) the tile's bounding sphere of point q.  The tile
// can be skipped iff that bound exceeds s = sqrt(tau) + CULL_EPS; tested on squares.
__device__ __forceinline__ bool tile_may_pass(const float (&f)[3 * NPTS], const TileHdr &h, float s) {
    const float r0 = h.s0.w + s, r10 = h.s10.w + s, r20 = h.s20.w + s;
    const float a0 = r0 * r0, a10 = r10 * r10, a20 = r20 * r20;
    const bool p10 = d2(f[30], f[31], f[32], h.s10) <= a10;
    const bool pdir = d2(f[0], f[1], f[2], h.s0) <= a0 && d2(f[60], f[61], f[62], h.s20) <= a20;
    const bool pinv = d2(f[0], f[1], f[2], h.s20) <= a20 && d2(f[60], f[61], f[62], h.s0) <= a0;
    return p10 && (pdir || pinv);
}

template <bool STATS>
__global__ void __launch_bounds__(NTHREADS, 3) k_classify(ClassifyParams p) {
    extern __shared__ __align__(128) unsigned char smem[];
    float4 *ring = reinterpret_cast<float4 *>(smem);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + STAGES * TILE_BYTES);
    uint64_t *empty = full + STAGES;
    uint32_t *tbits = reinterpret_cast<uint32_t *>(empty + STAGES);
    const int twords = (p.T + 31) >> 5;
    const int bwords = (p.B + 31) >> 5;
    uint32_t *bbits = tbits + twords;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < twords + bwords; i += NTHREADS) tbits[i] = 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, NCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }

    // ---- a1: fiber ingest (one fiber per consumer lane, 63 floats in registers) ----
    const bool consumer = warp < NCW;
    const int gi = blockIdx.x * FPC + warp * 32 + lane;
    const bool inrange = consumer && gi < p.n;
    const int fidx = inrange ? (p.perm ? __ldg(p.perm + gi) : gi) : 0;
    float f[3 * NPTS];
    bool finite = inrange;
    {
        const float *src = p.fibers + (size_t)fidx * (3 * NPTS);
#pragma unroll
        for (int k = 0; k < 3 * NPTS; ++k) {
            f[k] = inrange ? __ldg(src + k) : 0.f;
            finite = finite && isfinite(f[k]);
        }
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
        for (int b = 0; b < p.B; ++b) {
            const BundleHdr h = p.bh[b];
            bool pass = false;
            if (h.t1 > h.t0 && finite) {
                const float r = h.s10.w + h.thr + CULL_EPS;
                pass = d2(f[30], f[31], f[32], h.s10) <= r * r;
                if (STATS) { cnt[ST_SPHERE]++; cnt[ST_PDIST]++; }
            }
            if (__any_sync(0xffffffffu, pass) && lane == 0) atomicOr(bbits + (b >> 5), 1u << (b & 31));
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
                const bool bpass = finite && d2(f[30], f[31], f[32], h.s10) <= r * r;
                if (!__any_sync(0xffffffffu, bpass)) continue;
                for (int t = h.t0; t < h.t1; ++t) {
                    const TileHdr th = p.th[t];
                    const bool pass = bpass && tile_may_pass(f, th, s);
                    if (STATS && bpass) { cnt[ST_SPHERE]++; cnt[ST_PDIST] += 5; }
                    if (__any_sync(0xffffffffu, pass) && lane == 0) atomicOr(tbits + (t >> 5), 1u << (t & 31));
                }
            }
        }
    }
    __syncthreads();

    if (!consumer) {
        // ---- producer warp: stream the listed tiles through the ring with TMA bulk copies ----
        if (lane == 0) {
            int k = 0;
            for (int w = 0; w < twords; ++w) {
                uint32_t bits = tbits[w];
                while (bits) {
                    const int t = (w << 5) + __ffs(bits) - 1;
                    bits &= bits - 1;
                    const int s = k % STAGES, u = k / STAGES;
                    if (u > 0) mbar_wait(empty + s, (u - 1) & 1);
                    mbar_arrive_expect_tx(full + s, TILE_BYTES);
                    bulk_g2s(ring + s * TILE_F4, p.tiles + (size_t)t * TILE_F4, TILE_BYTES, full + s);
                    ++k;
                }
            }
        }
        return;
    }

    // ---- consumers: a2 (tight bound) .. a7 per listed tile ----
    float best2 = INFINITY;
    int bestb = INT_MAX;
    int k = 0;
    for (int w = 0; w < twords; ++w) {
        uint32_t bits = tbits[w];
        while (bits) {
            const int t = (w << 5) + __ffs(bits) - 1;
            bits &= bits - 1;
            const int s = k % STAGES, u = k / STAGES;
            ++k;
            const TileHdr th = p.th[t];
            const float thr2 = th.thr2;
            const int b = th.bundle;
            float tau = fminf(thr2, best2);
            const bool pass = finite && tile_may_pass(f, th, sqrtf(tau) + CULL_EPS);
            if (STATS) {
                if (lane == 0) cnt[ST_WT_LISTED]++;
                if (finite) { cnt[ST_SPHERE]++; cnt[ST_PDIST] += 5; }
            }
            mbar_wait(full + s, u & 1);
            if (__any_sync(0xffffffffu, pass)) {
                const float4 *T = ring + s * TILE_F4;
                if (STATS) {
                    if (lane == 0) cnt[ST_WT_COMPUTED]++;
                    if (pass) { cnt[ST_LT_PASS]++; cnt[ST_T1] += TILE; cnt[ST_PDIST] += TILE; }
                }
                // a3, test1: centre point of all 32 centroids ("first only the center point")
                uint32_t mask = 0;
#pragma unroll 8
                for (int c = 0; c < TILE; ++c) {
                    const float m10 = d2(f[30], f[31], f[32], T[10 * TILE + c]);
                    mask |= (m10 <= tau ? 1u : 0u) << c;
                }
                if (!pass) mask = 0;
                // a4-a7 for every surviving centroid of this lane
                while (mask) {
                    const int c = __ffs(mask) - 1;
                    mask &= mask - 1;
                    const float4 *q = T + c;
                    tau = fminf(thr2, best2);
                    // a4, test2: end points in both orientations
                    const float m10 = d2(f[30], f[31], f[32], q[10 * TILE]);
                    const float e00 = d2(f[0], f[1], f[2], q[0]);
                    const float e2020 = d2(f[60], f[61], f[62], q[20 * TILE]);
                    const float e020 = d2(f[0], f[1], f[2], q[20 * TILE]);
                    const float e200 = d2(f[60], f[61], f[62], q[0]);
                    const float rdir = fmaxf(fmaxf(e00, e2020), m10);
                    const float rinv = fmaxf(fmaxf(e020, e200), m10);
                    const bool adir = rdir <= tau, ainv = rinv <= tau;
                    if (STATS) { cnt[ST_T2]++; cnt[ST_PDIST] += 5; }
                    if (!(adir || ainv)) continue;
                    float r;
                    if (adir && ainv) {
                        // both orientations alive (rare): exact Eq. 2, both maxima in full
                        float rd = rdir, ri = rinv;
#pragma unroll
                        for (int i = 1; i < NPTS - 1; ++i) {
                            if (i == 10) continue;
                            rd = fmaxf(rd, d2(f[3 * i], f[3 * i + 1], f[3 * i + 2], q[i * TILE]));
                            ri = fmaxf(ri, d2(f[3 * i], f[3 * i + 1], f[3 * i + 2], q[(20 - i) * TILE]));
                        }
                        r = fminf(rd, ri);
                        if (STATS) { cnt[ST_T34] += 2; cnt[ST_FULL] += 2; cnt[ST_PDIST] += 36; }
                    } else {
                        // one orientation: centroid point paired with fiber point i is i (direct)
                        // or 20 - i (inverse); test3 = points {3, 17, 7, 13}, then test4 with an
                        // early exit after every group
                        const float4 *cb = adir ? q : q + 20 * TILE;
                        const int st = adir ? TILE : -TILE;
                        r = adir ? rdir : rinv;
#define SEG_STEP(i) r = fmaxf(r, d2(f[3 * (i)], f[3 * (i) + 1], f[3 * (i) + 2], cb[(i) * st]))
                        if (STATS) cnt[ST_T34]++;
                        SEG_STEP(3); SEG_STEP(17); SEG_STEP(7); SEG_STEP(13);
                        if (STATS) cnt[ST_PDIST] += 4;
                        if (r > tau) continue;
                        SEG_STEP(1); SEG_STEP(19); SEG_STEP(2); SEG_STEP(18);
                        if (STATS) cnt[ST_PDIST] += 4;
                        if (r > tau) continue;
                        SEG_STEP(4); SEG_STEP(16); SEG_STEP(5); SEG_STEP(15);
                        if (STATS) cnt[ST_PDIST] += 4;
                        if (r > tau) continue;
                        SEG_STEP(6); SEG_STEP(14); SEG_STEP(8); SEG_STEP(12); SEG_STEP(9); SEG_STEP(11);
                        if (STATS) { cnt[ST_PDIST] += 6; cnt[ST_FULL]++; }
#undef SEG_STEP
                    }
                    // a7: closest bundle, lexicographic (d^2, bundle) so tile order never matters
                    if (r <= thr2 && (r < best2 || (r == best2 && b < bestb))) {
                        best2 = r;
                        bestb = b;
                        if (STATS) cnt[ST_UPD]++;
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + s);
        }
    }

    // ---- a8: epilogue ----
    if (inrange) {
        int lab;
        float dd;
        if (!finite) {
            lab = -1;
            dd = __int_as_float(0x7fffffff);  // NaN
        } else if (bestb != INT_MAX) {
            lab = bestb;
            dd = __fsqrt_rn(best2);
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

size_t classify_smem_bytes(int B, int T) {
    return (size_t)STAGES * TILE_BYTES + 2 * STAGES * sizeof(uint64_t) +
           sizeof(uint32_t) * (size_t)(((T + 31) >> 5) + ((B + 31) >> 5));
}

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
