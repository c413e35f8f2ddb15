// group.cu -- row f3: the segmented bundles.  After seg_classify, the fibers
// grouped by label ("segmented bundles", PAPER.md:58 / Fig. 1B): a STABLE partition of the fiber
// indices by bundle (bundles in id order, unassigned fibers last), per-bundle offsets, and per-bundle
// distance summaries (min, max, sum).
//
// A three-kernel counting sort, HBM-bound (labels and distances read twice, the order written once):
//   kg_count   per block of GB fibers, a histogram of the labels (shared-memory atomics) plus the
//              per-bundle min / max / sum of the distances; written label-major hist[l][blk]
//   kg_scan    one warp per label: exclusive scan of hist[l][*] over the blocks (coalesced), the
//              label totals; then one warp: exclusive scan of the totals over the labels -> offsets
//   kg_scatter per block, its fibers in order, 256 at a time: within a warp the rank among equal
//              labels from __match_any_sync, across the block's warps a prefix in shared memory, so
//              the position keeps the fiber order inside every bundle (stable)
#include <cfloat>
#include <cstdint>

#include "seg_internal.cuh"

namespace seg {

constexpr int GB = 2048;        // fibers per block of kg_count / kg_scatter
constexpr int GT = 256;         // threads per block
constexpr int GW = GT / 32;     // warps per block

// label -> bin: bundles 0..B-1, everything else (unassigned -1, out of range) -> bin B
__device__ __forceinline__ int bin_of(int32_t lab, int B) { return (lab >= 0 && lab < B) ? lab : B; }

__global__ void __launch_bounds__(GT) kg_count(GroupParams p) {
    extern __shared__ uint32_t gsm[];
    const int nb = p.B + 1;
    uint32_t *cnt = gsm;                                   // [nb]
    uint32_t *mn = cnt + nb, *mx = mn + nb;                // [nb] float bits (distances >= 0)
    double *sm = reinterpret_cast<double *>(gsm + ((3 * nb + 1) & ~1));   // [nb], 8-B aligned
    for (int i = threadIdx.x; i < nb; i += GT) {
        cnt[i] = 0;
        mn[i] = 0x7f800000u;   // +inf
        mx[i] = 0u;
        sm[i] = 0.0;
    }
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * GB;
    for (int k = threadIdx.x; k < GB; k += GT) {
        const int64_t i = base + k;
        if (i >= p.n) break;
        const int bn = bin_of(__ldg(p.label + i), p.B);
        atomicAdd(cnt + bn, 1u);
        if (bn < p.B && p.dist) {
            const float d = __ldg(p.dist + i);
            atomicMin(mn + bn, __float_as_uint(d));
            atomicMax(mx + bn, __float_as_uint(d));
            atomicAdd(sm + bn, (double)d);
        }
    }
    __syncthreads();
    for (int l = threadIdx.x; l < nb; l += GT) {
        p.hist[(size_t)l * p.nblk + blockIdx.x] = cnt[l];
        if (l < p.B && p.dist && cnt[l]) {
            atomicMin(p.gmin + l, mn[l]);
            atomicMax(p.gmax + l, mx[l]);
            atomicAdd(p.dsum + l, sm[l]);
        }
    }
}

__global__ void kg_init(GroupParams p) {
    const int l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l < p.B) {
        p.gmin[l] = 0x7f800000u;   // +inf: an empty bundle keeps it
        p.gmax[l] = 0u;
        p.dsum[l] = 0.0;
    }
}

// one warp per label: hist[l][*] -> exclusive prefix over the blocks (in place), total[l]
__global__ void kg_scan_blocks(GroupParams p) {
    const int lane = threadIdx.x & 31;
    const int l = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (l > p.B) return;
    uint32_t *h = p.hist + (size_t)l * p.nblk;
    uint32_t carry = 0;
    for (int b0 = 0; b0 < p.nblk; b0 += 32) {
        const int b = b0 + lane;
        const uint32_t v = b < p.nblk ? h[b] : 0u;
        uint32_t incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (b < p.nblk) h[b] = carry + incl - v;
        carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) p.total[l] = carry;
}

// one warp: offsets[l] = exclusive prefix of the totals over the labels (int64), offsets[B+1] = N;
// the summaries of empty bundles are normalised (min = max = +inf / 0 already; sum 0)
__global__ void kg_scan_labels(GroupParams p) {
    const int lane = threadIdx.x;
    long long carry = 0;
    for (int l0 = 0; l0 <= p.B; l0 += 32) {
        const int l = l0 + lane;
        const long long v = l <= p.B ? (long long)p.total[l] : 0;
        long long incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (l <= p.B) p.offsets[l] = carry + incl - v;
        carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) p.offsets[p.B + 1] = carry;
}

__global__ void __launch_bounds__(GT) kg_scatter(GroupParams p) {
    extern __shared__ uint32_t gsm[];
    const int nb = p.B + 1;
    uint32_t *wcnt = gsm;                 // [GW][nb] this round's per-warp counts, then their prefix
    uint32_t *run = wcnt + GW * nb;       // [nb] block offset of each label so far (global position)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    for (int l = threadIdx.x; l < nb; l += GT)
        run[l] = (uint32_t)(p.offsets[l] + p.hist[(size_t)l * p.nblk + blockIdx.x]);
    const int64_t base = (int64_t)blockIdx.x * GB;
    for (int r = 0; r < GB; r += GT) {
        for (int i = threadIdx.x; i < GW * nb; i += GT) wcnt[i] = 0;
        __syncthreads();
        const int64_t i = base + r + threadIdx.x;   // warp w holds fibers r + 32w .. r + 32w + 31, in order
        const bool ok = i < p.n;
        const int bn = ok ? bin_of(__ldg(p.label + i), p.B) : nb;   // nb: no fiber
        const uint32_t peers = __match_any_sync(0xffffffffu, bn);
        const uint32_t rank = __popc(peers & lt);
        if (ok && rank == 0) wcnt[warp * nb + bn] = __popc(peers);
        __syncthreads();
        for (int l = threadIdx.x; l < nb; l += GT) {   // exclusive prefix over the warps, per label
            uint32_t s = run[l];
            for (int w = 0; w < GW; ++w) {
                const uint32_t c = wcnt[w * nb + l];
                wcnt[w * nb + l] = s;
                s += c;
            }
            run[l] = s;
        }
        __syncthreads();
        SEG_DCHECK(!ok || (int64_t)wcnt[warp * nb + bn] + rank < p.n);
        if (ok) p.order[wcnt[warp * nb + bn] + rank] = (int32_t)i;
        __syncthreads();
    }
}

size_t group_scratch_words(int64_t n, int B) {
    const int64_t nblk = (n + GB - 1) / GB;
    return (size_t)(B + 1) * (size_t)nblk + (size_t)(B + 1);   // hist[B+1][nblk], total[B+1]
}

cudaError_t launch_group(GroupParams p, cudaStream_t s) {
    p.nblk = (int)((p.n + GB - 1) / GB);
    const int nb = p.B + 1;
    const size_t smem_count = sizeof(uint32_t) * (size_t)((3 * nb + 1) & ~1) + sizeof(double) * (size_t)nb;
    const size_t smem_scatter = sizeof(uint32_t) * (size_t)(GW + 1) * nb;
    cudaError_t e;
    if (p.summ) kg_init<<<(p.B + 255) / 256, 256, 0, s>>>(p);
    if (p.n > 0) {
        e = cudaFuncSetAttribute(kg_count, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_count);
        if (e != cudaSuccess) return e;
        kg_count<<<p.nblk, GT, smem_count, s>>>(p);
        kg_scan_blocks<<<(nb + 7) / 8, 256, 0, s>>>(p);
    } else {
        e = cudaMemsetAsync(p.total, 0, sizeof(uint32_t) * nb, s);
        if (e != cudaSuccess) return e;
    }
    kg_scan_labels<<<1, 32, 0, s>>>(p);
    if (p.n > 0) {
        e = cudaFuncSetAttribute(kg_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_scatter);
        if (e != cudaSuccess) return e;
        kg_scatter<<<p.nblk, GT, smem_scatter, s>>>(p);
    }
    return cudaGetLastError();
}

int group_max_bundles() { return 4095; }

}  // namespace seg
