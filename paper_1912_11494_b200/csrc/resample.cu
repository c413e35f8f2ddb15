// resample.cu -- row f2: the step before the path.  Raw tractography
// streamlines of any length become the 21-point fibers the method compares: "subject fibers are
// resampled using 21 equidistant points".  Chord-length parameterisation with linear
// interpolation (reading R19, after SPEC.md:63-71): with s_j the cumulative chord length at input
// point j and L the total, output point k is the point at arc position k L / 20 on the polyline;
// points 0 and 20 are the input's end points exactly.
//
// One warp per fiber (grid-stride).  Fibers of up to 256 segments (the common case): one pass over the
// points, lane j the segment j of each 32-segment chunk, its length in double and a warp prefix give
// the cumulative arc lengths, kept in shared memory; then lanes 3..21 each binary-search their target
// k L / 20 (the first segment whose end reaches it), interpolate in double and round to FP32 once.
// Longer fibers stream the same arithmetic chunk by chunk and assign the targets by ballots.  The 21
// points are staged in shared memory and written as 63 consecutive floats (coalesced).  HBM-bound in
// principle (12 B read per input point, 252 B written per fiber); in practice latency-bound by the
// dependent double-precision scan and search.  A fiber with fewer than 2 points,
// zero length or non-finite points is invalid input: its 63 outputs are NaN, which seg_classify labels
// -1 / NaN.
#include <cmath>
#include <cstdint>

#include "seg_internal.cuh"

namespace seg {

constexpr int RT = 256;          // threads per block
constexpr int RW = RT / 32;      // fibers (warps) per block in flight
constexpr int RSEG = 256;        // segments a warp keeps in shared memory (longer fibers: streaming path)

// Short path (m - 1 <= RSEG segments): one pass over the points computes the cumulative arc lengths
// e_j (double, warp prefix per 32 segments) into shared memory; then lanes 1..19 each binary-search
// their target k L / 20 (the first segment whose end reaches it) and interpolate in parallel.
// Long path: the same arithmetic streamed chunk by chunk, the targets assigned by ballots.
__global__ void __launch_bounds__(RT) kr_resample(ResampleParams p) {
    extern __shared__ double rsm[];
    __shared__ float stage[RW][3 * NPTS];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float *st = stage[warp];
    double *E = rsm + (size_t)warp * RSEG;   // cumulative chord length at the end of each segment
    const int64_t nwarps = (int64_t)gridDim.x * RW;
    for (int64_t f = (int64_t)blockIdx.x * RW + warp; f < p.n; f += nwarps) {
        const int64_t beg = p.offsets[f], end = p.offsets[f + 1];
        const int64_t m = end - beg;   // points
        const float *P = p.points + 3 * beg;
        const int64_t nseg = m - 1;
        bool ok = m >= 2;
        if (ok && nseg <= RSEG) {
            double carry = 0.0;
            for (int64_t j0 = 0; j0 < nseg; j0 += 32) {
                const int64_t j = j0 + lane;
                double len = 0.0;
                if (j < nseg) {
                    const double dx = (double)P[3 * (j + 1)] - (double)P[3 * j];
                    const double dy = (double)P[3 * (j + 1) + 1] - (double)P[3 * j + 1];
                    const double dz = (double)P[3 * (j + 1) + 2] - (double)P[3 * j + 2];
                    len = sqrt(dx * dx + dy * dy + dz * dz);
                }
                double incl = len;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const double t = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += t;
                }
                if (j < nseg) E[j] = carry + incl;
                carry += __shfl_sync(0xffffffffu, incl, 31);
            }
            __syncwarp();
            const double L = carry;
            ok = L > 0.0 && isfinite(L);
            if (ok) {
                if (lane < 3) {
                    st[lane] = P[lane];                                    // point 0, exactly
                    st[3 * (NPTS - 1) + lane] = P[3 * (m - 1) + lane];     // point 20, exactly
                } else if (lane < NPTS - 1 + 2) {
                    const int k = lane - 2;                                // targets 1..19 on lanes 3..21
                    const double t = (double)k * L / (double)(NPTS - 1);
                    int64_t lo = 0, hi = nseg - 1;                         // first j with E[j] >= t
                    while (lo < hi) {
                        const int64_t mid = (lo + hi) >> 1;
                        if (E[mid] >= t) hi = mid; else lo = mid + 1;
                    }
                    const int64_t j = lo;
                    SEG_DCHECK(j >= 0 && j < nseg);
                    const double s = j > 0 ? E[j - 1] : 0.0;
                    const double ax = P[3 * j], ay = P[3 * j + 1], az = P[3 * j + 2];
                    const double bx = P[3 * (j + 1)], by = P[3 * (j + 1) + 1], bz = P[3 * (j + 1) + 2];
                    const double len = sqrt((bx - ax) * (bx - ax) + (by - ay) * (by - ay) + (bz - az) * (bz - az));
                    const double u = len > 0.0 ? fmin(fmax((t - s) / len, 0.0), 1.0) : 0.0;
                    st[3 * k + 0] = (float)(ax + u * (bx - ax));
                    st[3 * k + 1] = (float)(ay + u * (by - ay));
                    st[3 * k + 2] = (float)(az + u * (bz - az));
                }
            }
        } else if (ok) {
            // long fibers: total length first, then the chunks again with ballot-assigned targets
            double part = 0.0;
            for (int64_t j = lane; j < nseg; j += 32) {
                const double dx = (double)P[3 * (j + 1)] - (double)P[3 * j];
                const double dy = (double)P[3 * (j + 1) + 1] - (double)P[3 * j + 1];
                const double dz = (double)P[3 * (j + 1) + 2] - (double)P[3 * j + 2];
                part += sqrt(dx * dx + dy * dy + dz * dz);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
            const double L = part;
            ok = L > 0.0 && isfinite(L);
            if (ok) {
                if (lane < 3) {
                    st[lane] = P[lane];
                    st[3 * (NPTS - 1) + lane] = P[3 * (m - 1) + lane];
                }
                int k = 1;
                double carry = 0.0;
                for (int64_t j0 = 0; j0 < nseg && k < NPTS - 1; j0 += 32) {
                    const int64_t j = j0 + lane;
                    const bool seg = j < nseg;
                    double ax = 0, ay = 0, az = 0, bx = 0, by = 0, bz = 0, len = 0;
                    if (seg) {
                        ax = P[3 * j]; ay = P[3 * j + 1]; az = P[3 * j + 2];
                        bx = P[3 * (j + 1)]; by = P[3 * (j + 1) + 1]; bz = P[3 * (j + 1) + 2];
                        len = sqrt((bx - ax) * (bx - ax) + (by - ay) * (by - ay) + (bz - az) * (bz - az));
                    }
                    double incl = len;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const double t = __shfl_up_sync(0xffffffffu, incl, o);
                        if (lane >= o) incl += t;
                    }
                    const double e = carry + incl, s = e - len;
                    const bool last_chunk = j0 + 32 >= nseg;
                    while (k < NPTS - 1) {
                        const double t = (double)k * L / (double)(NPTS - 1);
                        const uint32_t reach = __ballot_sync(0xffffffffu, seg && e >= t);
                        const uint32_t segs = __ballot_sync(0xffffffffu, seg);
                        const int owner = reach ? __ffs(reach) - 1 : (last_chunk ? 31 - __clz(segs) : -1);
                        if (owner < 0) break;
                        SEG_DCHECK(k >= 1 && k < NPTS - 1);
                        if (lane == owner) {
                            const double u = len > 0.0 ? fmin(fmax((t - s) / len, 0.0), 1.0) : 0.0;
                            st[3 * k + 0] = (float)(ax + u * (bx - ax));
                            st[3 * k + 1] = (float)(ay + u * (by - ay));
                            st[3 * k + 2] = (float)(az + u * (bz - az));
                        }
                        ++k;
                    }
                    carry = __shfl_sync(0xffffffffu, e, 31);
                }
            }
        }
        if (!ok)
            for (int i = lane; i < 3 * NPTS; i += 32) st[i] = __int_as_float(0x7fffffff);
        __syncwarp();
        float *o = p.out + (size_t)f * 3 * NPTS;
        for (int i = lane; i < 3 * NPTS; i += 32) o[i] = st[i];
        __syncwarp();
    }
}

cudaError_t launch_resample(const ResampleParams &p, int sm_count, cudaStream_t s) {
    if (p.n <= 0) return cudaSuccess;
    const int64_t want = (p.n + RW - 1) / RW;
    const int grid = (int)std::min<int64_t>(want, (int64_t)sm_count * 8);
    const size_t smem = sizeof(double) * (size_t)RW * RSEG;
    cudaError_t e = cudaFuncSetAttribute(kr_resample, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kr_resample<<<grid, RT, smem, s>>>(p);
    return cudaGetLastError();
}

}  // namespace seg
