// seg_internal.cuh -- device data layout shared by the C-ABI layer (seg_api.cu) and the
// sm_100a kernels (classify.cu).  Product code only; the oracle never includes it.
#pragma once
#include <cmath>
#include <cstdint>
#include <cuda_runtime.h>

namespace seg {

// Checked build (-DSEG_DEBUG, scripts/checked_build.sh): every shared-memory queue index, ring stage,
// tile index and scatter position is checked on the device and a violation traps (a sticky launch
// error the host reports).  compute-sanitizer is not available on the GPU pool; this is its stand-in.
#ifdef SEG_DEBUG
#define SEG_DCHECK(cond) do { if (!(cond)) __trap(); } while (0)
#else
#define SEG_DCHECK(cond) do { } while (0)
#endif

constexpr int NPTS = 21;                 // points per fiber / centroid
constexpr int TILE = 32;                 // centroids per tile (one bit per centroid in a u32 mask)
constexpr int TILE_MID = NPTS - 3;       // points other than 0, 10, 20
// plane slot of point i (i != 0, 10, 20) among the middle points; the reversed point 20 - i sits in slot
// TILE_MID - 1 - mid_slot(i)
__host__ __device__ constexpr int mid_slot(int i) { return i < 10 ? i - 1 : i - 2; }
// The tile image (one 1-D TMA bulk copy) after its 144-B TileHdr: points 0 / 10 / 20 of the 32 centroids as
// float4 (w = the screen's lowered half norm, Sec. below); per centroid the chord length and a stored-reversed
// flag (paper mode, else 0); then the 18 middle points as an xy plane (float2) and a z plane, [slot][centroid]
// -- no unused w words, so four stages fit in k_classify's shared memory
constexpr int TI_P0 = 0, TI_P10 = TILE, TI_P20 = 2 * TILE;   // float4 index after the header
constexpr int TI_LEN = 3 * TILE * 4;                          // float index: chord length [32]
constexpr int TI_FLIP = TI_LEN + TILE;                        // float index: 1 = stored reversed [32]
constexpr int TI_MXY = TI_FLIP + TILE;                        // float index: xy plane [18][32] of float2
constexpr int TI_MZ = TI_MXY + 2 * TILE_MID * TILE;           // float index: z plane [18][32]
constexpr int TILE_F4 = (TI_MZ + TILE_MID * TILE) / 4;        // 544 float4 of tile data
static_assert((TI_MZ + TILE_MID * TILE) % 4 == 0 && TI_MXY % 2 == 0, "tile image layout");
// -DSEG_PAIRBOX=0: the round-2 header (112 B, the six end-point boxes as float4 lo / hi per point)
#ifndef SEG_PAIRBOX
#define SEG_PAIRBOX 1
#endif
constexpr int TILE_HDR_F4 = SEG_PAIRBOX ? 9 : 7;   // the tile's TileHdr (144 B) travels in front of its data
constexpr int TILE_STRIDE_F4 = TILE_HDR_F4 + TILE_F4;
constexpr int TILE_STRIDE_BYTES = TILE_STRIDE_F4 * 16;  // 8,848 B -> one 1-D TMA bulk copy
constexpr float CULL_EPS = 1e-3f;        // mm margin on every sphere lower bound

// Exact mode's dot-product screen for test1 / test2.  Each squared distance of the
// dense loop is estimated as h = (|a|^2/2)' + (|c|^2/2)' - a.c (one FADD + three FFMA, against three
// FADD + FMUL + two FFMA for d2), where (|x|^2/2)' = |x|^2/2 * (1 - 2^-18) - 2^-62 rounded down: the
// lowered half norms.  Bound: the four roundings of h cost at most 4u(|a|^2 + |c|^2), the kernel's own
// d2 differs from the true value by at most 8u(|a|^2 + |c|^2) (u = 2^-24, |a - c|^2 <= 2(|a|^2 + |c|^2)),
// and the fiber's half norm is computed in FP32 with at most 5u of its own error; the 2^-18 = 64u
// lowering exceeds their sum, and 2^-62 covers subnormal roundings.  So h <= d2/2 for every pair:
// "h <= tau/2" keeps every pair "d2 <= tau" keeps (a superset; the candidate rounds then evaluate
// exactly, from d2).  A point with a coordinate beyond 2^50 gets -inf (its products stay exact inside
// the FMA, so h = -inf: always kept) -- no overflow is possible below that.
constexpr float SCREEN_SAFE = 0x1p50f;
inline float screen_half_norm_host(const float *c) {
    if (!(std::fabs(c[0]) <= SCREEN_SAFE && std::fabs(c[1]) <= SCREEN_SAFE && std::fabs(c[2]) <= SCREEN_SAFE))
        return -INFINITY;
    const double n = (double)c[0] * c[0] + (double)c[1] * c[1] + (double)c[2] * c[2];
    const double v = 0.5 * n * (1.0 - 0x1p-18) - 0x1p-62;
    float f = (float)v;
    while ((double)f > v) f = std::nextafter(f, -INFINITY);
    return f;
}
constexpr int MORTON_BITS = 6;           // per axis, the grid seg_create scales (inv_cell) for
constexpr int MORTON_BUCKETS = 1 << (3 * MORTON_BITS);
// the prepass grid per call: 7 bits per axis (2^21 buckets) from this many fibers on, else 6 (2^18):
// finer cells order the fibers inside today's cells and spread the scatter's atomics (cfg 3 -1.8%);
// small inputs pay more for the larger histogram than they gain
constexpr int MORTON_FINE_N = 1 << 19;
__host__ __device__ constexpr int morton_bits_for(int n) { return n >= MORTON_FINE_N ? 7 : 6; }

// Per-tile header: the tile's bundle and threshold (FP32, squared too), and the axis-aligned boxes of
// centroid points 0, 10, 20 over the tile's members (exact FP32 min / max, canonical orientation): the
// live tile bound of k_classify.  Boxes leave 0.59-0.81 of the spheres' (fiber, tile) passes at the live
// cutoff; k_cull keeps spheres (CullTile) for its threshold-only list.
// The end-point boxes are stored as f32x2 pairs matching the fiber's packed end points (x0, x20), (y0, y20),
// (z0, z20), so the four end-point box distances take packed FADD2 / FMUL2 / FFMA2 (bit for bit the scalar
// values): d* = (box of point 0, box of point 20) for the direct orientation, i* = (box 20, box 0) for the
// inverse one.
struct __align__(16) TileHdr {
    int bundle;
    float thr2;
    float thr;
    int pad;
#if SEG_PAIRBOX
    float4 lo10, hi10;
    float4 dxy_lo;   // (lo0.x, lo20.x, lo0.y, lo20.y)
    float4 dxy_hi;   // (hi0.x, hi20.x, hi0.y, hi20.y)
    float4 dz;       // (lo0.z, lo20.z, hi0.z, hi20.z)
    float4 ixy_lo;   // (lo20.x, lo0.x, lo20.y, lo0.y)
    float4 ixy_hi;   // (hi20.x, hi0.x, hi20.y, hi0.y)
    float4 iz;       // (lo20.z, lo0.z, hi20.z, hi0.z)
#else
    float4 lo0, hi0, lo10, hi10, lo20, hi20;
#endif
};
static_assert(sizeof(TileHdr) == 16 * TILE_HDR_F4, "TileHdr fills TILE_HDR_F4 float4");

// k_cull's copy of a tile's bounds, squared and grown once at seg_create: c0 / c10 / c20 = sphere centre
// of points 0 / 10 / 20 with w = (radius + thr + CULL_EPS)^2 (the threshold-only bound, rounded up in
// double so it is never smaller than the exact bound), q = (radius + CULL_EPS)^2 per point (the
// "inside" priority test; x, y, z = points 0, 10, 20).
struct __align__(16) CullTile {
    float4 c0, c10, c20, q;
};
static_assert(sizeof(CullTile) == 64, "CullTile is 64 B");

// Per-bundle header: bounding sphere of point 10 over the bundle, tile range [t0, t1).
struct __align__(16) BundleHdr {
    float4 s10;
    int t0, t1;
    float thr;
    float thr2;
};
static_assert(sizeof(BundleHdr) == 32, "BundleHdr is 32 B");

struct ClassifyParams {
    const unsigned long long *seed;  // nullable [n] initial best keys (d2 bits << 32 | bundle), by caller index
    const float *fibers;      // [n][21][3]
    int n;
    const int32_t *perm;      // nullable: processing order -> caller index
    int32_t *label;           // [n]
    float *dist;              // [n]
    const float4 *tiles;      // [T][TILE_STRIDE_F4]: TileHdr, then [21][32] points
    const TileHdr *th;        // [T]
    const CullTile *ct;       // [T] k_cull's precomputed squared bounds
    const BundleHdr *bh;      // [B]
    int B, T;
    unsigned long long *stats; // [SEG_NSTATS] (stats instantiation only)
    uint32_t *tile_bits;       // scratch: per CTA of FPC fibers, [count, tiles...] as u16 (cull_stride(T)): k_cull -> k_classify
    int paper;                 // 0 = exact Eq. 2 (north_star), 1 = paper semantics (Eq. 3 TN, inferred orientation)
    unsigned long long *keys;  // nullable [n]: write the best keys (row f4) instead of label / dist
    int32_t *seed_code;            // nullable [n] by fiber: k_cull's seed candidate, (tile << 6) | (centroid << 1) | o, -1 = none
    const float4 *tiles_cm;        // [T][32][21] centroid-major copy of the tile points (the seed evaluation)
    int32_t *cta_order = nullptr;  // nullable [grid]: k_classify's CTA i works on fiber window cta_order[i]
    uint32_t *masks = nullptr;     // nullable [n][mwords]: multi-label output (row f4), bit b = bundle b within threshold
    int mwords = 0;
};

struct MortonParams {
    const float *fibers;
    int n;
    float3 lo;
    float3 inv_cell;          // buckets per mm along each axis
    uint32_t *key;            // [n]
    uint32_t *hist;           // [MORTON_BUCKETS]
    uint32_t *bsum;           // [MORTON_BUCKETS / 1024] per-block totals, then offsets
    int32_t *perm;            // [n]
    int bits;                 // grid bits per axis for this call (morton_bits_for(n))
    uint32_t *rank = nullptr; // [n] each fiber's arrival rank in its bucket (k_morton_hist's atomic)
};

// Row f3 (group.cu): the stable partition of the fibers by label.
struct GroupParams {
    const int32_t *label;      // [n]
    const float *dist;         // [n] nullable: no summaries
    int64_t n;
    int B;
    int nblk;                  // set by launch_group
    uint32_t *hist;            // scratch [B+1][nblk]
    uint32_t *total;           // scratch [B+1]
    int64_t *offsets;          // [B+2]
    int32_t *order;            // [n]
    uint32_t *gmin, *gmax;     // [B] float bits (distances >= 0)
    double *dsum;              // [B]
    int summ;                  // summaries requested (gmin / gmax / dsum written, even for n = 0)
};

// Row f2 (resample.cu): raw polylines -> 21 points equidistant in chord length.
struct ResampleParams {
    const float *points;       // [P][3]
    const int64_t *offsets;    // [n + 1]: fiber f = points[offsets[f] .. offsets[f + 1])
    int64_t n;
    float *out;                // [n][21][3]
};

// Launchers (classify.cu, group.cu, resample.cu).  All are asynchronous on `s`.
cudaError_t launch_morton_prepass(const MortonParams &p, cudaStream_t s);
size_t morton_scratch_words(int bits);   // hist + block offsets
cudaError_t launch_classify(const ClassifyParams &p, bool stats, cudaStream_t s, cudaEvent_t after_cull = nullptr);
size_t classify_smem_bytes(int B, int T);
size_t cull_bits_words(int n, int T);
int classify_max_tiles();
int classify_multi_max_bundles();
int classify_fibers_per_cta();
cudaError_t launch_group(GroupParams p, cudaStream_t s);
size_t group_scratch_words(int64_t n, int B);
int group_max_bundles();
cudaError_t launch_resample(const ResampleParams &p, int sm_count, cudaStream_t s);
cudaError_t launch_keys_to_labels(const unsigned long long *keys, int64_t n, int paper, int32_t *label, float *dist,
                                  cudaStream_t s);

}  // namespace seg
