// seg_api.cu -- the C ABI of libsegb200.so (include/seg.h): argument validation, the
// host-side atlas preparation, the device launch sequence and the
// host-buffer streaming path.  Every step of the hot path runs in the kernels of classify.cu;
// this file only plans, copies and launches.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/seg.h"
#include "seg_internal.cuh"

using namespace seg;

// ----------------------------------------------------------------------------------------
// errors
// ----------------------------------------------------------------------------------------
static thread_local std::string g_err;

static int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}
static int cuda_fail(cudaError_t e, const char *what) {
    std::string m = std::string(what) + ": " + cudaGetErrorString(e);
    cudaGetLastError();  // clear sticky-less error state
    return fail(SEG_ECUDA, m);
}
#define SEG_CUDA(call, what)                          \
    do {                                              \
        cudaError_t e__ = (call);                     \
        if (e__ != cudaSuccess) return cuda_fail(e__, what); \
    } while (0)

extern "C" const char *seg_last_error(void) { return g_err.c_str(); }

// ----------------------------------------------------------------------------------------
// the atlas context
// ----------------------------------------------------------------------------------------
struct seg_atlas {
    int device = 0;
    int64_t M = 0;
    int B = 0, T = 0;
    int paper = 0;                // SEG_MODE_PAPER: score = d_ME (inferred orientation) + TN
    int sms = 148;                // SM count of the device (k_classify's launch-order heuristic)
    float4 *tiles = nullptr;      // [T][TILE_STRIDE_F4]: header + [21][32] points (point 0's w = chord length)
    float4 *tiles_cm = nullptr;   // [T][32][21] the same points centroid-major (the seed evaluation's loads)
    TileHdr *th = nullptr;        // [T]
    CullTile *ct = nullptr;       // [T] squared bounds for k_cull
    BundleHdr *bh = nullptr;      // [B]
    float3 lo{}, inv_cell{};      // Morton grid of the prepass
    int64_t bytes = 0;
    // the atlas's own stream-ordered memory pool for per-call scratch, kept cached between calls (release
    // threshold: never); nullptr -> the device's default pool, left as the caller configured it
    cudaMemPool_t pool = nullptr;
    // profiling hook (seg_profile_enable / seg_profile_read); mutable, not thread-safe
    mutable std::vector<cudaEvent_t> prof_ev;  // 4 per recorded call
    mutable int prof_cap = 0, prof_n = 0;
};

namespace {

struct DeviceGuard {  // restores the caller's current device
    int prev = -1;
    bool ok = false;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) { cudaGetLastError(); return; }
        ok = (prev == dev) || cudaSetDevice(dev) == cudaSuccess;
        if (!ok) cudaGetLastError();
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// The library's own stream-ordered pool per device, for the entry points without an atlas
// (seg_group_by_bundle): created once, kept cached (release threshold: never), so repeated calls do
// not map fresh memory; the device's default pool is left as the caller configured it.  nullptr if a
// pool cannot be created (the default pool is used then).
cudaMemPool_t lib_pool(int dev) {
    static std::mutex mu;
    static cudaMemPool_t pools[64] = {};
    static bool tried[64] = {};
    if (dev < 0 || dev >= 64) return nullptr;
    std::lock_guard<std::mutex> lock(mu);
    if (!tried[dev]) {
        tried[dev] = true;
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        if (cudaMemPoolCreate(&pools[dev], &props) == cudaSuccess) {
            uint64_t thr_bytes = UINT64_MAX;
            cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &thr_bytes);
        } else {
            pools[dev] = nullptr;
            cudaGetLastError();
        }
    }
    return pools[dev];
}

// 1 = device (or managed) memory, 0 = host memory, -1 = CUDA unavailable
int pointer_kind(const void *p, int *dev) {
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) {
        *dev = a.device;
        return 1;
    }
    return 0;
}

// Tile plan (row a0): group by bundle, canonicalise each centroid's point order against the
// bundle's first member (d_ME is invariant under reversing a centroid, Eq. 2, so this is
// exact), split every bundle recursively at the median of its widest feature among
// points 0/10/20 into tiles of 32, pad the last tile by repeating a real member (a duplicate
// of a member of the same bundle can never change a (distance, bundle) minimum), and bound
// points 0/10/20 of each tile by spheres (double precision, radius rounded up to FP32).
struct Plan {
    int T = 0;
    std::vector<int> tile_bundle;           // [T]
    std::vector<int> members;               // [T*32] caller centroid index
    std::vector<unsigned char> flipped;     // [M] stored reversed?
    std::vector<float> spheres;             // [T*12]
    std::vector<int> b_t0, b_t1;            // [B]
    std::vector<float> b_s10;               // [B*4]
};

void sphere(const float *cents, const std::vector<unsigned char> &flipped, const int *mem, int cnt, int point,
            float out[4]) {
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    auto pt = [&](int m, int k) -> double {
        const int pp = flipped[m] ? (NPTS - 1 - point) : point;
        return (double)cents[(size_t)m * 3 * NPTS + 3 * pp + k];
    };
    for (int j = 0; j < cnt; ++j)
        for (int k = 0; k < 3; ++k) {
            lo[k] = std::min(lo[k], pt(mem[j], k));
            hi[k] = std::max(hi[k], pt(mem[j], k));
        }
    float c[3];
    for (int k = 0; k < 3; ++k) c[k] = (float)(0.5 * (lo[k] + hi[k]));
    double r2 = 0.0;
    for (int j = 0; j < cnt; ++j) {
        double s = 0.0;
        for (int k = 0; k < 3; ++k) {
            const double d = pt(mem[j], k) - (double)c[k];
            s += d * d;
        }
        r2 = std::max(r2, s);
    }
    const double r = std::sqrt(r2);
    float rf = (float)r;
    while ((double)rf < r) rf = std::nextafter(rf, INFINITY);
    out[0] = c[0];
    out[1] = c[1];
    out[2] = c[2];
    out[3] = rf;
}

void split_tiles(const float *cents, const std::vector<unsigned char> &flipped, std::vector<int> &ids, int lo,
                 int hi, std::vector<std::vector<int>> &tiles_out) {
    const int n = hi - lo;
    if (n <= TILE) {
        tiles_out.emplace_back(ids.begin() + lo, ids.begin() + hi);
        return;
    }
    const int ntiles = (n + TILE - 1) / TILE;
    const int left = (ntiles / 2) * TILE;
    auto feat = [&](int m, int d) -> float {
        const int point = (d / 3) == 0 ? 0 : ((d / 3) == 1 ? 10 : 20);
        const int pp = flipped[m] ? (NPTS - 1 - point) : point;
        return cents[(size_t)m * 3 * NPTS + 3 * pp + (d % 3)];
    };
    int best_d = 0;
    float best_ext = -1.f;
    for (int d = 0; d < 9; ++d) {
        float mn = INFINITY, mx = -INFINITY;
        for (int j = lo; j < hi; ++j) {
            const float v = feat(ids[j], d);
            mn = std::min(mn, v);
            mx = std::max(mx, v);
        }
        if (mx - mn > best_ext) {
            best_ext = mx - mn;
            best_d = d;
        }
    }
    std::nth_element(ids.begin() + lo, ids.begin() + lo + left, ids.begin() + hi, [&](int a, int b) {
        const float fa = feat(a, best_d), fb = feat(b, best_d);
        return fa < fb || (fa == fb && a < b);
    });
    split_tiles(cents, flipped, ids, lo, lo + left, tiles_out);
    split_tiles(cents, flipped, ids, lo + left, hi, tiles_out);
}

int make_plan(const float *cents, const int32_t *bid, int64_t M, int B, Plan &P) {
    try {
        std::vector<std::vector<int>> by_b(B);
        for (int64_t m = 0; m < M; ++m) by_b[bid[m]].push_back((int)m);
        P.flipped.assign(M, 0);
        auto at = [&](int m, int point, int k) { return (double)cents[(size_t)m * 3 * NPTS + 3 * point + k]; };
        for (int b = 0; b < B; ++b) {
            if (by_b[b].empty()) continue;
            const int r = by_b[b][0];
            for (int m : by_b[b]) {
                double same = 0, rev = 0;
                for (int k = 0; k < 3; ++k) {
                    const double a0 = at(m, 0, k) - at(r, 0, k), a1 = at(m, 20, k) - at(r, 20, k);
                    const double b0 = at(m, 20, k) - at(r, 0, k), b1 = at(m, 0, k) - at(r, 20, k);
                    same += a0 * a0 + a1 * a1;
                    rev += b0 * b0 + b1 * b1;
                }
                P.flipped[m] = rev < same ? 1 : 0;
            }
        }
        P.b_t0.assign(B, 0);
        P.b_t1.assign(B, 0);
        P.b_s10.assign((size_t)B * 4, 0.f);
        P.T = 0;
        P.tile_bundle.clear();
        P.members.clear();
        P.spheres.clear();
        for (int b = 0; b < B; ++b) {
            P.b_t0[b] = P.T;
            if (by_b[b].empty()) {
                P.b_t1[b] = P.T;
                continue;
            }
            std::vector<std::vector<int>> tl;
            split_tiles(cents, P.flipped, by_b[b], 0, (int)by_b[b].size(), tl);
            for (auto &t : tl) {
                std::sort(t.begin(), t.end());
                P.tile_bundle.push_back(b);
                for (int k = 0; k < TILE; ++k) P.members.push_back(t[std::min<int>(k, (int)t.size() - 1)]);
                float s[4];
                for (int q = 0; q < 3; ++q) {
                    sphere(cents, P.flipped, t.data(), (int)t.size(), q == 0 ? 0 : (q == 1 ? 10 : 20), s);
                    for (int k = 0; k < 4; ++k) P.spheres.push_back(s[k]);
                }
                ++P.T;
            }
            P.b_t1[b] = P.T;
            sphere(cents, P.flipped, by_b[b].data(), (int)by_b[b].size(), 10, &P.b_s10[(size_t)b * 4]);
        }
    } catch (const std::bad_alloc &) {
        return fail(SEG_ENOMEM, "seg_create: host allocation failed");
    }
    return SEG_OK;
}

int validate_atlas_host(const float *cents, const int32_t *bid, int64_t M, const float *thr, int B) {
    for (int64_t m = 0; m < M; ++m)
        if (bid[m] < 0 || bid[m] >= B)
            return fail(SEG_EINVAL, "seg_create: bundle_id[" + std::to_string(m) + "] = " +
                                        std::to_string(bid[m]) + " not in [0, B)");
    for (size_t i = 0; i < (size_t)M * 3 * NPTS; ++i)
        if (!std::isfinite(cents[i]))
            return fail(SEG_EINVAL, "seg_create: non-finite centroid coordinate at flat index " + std::to_string(i));
    if (thr)
        for (int b = 0; b < B; ++b)
            if (!std::isfinite(thr[b]) || !(thr[b] > 0.f))
                return fail(SEG_EINVAL, "seg_create: thresh[" + std::to_string(b) + "] must be finite and > 0");
    return SEG_OK;
}

// Stage a caller array (host or device) into a host vector.
template <class T>
int to_host(const T *p, size_t n, std::vector<T> &out, int *dev_seen) {
    int dev = -1;
    const int kind = pointer_kind(p, &dev);
    try {
        out.resize(n);
    } catch (const std::bad_alloc &) {
        return fail(SEG_ENOMEM, "seg_create: host allocation failed");
    }
    if (kind == 1) {
        *dev_seen = dev;
        SEG_CUDA(cudaMemcpy(out.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost), "seg_create: cudaMemcpy D2H");
    } else if (kind == 0) {
        std::memcpy(out.data(), p, n * sizeof(T));
    } else {
        return fail(SEG_ECUDA, "seg_create: no usable CUDA device");
    }
    return SEG_OK;
}

}  // namespace

// ----------------------------------------------------------------------------------------
// seg_plan_tiles (host only)
// ----------------------------------------------------------------------------------------
extern "C" int seg_plan_tiles(const float *centroids, const int32_t *bundle_id, int64_t M, int32_t B,
                              int32_t max_tiles, int32_t *n_tiles, int32_t *tile_bundle, int32_t *tile_members,
                              float *tile_spheres) {
    if (!centroids || !bundle_id || !n_tiles) return fail(SEG_EINVAL, "seg_plan_tiles: null pointer");
    if (M < 1 || M > INT32_MAX || B < 1) return fail(SEG_EINVAL, "seg_plan_tiles: M and B must be >= 1");
    int rc = validate_atlas_host(centroids, bundle_id, M, nullptr, B);
    if (rc) return rc;
    Plan P;
    rc = make_plan(centroids, bundle_id, M, B, P);
    if (rc) return rc;
    *n_tiles = P.T;
    const int nt = std::min(P.T, std::max(0, max_tiles));
    for (int t = 0; t < nt; ++t) {
        if (tile_bundle) tile_bundle[t] = P.tile_bundle[t];
        if (tile_members)
            for (int k = 0; k < TILE; ++k) tile_members[t * TILE + k] = P.members[(size_t)t * TILE + k];
        if (tile_spheres)
            for (int k = 0; k < 12; ++k) tile_spheres[t * 12 + k] = P.spheres[(size_t)t * 12 + k];
    }
    g_err.clear();
    return SEG_OK;
}

// ----------------------------------------------------------------------------------------
// seg_create / seg_destroy / seg_get_atlas_info
// ----------------------------------------------------------------------------------------
static void free_prof(const seg_atlas *a) {
    for (cudaEvent_t e : a->prof_ev) cudaEventDestroy(e);
    a->prof_ev.clear();
    a->prof_cap = a->prof_n = 0;
}

static void free_atlas(seg_atlas *a) {
    if (!a) return;
    DeviceGuard g(a->device);
    free_prof(a);
    cudaFree(a->tiles);
    cudaFree(a->tiles_cm);
    cudaFree(a->th);
    cudaFree(a->ct);
    cudaFree(a->bh);
    // outstanding stream-ordered frees are completed by the driver before the pool goes away
    if (a->pool) cudaMemPoolDestroy(a->pool);
    delete a;
}

extern "C" void seg_destroy(seg_atlas *a) { free_atlas(a); }

extern "C" int seg_create_ex(const float *centroids, const int32_t *bundle_id, int64_t M, const float *thresh,
                             int32_t B, int device, uint32_t flags, seg_atlas **out) {
    if (out) *out = nullptr;
    if (flags & ~(uint32_t)SEG_MODE_PAPER) return fail(SEG_EINVAL, "seg_create_ex: unknown flags");
    if (!centroids || !bundle_id || !thresh || !out) return fail(SEG_EINVAL, "seg_create: null pointer");
    if (M < 1 || M > INT32_MAX) return fail(SEG_EINVAL, "seg_create: M must be in [1, 2^31-1]");
    if (B < 1) return fail(SEG_EINVAL, "seg_create: B must be >= 1");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
        cudaGetLastError();
        return fail(SEG_ECUDA, "seg_create: no usable CUDA device");
    }
    if (device < 0) SEG_CUDA(cudaGetDevice(&device), "seg_create: cudaGetDevice");
    if (device >= ndev) return fail(SEG_EINVAL, "seg_create: device ordinal out of range");
    DeviceGuard guard(device);
    if (!guard.ok) return fail(SEG_ECUDA, "seg_create: cudaSetDevice failed");

    std::vector<float> cents, thr;
    std::vector<int32_t> bid;
    int dev_seen = device;
    int rc = to_host(centroids, (size_t)M * 3 * NPTS, cents, &dev_seen);
    if (!rc) rc = to_host(bundle_id, (size_t)M, bid, &dev_seen);
    if (!rc) rc = to_host(thresh, (size_t)B, thr, &dev_seen);
    if (rc) return rc;
    rc = validate_atlas_host(cents.data(), bid.data(), M, thr.data(), B);
    if (rc) return rc;
    Plan P;
    rc = make_plan(cents.data(), bid.data(), M, B, P);
    if (rc) return rc;
    if (P.T > classify_max_tiles())
        return fail(SEG_EINVAL, "seg_create: atlas needs " + std::to_string(P.T) + " tiles of 32 centroids; this build "
                                "supports at most " + std::to_string(classify_max_tiles()));

    // device images
    std::vector<float4> tiles((size_t)P.T * TILE_STRIDE_F4);
    std::vector<float4> tiles_cm((size_t)P.T * TILE * NPTS);
    // chord length of every centroid's 21-point polyline (Eq. 3's l_C, reading R16), in double
    std::vector<float> clen((size_t)M);
    for (int64_t m = 0; m < M; ++m) {
        double l = 0.0;
        for (int i = 0; i + 1 < NPTS; ++i) {
            double s2 = 0.0;
            for (int d = 0; d < 3; ++d) {
                const double df = (double)cents[(size_t)m * 3 * NPTS + 3 * (i + 1) + d] - (double)cents[(size_t)m * 3 * NPTS + 3 * i + d];
                s2 += df * df;
            }
            l += std::sqrt(s2);
        }
        clen[(size_t)m] = (float)l;
    }
    std::vector<TileHdr> th(P.T);
    std::vector<CullTile> ct(P.T);
    auto sq_up = [](double r) {   // r^2 rounded up to FP32
        const double v = r * r;
        float f = (float)v;
        while ((double)f < v) f = std::nextafter(f, INFINITY);
        return f;
    };
    std::vector<BundleHdr> bh(B);
    float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int t = 0; t < P.T; ++t) {
        for (int k = 0; k < TILE; ++k) {
            const int m = P.members[(size_t)t * TILE + k];
            for (int i = 0; i < NPTS; ++i) {
                const int src = P.flipped[m] ? (NPTS - 1 - i) : i;
                const float *c = &cents[(size_t)m * 3 * NPTS + 3 * src];
                // points 0, 10, 20 carry the lowered half squared norm of k_classify's dot-product screen in w
                // (seg_internal.cuh), both modes; paper mode also the chord length (Eq. 3) and a 1 when the
                // centroid is stored reversed (an exact end-point tie then picks the caller's direct
                // orientation, so the result does not depend on the stored order)
                const bool paper = (flags & SEG_MODE_PAPER) != 0;
                float4 *t4 = &tiles[(size_t)t * TILE_STRIDE_F4 + TILE_HDR_F4];
                float *tf = reinterpret_cast<float *>(t4);
                if (i == 0 || i == 10 || i == 20) {
                    t4[(i == 0 ? TI_P0 : i == 10 ? TI_P10 : TI_P20) + k] = make_float4(c[0], c[1], c[2], screen_half_norm_host(c));
                } else {
                    tf[TI_MXY + 2 * (mid_slot(i) * TILE + k)] = c[0];
                    tf[TI_MXY + 2 * (mid_slot(i) * TILE + k) + 1] = c[1];
                    tf[TI_MZ + mid_slot(i) * TILE + k] = c[2];
                }
                if (i == 0) {
                    tf[TI_LEN + k] = paper ? clen[(size_t)m] : 0.f;
                    tf[TI_FLIP + k] = paper && P.flipped[m] ? 1.f : 0.f;
                }
                tiles_cm[((size_t)t * TILE + k) * NPTS + i] = make_float4(c[0], c[1], c[2], 0.f);
                for (int d = 0; d < 3; ++d) {
                    lo[d] = std::min(lo[d], c[d]);
                    hi[d] = std::max(hi[d], c[d]);
                }
            }
        }
        const float *s = &P.spheres[(size_t)t * 12];
        const int b = P.tile_bundle[t];
        th[t].bundle = b;
        th[t].thr = thr[b];
        th[t].thr2 = thr[b] * thr[b];
        th[t].pad = 0;
        {   // the boxes of points 0, 10, 20 over the tile's members (padding slots repeat a member)
            float blo[3][3], bhi[3][3];
            for (int q = 0; q < 3; ++q)
                for (int d = 0; d < 3; ++d) { blo[q][d] = INFINITY; bhi[q][d] = -INFINITY; }
            for (int k = 0; k < TILE; ++k) {
                const int m = P.members[(size_t)t * TILE + k];
                const int pts[3] = {0, 10, 20};
                for (int q = 0; q < 3; ++q) {
                    const int src = P.flipped[m] ? (NPTS - 1 - pts[q]) : pts[q];
                    const float *c = &cents[(size_t)m * 3 * NPTS + 3 * src];
                    for (int d = 0; d < 3; ++d) {
                        blo[q][d] = std::min(blo[q][d], c[d]);
                        bhi[q][d] = std::max(bhi[q][d], c[d]);
                    }
                }
            }
            th[t].lo10 = make_float4(blo[1][0], blo[1][1], blo[1][2], 0.f);
            th[t].hi10 = make_float4(bhi[1][0], bhi[1][1], bhi[1][2], 0.f);
#if SEG_PAIRBOX
            // end-point boxes as (point 0, point 20) pairs and swapped (seg_internal.cuh)
            th[t].dxy_lo = make_float4(blo[0][0], blo[2][0], blo[0][1], blo[2][1]);
            th[t].dxy_hi = make_float4(bhi[0][0], bhi[2][0], bhi[0][1], bhi[2][1]);
            th[t].dz = make_float4(blo[0][2], blo[2][2], bhi[0][2], bhi[2][2]);
            th[t].ixy_lo = make_float4(blo[2][0], blo[0][0], blo[2][1], blo[0][1]);
            th[t].ixy_hi = make_float4(bhi[2][0], bhi[0][0], bhi[2][1], bhi[0][1]);
            th[t].iz = make_float4(blo[2][2], blo[0][2], bhi[2][2], bhi[0][2]);
#else
            th[t].lo0 = make_float4(blo[0][0], blo[0][1], blo[0][2], 0.f);
            th[t].hi0 = make_float4(bhi[0][0], bhi[0][1], bhi[0][2], 0.f);
            th[t].lo20 = make_float4(blo[2][0], blo[2][1], blo[2][2], 0.f);
            th[t].hi20 = make_float4(bhi[2][0], bhi[2][1], bhi[2][2], 0.f);
#endif
        }
        {
            const double sv = (double)thr[b] + (double)CULL_EPS;
            ct[t].c0 = make_float4(s[0], s[1], s[2], sq_up((double)s[3] + sv));
            ct[t].c10 = make_float4(s[4], s[5], s[6], sq_up((double)s[7] + sv));
            ct[t].c20 = make_float4(s[8], s[9], s[10], sq_up((double)s[11] + sv));
            ct[t].q = make_float4(sq_up((double)s[3] + CULL_EPS), sq_up((double)s[7] + CULL_EPS),
                                  sq_up((double)s[11] + CULL_EPS), 0.f);
        }
        std::memcpy(&tiles[(size_t)t * TILE_STRIDE_F4], &th[t], sizeof(TileHdr));
    }
    float maxthr = 0.f;
    for (int b = 0; b < B; ++b) {
        const float *s = &P.b_s10[(size_t)b * 4];
        bh[b].s10 = make_float4(s[0], s[1], s[2], s[3]);
        bh[b].t0 = P.b_t0[b];
        bh[b].t1 = P.b_t1[b];
        bh[b].thr = thr[b];
        bh[b].thr2 = thr[b] * thr[b];
        maxthr = std::max(maxthr, thr[b]);
    }

    seg_atlas *a = new (std::nothrow) seg_atlas();
    if (!a) return fail(SEG_ENOMEM, "seg_create: host allocation failed");
    a->device = device;
    a->paper = (flags & SEG_MODE_PAPER) ? 1 : 0;
    if (cudaDeviceGetAttribute(&a->sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) a->sms = 148;
    a->M = M;
    a->B = B;
    a->T = P.T;
    float ext[3];
    for (int d = 0; d < 3; ++d) {
        lo[d] -= maxthr;
        hi[d] += maxthr;
        ext[d] = std::max(hi[d] - lo[d], 1e-3f);
    }
    const float nb = (float)(1 << MORTON_BITS);
    a->lo = make_float3(lo[0], lo[1], lo[2]);
    a->inv_cell = make_float3(nb / ext[0], nb / ext[1], nb / ext[2]);
    const size_t bt = tiles.size() * sizeof(float4), bth = th.size() * sizeof(TileHdr),
                 bbh = bh.size() * sizeof(BundleHdr);
    cudaError_t e = cudaMalloc(&a->tiles, bt);
    if (e == cudaSuccess) e = cudaMalloc(&a->tiles_cm, tiles_cm.size() * sizeof(float4));
    if (e == cudaSuccess) e = cudaMalloc(&a->th, bth);
    if (e == cudaSuccess) e = cudaMalloc(&a->ct, sizeof(CullTile) * ct.size());
    if (e == cudaSuccess) e = cudaMalloc(&a->bh, bbh);
    if (e != cudaSuccess) {
        free_atlas(a);
        cudaGetLastError();
        return fail(e == cudaErrorMemoryAllocation ? SEG_ENOMEM : SEG_ECUDA,
                    std::string("seg_create: cudaMalloc: ") + cudaGetErrorString(e));
    }
    e = cudaMemcpy(a->tiles, tiles.data(), bt, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(a->tiles_cm, tiles_cm.data(), tiles_cm.size() * sizeof(float4), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(a->th, th.data(), bth, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(a->ct, ct.data(), sizeof(CullTile) * ct.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(a->bh, bh.data(), bbh, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        free_atlas(a);
        return cuda_fail(e, "seg_create: cudaMemcpy H2D");
    }
    a->bytes = (int64_t)(bt + bth + bbh + sizeof(CullTile) * ct.size() + tiles_cm.size() * sizeof(float4));
    // a private pool keeps the per-call scratch cached between seg_classify calls without changing the
    // device's default pool; if one cannot be created the default pool is used as it is
    {
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = device;
        if (cudaMemPoolCreate(&a->pool, &props) == cudaSuccess) {
            uint64_t thr_bytes = UINT64_MAX;
            cudaMemPoolSetAttribute(a->pool, cudaMemPoolAttrReleaseThreshold, &thr_bytes);
        } else {
            a->pool = nullptr;
        }
    }
    cudaGetLastError();
    *out = a;
    g_err.clear();
    return SEG_OK;
}

extern "C" int seg_create(const float *centroids, const int32_t *bundle_id, int64_t M, const float *thresh,
                          int32_t B, int device, seg_atlas **out) {
    return seg_create_ex(centroids, bundle_id, M, thresh, B, device, SEG_MODE_EXACT, out);
}

extern "C" int seg_get_atlas_info(const seg_atlas *a, seg_atlas_info *info) {
    if (!a || !info) return fail(SEG_EINVAL, "seg_get_atlas_info: null pointer");
    info->n_centroids = a->M;
    info->n_bundles = a->B;
    info->n_tiles = a->T;
    info->tile_size = TILE;
    info->device = a->device;
    info->device_bytes = a->bytes;
    info->mode = a->paper ? SEG_MODE_PAPER : SEG_MODE_EXACT;
    return SEG_OK;
}

// ----------------------------------------------------------------------------------------
// seg_classify
// ----------------------------------------------------------------------------------------
namespace {

constexpr int SORT_MIN_N = 4096;   // below this the prepass costs more than it saves

// Stream-ordered scratch from the atlas's pool; everything obtained is released (stream-ordered) when the
// holder goes out of scope, on every return path.
struct Scratch {
    cudaStream_t s;
    cudaMemPool_t pool;
    void *ptrs[8] = {};
    int n = 0;
    Scratch(cudaStream_t s_, cudaMemPool_t pool_) : s(s_), pool(pool_) {}
    Scratch(const Scratch &) = delete;
    Scratch &operator=(const Scratch &) = delete;
    template <class T>
    cudaError_t get(T **p, size_t bytes) {
        void *q = nullptr;
        if (n == 8) return cudaErrorMemoryAllocation;
        const cudaError_t e = pool ? cudaMallocFromPoolAsync(&q, bytes, pool, s) : cudaMallocAsync(&q, bytes, s);
        if (e != cudaSuccess) return e;
        ptrs[n++] = q;
        *p = static_cast<T *>(q);
        return cudaSuccess;
    }
    ~Scratch() {
        for (int i = 0; i < n; ++i) cudaFreeAsync(ptrs[i], s);
    }
};

// Device pointers, asynchronous on s.
int classify_device(const seg_atlas *a, const float *fib, int n, int32_t *lab, float *dist, cudaStream_t s,
                    unsigned long long *d_stats, const unsigned long long *seed = nullptr,
                    unsigned long long *keys = nullptr, uint32_t *masks = nullptr, int mwords = 0) {
    if (n == 0) return SEG_OK;
    cudaEvent_t *ev = nullptr;
    if (a->prof_n < a->prof_cap) ev = &a->prof_ev[4 * (a->prof_n++)];
    if (ev) SEG_CUDA(cudaEventRecord(ev[0], s), "seg_classify: profile event");
    Scratch sc(s, a->pool);
    uint32_t *key = nullptr, *hist = nullptr;
    int32_t *perm = nullptr;
    if (n >= SORT_MIN_N) {
        SEG_CUDA(sc.get(&key, sizeof(uint32_t) * (size_t)n), "seg_classify: scratch allocation");
        SEG_CUDA(sc.get(&perm, sizeof(int32_t) * (size_t)n), "seg_classify: scratch allocation");
        const int bits = morton_bits_for(n);
        SEG_CUDA(sc.get(&hist, sizeof(uint32_t) * morton_scratch_words(bits)), "seg_classify: scratch allocation");
        MortonParams mp{fib, n, a->lo, a->inv_cell, key, hist, hist + ((size_t)1 << (3 * bits)), perm, bits};
        SEG_CUDA(sc.get(&mp.rank, sizeof(uint32_t) * (size_t)n), "seg_classify: scratch allocation");
        SEG_CUDA(launch_morton_prepass(mp, s), "seg_classify: prepass launch");
    }
    uint32_t *tbits = nullptr;
    SEG_CUDA(sc.get(&tbits, sizeof(uint32_t) * cull_bits_words(n, a->T)), "seg_classify: scratch allocation");
    ClassifyParams cp{seed, fib, n, perm, lab, dist, a->tiles, a->th, a->ct, a->bh, a->B, a->T, d_stats, tbits, a->paper, keys,
                      nullptr, a->tiles_cm};
    cp.masks = masks;
    cp.mwords = mwords;
#ifndef SEG_NOPAPERSEED
    if (!masks) {   // k_cull names each fiber's seed candidate, k_classify evaluates it (no seed for multi-label)
#else
    if (!a->paper && !masks) {
#endif
        SEG_CUDA(sc.get(&cp.seed_code, sizeof(int32_t) * (size_t)n), "seg_classify: scratch allocation");
    }
#ifndef SEG_NO_LPT
#ifndef SEG_LPT_WAVES
#define SEG_LPT_WAVES 64
#endif
    {   // longest-list-first launch order (k_cta_order) where the grid's last wave is a visible share:
        // up to 64 waves of 2 CTAs per SM (cfg 1: -9%, cfg 3: -0.4%; cfg 4's 105 waves: +0.2% without it, and
        // again +0.15% with it at the end of round 2 -- the ordering kernel costs what the order saves)
        const int grid = (int)((n + classify_fibers_per_cta() - 1) / classify_fibers_per_cta());
        if (grid <= SEG_LPT_WAVES * 2 * a->sms)
            SEG_CUDA(sc.get(&cp.cta_order, sizeof(int32_t) * (size_t)grid), "seg_classify: scratch allocation");
    }
#endif
    if (ev) SEG_CUDA(cudaEventRecord(ev[1], s), "seg_classify: profile event");
    cudaError_t e = launch_classify(cp, d_stats != nullptr, s, ev ? ev[2] : nullptr);
    if (ev && e == cudaSuccess) e = cudaEventRecord(ev[3], s);
    if (e != cudaSuccess) return cuda_fail(e, "seg_classify: kernel launch");
    return SEG_OK;
}

// Device inputs are classified in slices of at most DEV_CHUNK fibers.  Fibers are independent, so the
// result does not depend on the slicing; it bounds the per-call scratch (Morton keys, bucket ranks,
// permutation and seed codes, 16 B per fiber; the per-CTA tile lists, (T + 2) x 2 B per 256 fibers) whatever N is.  Configurations
// up to 8.4 M fibers run as one slice.
constexpr int64_t DEV_CHUNK = int64_t(1) << 23;
int classify_device_sliced(const seg_atlas *a, const float *fib, int64_t N, int32_t *lab, float *dist,
                           cudaStream_t s, unsigned long long *d_stats, const unsigned long long *seed = nullptr,
                           unsigned long long *keys = nullptr, uint32_t *masks = nullptr, int mwords = 0) {
    // SEG_DEV_CHUNK (tests only): a smaller slice, to exercise the slicing at small N
    static const int64_t chunk = [] {
        const char *e = std::getenv("SEG_DEV_CHUNK");
        const long long v = e ? std::atoll(e) : 0;
        return v > 0 ? std::min<int64_t>(v, DEV_CHUNK) : DEV_CHUNK;
    }();
    for (int64_t c0 = 0; c0 < N; c0 += chunk) {
        const int n = (int)std::min<int64_t>(chunk, N - c0);
        const int rc = classify_device(a, fib + c0 * 3 * NPTS, n, lab ? lab + c0 : nullptr, dist ? dist + c0 : nullptr,
                                       s, d_stats, seed ? seed + c0 : nullptr, keys ? keys + c0 : nullptr,
                                       masks ? masks + c0 * mwords : nullptr, mwords);
        if (rc) return rc;
    }
    return SEG_OK;
}

// Host pointers: chunked H2D -> classify -> D2H over three streams (copy-in, the caller's stream
// for the kernels, copy-out) and NB device buffer sets, so that the host->device copy of chunk c+1
// runs while chunk c is classified and chunk c-1 is copied back.  Buffer set i is reused by chunk
// c + NB only after classify(c) has read its fibers (H2D waits on done[i]) and D2H(c) has read its
// results (classify waits on out[i]).  Synchronous: returns when every result is on the host.
int classify_host(const seg_atlas *a, const float *fib, int64_t N, int32_t *lab, float *dist, cudaStream_t s) {
    constexpr int64_t CH = 1 << 18;  // fibers per chunk (63 MB): the non-overlapped tail is one chunk
    constexpr int NBMAX = 3;
    const int64_t nchunks = (N + CH - 1) / CH;
    const int nb = (int)std::min<int64_t>(NBMAX, nchunks);
    const int64_t cap = std::min<int64_t>(N, CH);
    cudaStream_t cin = nullptr, cout = nullptr;
    SEG_CUDA(cudaStreamCreateWithFlags(&cin, cudaStreamNonBlocking), "seg_classify: cudaStreamCreate");
    if (cudaStreamCreateWithFlags(&cout, cudaStreamNonBlocking) != cudaSuccess) {
        cudaStreamDestroy(cin);
        return cuda_fail(cudaGetLastError(), "seg_classify: cudaStreamCreate");
    }
    cudaEvent_t ev_in[NBMAX] = {}, ev_done[NBMAX] = {}, ev_out[NBMAX] = {};
    float *dfib[NBMAX] = {};
    int32_t *dlab[NBMAX] = {};
    float *ddist[NBMAX] = {};
    int rc = SEG_OK;
    cudaError_t e = cudaSuccess;
    for (int i = 0; i < nb && e == cudaSuccess; ++i) {
        auto get = [&](void **p, size_t bytes) {
            return a->pool ? cudaMallocFromPoolAsync(p, bytes, a->pool, s) : cudaMallocAsync(p, bytes, s);
        };
        e = get((void **)&dfib[i], sizeof(float) * 3 * NPTS * cap);
        if (e == cudaSuccess) e = get((void **)&dlab[i], sizeof(int32_t) * cap);
        if (e == cudaSuccess) e = get((void **)&ddist[i], sizeof(float) * cap);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_in[i], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_done[i], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_out[i], cudaEventDisableTiming);
    }
    // the copy streams must see the allocations made on s
    cudaEvent_t ev_alloc = nullptr;
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_alloc, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(ev_alloc, s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cin, ev_alloc, 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cout, ev_alloc, 0);
    for (int64_t c = 0; c < nchunks && e == cudaSuccess && rc == SEG_OK; ++c) {
        const int i = (int)(c % nb);
        const int64_t lo = c * CH, n = std::min(CH, N - lo);
        if (c >= nb) e = cudaStreamWaitEvent(cin, ev_done[i], 0);   // classify(c - nb) read dfib[i]
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(dfib[i], fib + lo * 3 * NPTS, sizeof(float) * 3 * NPTS * n, cudaMemcpyHostToDevice, cin);
        if (e == cudaSuccess) e = cudaEventRecord(ev_in[i], cin);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ev_in[i], 0);
        if (e == cudaSuccess && c >= nb) e = cudaStreamWaitEvent(s, ev_out[i], 0);   // D2H(c - nb) read dlab[i]
        if (e != cudaSuccess) break;
        rc = classify_device(a, dfib[i], (int)n, dlab[i], ddist[i], s, nullptr);
        if (rc) break;
        e = cudaEventRecord(ev_done[i], s);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(cout, ev_done[i], 0);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(lab + lo, dlab[i], sizeof(int32_t) * n, cudaMemcpyDeviceToHost, cout);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(dist + lo, ddist[i], sizeof(float) * n, cudaMemcpyDeviceToHost, cout);
        if (e == cudaSuccess) e = cudaEventRecord(ev_out[i], cout);
    }
    cudaError_t e2 = cudaStreamSynchronize(cin);
    if (e == cudaSuccess) e = e2;
    e2 = cudaStreamSynchronize(cout);
    if (e == cudaSuccess) e = e2;
    // the frees are ordered after the last copies on s
    cudaEvent_t ev_fin = nullptr;
    if (cudaEventCreateWithFlags(&ev_fin, cudaEventDisableTiming) == cudaSuccess) {
        cudaEventRecord(ev_fin, cout);
        cudaStreamWaitEvent(s, ev_fin, 0);
    }
    for (int i = 0; i < nb; ++i) {
        if (dfib[i]) cudaFreeAsync(dfib[i], s);
        if (dlab[i]) cudaFreeAsync(dlab[i], s);
        if (ddist[i]) cudaFreeAsync(ddist[i], s);
        if (ev_in[i]) cudaEventDestroy(ev_in[i]);
        if (ev_done[i]) cudaEventDestroy(ev_done[i]);
        if (ev_out[i]) cudaEventDestroy(ev_out[i]);
    }
    e2 = cudaStreamSynchronize(s);
    if (e == cudaSuccess) e = e2;
    if (ev_alloc) cudaEventDestroy(ev_alloc);
    if (ev_fin) cudaEventDestroy(ev_fin);
    cudaStreamDestroy(cin);
    cudaStreamDestroy(cout);
    if (rc) return rc;
    if (e != cudaSuccess) return cuda_fail(e, "seg_classify: host-buffer pipeline");
    return SEG_OK;
}

int classify_common(const seg_atlas *a, const float *fibers, int64_t N, int32_t *label, float *dist, void *stream,
                    uint64_t *stats, const uint64_t *seed = nullptr) {
    if (!a) return fail(SEG_EINVAL, "seg_classify: null atlas");
    if (N < 0 || N > INT32_MAX) return fail(SEG_EINVAL, "seg_classify: N must be in [0, 2^31-1]");
    if (N == 0) {
        g_err.clear();
        return SEG_OK;
    }
    if (!fibers || !label || !dist) return fail(SEG_EINVAL, "seg_classify: null pointer with N > 0");
    if (((uintptr_t)fibers & 3) || ((uintptr_t)label & 3) || ((uintptr_t)dist & 3))
        return fail(SEG_EINVAL, "seg_classify: pointers must be 4-byte aligned");
    int d0 = -1, d1 = -1, d2 = -1;
    const int k0 = pointer_kind(fibers, &d0), k1 = pointer_kind(label, &d1), k2 = pointer_kind(dist, &d2);
    if (k0 < 0 || k1 < 0 || k2 < 0) return fail(SEG_ECUDA, "seg_classify: no usable CUDA device");
    if (k0 != k1 || k0 != k2) return fail(SEG_EINVAL, "seg_classify: fibers/label/dist mix host and device memory");
    if (k0 == 1 && d0 != a->device)
        return fail(SEG_EINVAL, "seg_classify: device pointer not on the atlas's device");
    if (k0 == 1) {
        // label / dist may live on a peer GPU the atlas's device can access (the fused gather, seg.h)
        for (int d : {d1, d2}) {
            if (d == a->device) continue;
            int ok = 0;
            if (cudaDeviceCanAccessPeer(&ok, a->device, d) != cudaSuccess || !ok) {
                cudaGetLastError();
                return fail(SEG_EINVAL, "seg_classify: label / dist on a device the atlas's device cannot access");
            }
            DeviceGuard pg(a->device);   // the kernel runs on the atlas's device: map the peer into it (idempotent)
            const cudaError_t pe = cudaDeviceEnablePeerAccess(d, 0);
            if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled)
                return cuda_fail(pe, "seg_classify: cudaDeviceEnablePeerAccess");
            cudaGetLastError();
        }
    }
    DeviceGuard guard(a->device);
    if (!guard.ok) return fail(SEG_ECUDA, "seg_classify: cudaSetDevice failed");
    cudaStream_t s = (cudaStream_t)stream;
    if (k0 == 0) {
        if (stats || seed) return fail(SEG_EINVAL, "seg_classify_stats / seeded: device pointers only");
        const int rc = classify_host(a, fibers, N, label, dist, s);
        if (!rc) g_err.clear();
        return rc;
    }
    unsigned long long *d_stats = nullptr;
    if (stats) {
        const size_t bytes = sizeof(unsigned long long) * SEG_NSTATS;
        SEG_CUDA(a->pool ? cudaMallocFromPoolAsync((void **)&d_stats, bytes, a->pool, s) : cudaMallocAsync((void **)&d_stats, bytes, s),
                 "seg_classify_stats: scratch allocation");
        const cudaError_t em = cudaMemsetAsync(d_stats, 0, bytes, s);
        if (em != cudaSuccess) {
            cudaFreeAsync(d_stats, s);   // freed on every path
            return cuda_fail(em, "seg_classify_stats: memset");
        }
    }
    int rc = classify_device_sliced(a, fibers, N, label, dist, s, d_stats,
                                    reinterpret_cast<const unsigned long long *>(seed));
    if (stats) {
        unsigned long long h[SEG_NSTATS];
        cudaError_t e = cudaMemcpyAsync(h, d_stats, sizeof(h), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        cudaFreeAsync(d_stats, s);
        if (!rc && e != cudaSuccess) return cuda_fail(e, "seg_classify_stats: readback");
        // the counters are added only when both the classification and the readback succeeded
        if (!rc && e == cudaSuccess)
            for (int k = 0; k < SEG_NSTATS; ++k) stats[k] += h[k];
    }
    if (!rc) g_err.clear();
    return rc;
}

}  // namespace

extern "C" int seg_classify(const seg_atlas *a, const float *fibers, int64_t N, int32_t *label, float *dist,
                            void *stream) {
    return classify_common(a, fibers, N, label, dist, stream, nullptr);
}

extern "C" int seg_classify_stats(const seg_atlas *a, const float *fibers, int64_t N, int32_t *label, float *dist,
                                  uint64_t *stats, void *stream) {
    if (!stats) return fail(SEG_EINVAL, "seg_classify_stats: null stats");
    return classify_common(a, fibers, N, label, dist, stream, stats);
}

// ----------------------------------------------------------------------------------------
// seg_group_by_bundle (row f3)
// ----------------------------------------------------------------------------------------
extern "C" int seg_group_by_bundle(const int32_t *label, const float *dist, int64_t N, int32_t B, int32_t *order,
                                   int64_t *offsets, float *dmin, float *dmax, double *dsum, void *stream) {
    if (N < 0 || N > INT32_MAX) return fail(SEG_EINVAL, "seg_group_by_bundle: N must be in [0, 2^31-1]");
    if (B < 1 || B > group_max_bundles())
        return fail(SEG_EINVAL, "seg_group_by_bundle: B must be in [1, " + std::to_string(group_max_bundles()) + "]");
    if (!offsets || (N > 0 && (!label || !order)))
        return fail(SEG_EINVAL, "seg_group_by_bundle: null pointer");
    const bool summ = dmin != nullptr;   // summaries requested
    if (summ && (!dmax || !dsum || (N > 0 && !dist)))
        return fail(SEG_EINVAL, "seg_group_by_bundle: summaries need dist (N > 0), dmin, dmax and dsum");
    if (!summ && (dmax || dsum))
        return fail(SEG_EINVAL, "seg_group_by_bundle: dmax / dsum without dmin");
    int dev = -1, d2 = -1;
    const void *ptrs[] = {label, dist, order, offsets, dmin, dmax, dsum};
    for (const void *q : ptrs) {
        if (!q) continue;
        const int k = pointer_kind(q, &d2);
        if (k < 0) return fail(SEG_ECUDA, "seg_group_by_bundle: no usable CUDA device");
        if (k != 1) return fail(SEG_EINVAL, "seg_group_by_bundle: all arrays must be device memory");
        if (dev >= 0 && d2 != dev) return fail(SEG_EINVAL, "seg_group_by_bundle: arrays on different devices");
        dev = d2;
    }
    DeviceGuard guard(dev);
    if (!guard.ok) return fail(SEG_ECUDA, "seg_group_by_bundle: cudaSetDevice failed");
    cudaStream_t s = (cudaStream_t)stream;
    uint32_t *scratch = nullptr;
    const size_t words = group_scratch_words(N, B);
    {
        cudaMemPool_t pool = lib_pool(dev);
        const size_t bytes = sizeof(uint32_t) * words;
        SEG_CUDA(pool ? cudaMallocFromPoolAsync((void **)&scratch, bytes, pool, s) : cudaMallocAsync((void **)&scratch, bytes, s),
                 "seg_group_by_bundle: scratch allocation");
    }
    GroupParams gp{};
    gp.label = label;
    gp.dist = summ ? dist : nullptr;
    gp.summ = summ ? 1 : 0;
    gp.n = N;
    gp.B = B;
    gp.hist = scratch;
    gp.total = scratch + (words - (size_t)(B + 1));
    gp.offsets = offsets;
    gp.order = order;
    gp.gmin = reinterpret_cast<uint32_t *>(dmin);
    gp.gmax = reinterpret_cast<uint32_t *>(dmax);
    gp.dsum = dsum;
    cudaError_t e = launch_group(gp, s);
    cudaFreeAsync(scratch, s);
    if (e != cudaSuccess) return cuda_fail(e, "seg_group_by_bundle: launch");
    g_err.clear();
    return SEG_OK;
}

// ----------------------------------------------------------------------------------------
// seg_resample (row f2)
// ----------------------------------------------------------------------------------------
extern "C" int seg_resample(const float *points, const int64_t *offsets, int64_t N, float *out, void *stream) {
    if (N < 0 || N > INT32_MAX) return fail(SEG_EINVAL, "seg_resample: N must be in [0, 2^31-1]");
    if (N == 0) {
        g_err.clear();
        return SEG_OK;
    }
    if (!points || !offsets || !out) return fail(SEG_EINVAL, "seg_resample: null pointer with N > 0");
    if (((uintptr_t)points & 3) || ((uintptr_t)offsets & 7) || ((uintptr_t)out & 3))
        return fail(SEG_EINVAL, "seg_resample: misaligned pointer");
    int dev = -1, d2 = -1;
    const void *ptrs[] = {points, offsets, out};
    for (const void *q : ptrs) {
        const int k = pointer_kind(q, &d2);
        if (k < 0) return fail(SEG_ECUDA, "seg_resample: no usable CUDA device");
        if (k != 1) return fail(SEG_EINVAL, "seg_resample: all arrays must be device memory");
        if (dev >= 0 && d2 != dev) return fail(SEG_EINVAL, "seg_resample: arrays on different devices");
        dev = d2;
    }
    DeviceGuard guard(dev);
    if (!guard.ok) return fail(SEG_ECUDA, "seg_resample: cudaSetDevice failed");
    int sms = 0;
    SEG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "seg_resample: device attribute");
    const ResampleParams rp{points, offsets, N, out};
    SEG_CUDA(launch_resample(rp, sms, (cudaStream_t)stream), "seg_resample: launch");
    g_err.clear();
    return SEG_OK;
}

// ----------------------------------------------------------------------------------------
// seg_classify_keys / seg_keys_to_labels (row f4)
// ----------------------------------------------------------------------------------------
extern "C" int seg_classify_keys(const seg_atlas *a, const float *fibers, int64_t N, uint64_t *keys, void *stream) {
    if (!a) return fail(SEG_EINVAL, "seg_classify_keys: null atlas");
    if (N < 0 || N > INT32_MAX) return fail(SEG_EINVAL, "seg_classify_keys: N must be in [0, 2^31-1]");
    if (N == 0) {
        g_err.clear();
        return SEG_OK;
    }
    if (!fibers || !keys) return fail(SEG_EINVAL, "seg_classify_keys: null pointer with N > 0");
    if (((uintptr_t)fibers & 3) || ((uintptr_t)keys & 7)) return fail(SEG_EINVAL, "seg_classify_keys: misaligned pointer");
    int d0 = -1, d1 = -1;
    const int k0 = pointer_kind(fibers, &d0), k1 = pointer_kind(keys, &d1);
    if (k0 < 0 || k1 < 0) return fail(SEG_ECUDA, "seg_classify_keys: no usable CUDA device");
    if (k0 != 1 || k1 != 1 || d0 != a->device || d1 != a->device)
        return fail(SEG_EINVAL, "seg_classify_keys: device pointers on the atlas's device only");
    DeviceGuard guard(a->device);
    if (!guard.ok) return fail(SEG_ECUDA, "seg_classify_keys: cudaSetDevice failed");
    const int rc = classify_device_sliced(a, fibers, N, nullptr, nullptr, (cudaStream_t)stream, nullptr, nullptr,
                                          reinterpret_cast<unsigned long long *>(keys));
    if (!rc) g_err.clear();
    return rc;
}

// ----------------------------------------------------------------------------------------
// seg_classify_multi (row f4's optional half: the original DWM multi-label assignment)
// ----------------------------------------------------------------------------------------
extern "C" int seg_classify_multi(const seg_atlas *a, const float *fibers, int64_t N, uint32_t *masks, int32_t words,
                                  void *stream) {
    if (!a) return fail(SEG_EINVAL, "seg_classify_multi: null atlas");
    if (a->paper) return fail(SEG_EINVAL, "seg_classify_multi: exact-mode atlases only");
    if (a->B > classify_multi_max_bundles())
        return fail(SEG_EINVAL, "seg_classify_multi: at most " + std::to_string(classify_multi_max_bundles()) + " bundles");
    if (words < (a->B + 31) / 32 || words > 1024)
        return fail(SEG_EINVAL, "seg_classify_multi: words must be in [ceil(B / 32), 1024]");
    if (N < 0 || N > INT32_MAX) return fail(SEG_EINVAL, "seg_classify_multi: N must be in [0, 2^31-1]");
    if (N == 0) {
        g_err.clear();
        return SEG_OK;
    }
    if (!fibers || !masks) return fail(SEG_EINVAL, "seg_classify_multi: null pointer with N > 0");
    if (((uintptr_t)fibers & 3) || ((uintptr_t)masks & 3)) return fail(SEG_EINVAL, "seg_classify_multi: misaligned pointer");
    int d0 = -1, d1 = -1;
    const int k0 = pointer_kind(fibers, &d0), k1 = pointer_kind(masks, &d1);
    if (k0 < 0 || k1 < 0) return fail(SEG_ECUDA, "seg_classify_multi: no usable CUDA device");
    if (k0 != 1 || k1 != 1 || d0 != a->device || d1 != a->device)
        return fail(SEG_EINVAL, "seg_classify_multi: device pointers on the atlas's device only");
    DeviceGuard guard(a->device);
    if (!guard.ok) return fail(SEG_ECUDA, "seg_classify_multi: cudaSetDevice failed");
    const int rc = classify_device_sliced(a, fibers, N, nullptr, nullptr, (cudaStream_t)stream, nullptr, nullptr,
                                          nullptr, masks, words);
    if (!rc) g_err.clear();
    return rc;
}

extern "C" int seg_keys_to_labels(const uint64_t *keys, int64_t N, int32_t mode, int32_t *label, float *dist,
                                  void *stream) {
    if (N < 0 || N > INT32_MAX) return fail(SEG_EINVAL, "seg_keys_to_labels: N must be in [0, 2^31-1]");
    if (mode != SEG_MODE_EXACT && mode != SEG_MODE_PAPER) return fail(SEG_EINVAL, "seg_keys_to_labels: unknown mode");
    if (N == 0) {
        g_err.clear();
        return SEG_OK;
    }
    if (!keys || !label || !dist) return fail(SEG_EINVAL, "seg_keys_to_labels: null pointer with N > 0");
    int dev = -1, d2 = -1;
    const void *ptrs[] = {keys, label, dist};
    for (const void *q : ptrs) {
        const int k = pointer_kind(q, &d2);
        if (k < 0) return fail(SEG_ECUDA, "seg_keys_to_labels: no usable CUDA device");
        if (k != 1) return fail(SEG_EINVAL, "seg_keys_to_labels: all arrays must be device memory");
        if (dev >= 0 && d2 != dev) return fail(SEG_EINVAL, "seg_keys_to_labels: arrays on different devices");
        dev = d2;
    }
    DeviceGuard guard(dev);
    if (!guard.ok) return fail(SEG_ECUDA, "seg_keys_to_labels: cudaSetDevice failed");
    SEG_CUDA(launch_keys_to_labels(reinterpret_cast<const unsigned long long *>(keys), N, mode == SEG_MODE_PAPER,
                                   label, dist, (cudaStream_t)stream),
             "seg_keys_to_labels: launch");
    g_err.clear();
    return SEG_OK;
}

extern "C" int seg_profile_enable(seg_atlas *a, int32_t cap) {
    if (!a || cap < 0) return fail(SEG_EINVAL, "seg_profile_enable: null atlas or negative capacity");
    DeviceGuard guard(a->device);
    free_prof(a);
    if (cap == 0) return SEG_OK;
    try {
        a->prof_ev.resize((size_t)4 * cap);
    } catch (const std::bad_alloc &) {
        return fail(SEG_ENOMEM, "seg_profile_enable: host allocation failed");
    }
    for (auto &e : a->prof_ev) {
        cudaError_t r = cudaEventCreate(&e);
        if (r != cudaSuccess) {
            e = nullptr;
            free_prof(a);
            return cuda_fail(r, "seg_profile_enable: cudaEventCreate");
        }
    }
    a->prof_cap = cap;
    a->prof_n = 0;
    return SEG_OK;
}

extern "C" int seg_profile_read(seg_atlas *a, float *prepass_ms, float *cull_ms, float *classify_ms, int32_t cap,
                                int32_t *count) {
    if (!a || !count) return fail(SEG_EINVAL, "seg_profile_read: null pointer");
    DeviceGuard guard(a->device);
    *count = a->prof_n;
    const int n = std::min(a->prof_n, std::max(0, (int)cap));
    for (int i = 0; i < n; ++i) {
        cudaEvent_t *ev = &a->prof_ev[4 * i];
        SEG_CUDA(cudaEventSynchronize(ev[3]), "seg_profile_read: cudaEventSynchronize");
        float t2 = 0.f;
        SEG_CUDA(cudaEventElapsedTime(&t2, ev[2], ev[3]), "seg_profile_read: elapsed");
        float t0 = 0.f, t1 = 0.f;
        SEG_CUDA(cudaEventElapsedTime(&t0, ev[0], ev[1]), "seg_profile_read: elapsed");
        SEG_CUDA(cudaEventElapsedTime(&t1, ev[1], ev[2]), "seg_profile_read: elapsed");
        if (prepass_ms) prepass_ms[i] = t0;
        if (cull_ms) cull_ms[i] = t1;
        if (classify_ms) classify_ms[i] = t2;
    }
    return SEG_OK;
}

extern "C" int seg_debug_classify_seeded(const seg_atlas *a, const float *fibers, int64_t N, const uint64_t *seed,
                                         int32_t *label, float *dist, uint64_t *stats, void *stream) {
    if (!seed && N > 0) return fail(SEG_EINVAL, "seg_debug_classify_seeded: null seed_keys");
    return classify_common(a, fibers, N, label, dist, stream, stats, seed);
}
