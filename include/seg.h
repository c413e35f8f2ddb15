/*
 * seg.h -- C ABI of libsegb200.so, the B200 (sm_100a) hot path of atlas-based
 * white-matter fiber segmentation (arXiv 1912.11494, "parallel segmentation",
 * Alg. 1).
 *
 * What the library computes (reading list: DESIGN.md Sec. 3):
 *   For every subject fiber a (21 points) and every atlas centroid c
 *   (21 points) the maximum Euclidean distance of Eq. 2
 *   (PAPER.md:73-76), min over the direct and the inverse point order:
 *       d_ME(a, c) = min( max_i ||a_i - c_i||, max_i ||a_i - c_{20-i}|| ),  i = 0..20.
 *   Each fiber is labelled with the bundle b of its closest centroid among the
 *   centroids with d_ME <= thr_b (the per-bundle threshold; "only the
 *   closest bundle"; Alg. 1 lines 13-16), ties to the
 *   lowest bundle id, label -1 when no bundle qualifies.  The paper's progressive
 *   discarding (test1 center point, test2 end points, test3 four points, test4 all 21
 *   points with early exit) and an exact bundle/tile
 *   lower-bound cull run inside the kernel; they are sound, so the result equals the
 *   plain definition above (up to FP32 rounding of the distances).
 *
 * Arithmetic: FP32 on the CUDA cores (squared distances, no sqrt except for the
 * returned distance, which is __fsqrt_rn of the winning squared distance).
 *
 * Data layout (all arrays C-contiguous, little endian):
 *   fibers / centroids  float32 [n][21][3]   (x,y,z of point 0, point 1, ..., point 20), mm
 *   bundle_id           int32   [M]          values in [0, B)
 *   thresh              float32 [B]          mm, finite and > 0
 *   label               int32   [N]          bundle id or -1
 *   dist                float32 [N]          d_ME of the winner in mm; +inf when label = -1;
 *                                            NaN (and label -1) for a fiber with a
 *                                            non-finite coordinate
 *
 * Error behaviour: every entry point returns SEG_OK (0) or a negative code and then
 * seg_last_error() (thread-local) describes the failure.  There is no CPU fallback:
 * without a usable CUDA device the calls fail with SEG_ECUDA.
 */
#ifndef SEG_H
#define SEG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SEG_NPTS 21 /* points per fiber and per centroid */

enum {
    SEG_OK = 0,
    SEG_EINVAL = -1, /* invalid argument (null pointer, size, range, alignment, non-finite) */
    SEG_ENOMEM = -2, /* host or device allocation failed */
    SEG_ECUDA = -3   /* CUDA runtime error or no usable device */
};

/* Opaque immutable atlas context living on one device. */
typedef struct seg_atlas seg_atlas;

/*
 * seg_create -- build an atlas context on `device` (-1 = the calling thread's current
 * device).  Groups centroids by bundle (the paper's atlasData[j]),
 * orders each bundle spatially, cuts it into tiles of 32 centroids that never cross a
 * bundle, and uploads the tiles plus per-tile / per-bundle bounding spheres and per-tile
 * axis-aligned boxes of points 0, 10 and 20 (the exact lower bounds of the cull: spheres for
 * the per-CTA tile lists, boxes for the live per-fiber test).
 *   centroids  float32 [M][21][3], host or device memory (detected)
 *   bundle_id  int32 [M] in [0, B), host or device memory
 *   M >= 1, B >= 1; thresh float32 [B], finite and > 0 (host or device memory)
 *   out        receives the context; set to NULL on error
 * The library copies everything; the caller may free its inputs on return.
 * Synchronous.  Bundles with no centroid are allowed (they never win).
 * Errors: SEG_EINVAL (null pointer, M < 1, B < 1, bundle id out of range, threshold
 * not finite or <= 0, non-finite centroid coordinate, more than 30,000 tiles -- i.e. roughly
 * 960,000 centroids -- in this build), SEG_ENOMEM, SEG_ECUDA.
 */
int seg_create(const float *centroids, const int32_t *bundle_id, int64_t M,
               const float *thresh, int32_t B, int device, seg_atlas **out);

/* Scoring modes of seg_create_ex. */
enum {
    SEG_MODE_EXACT = 0,  /* Eq. 2 d_ME, min over both orientations (BASELINE.json north_star) */
    SEG_MODE_PAPER = 1   /* the paper's final classifier: score =
                            d_ME in the orientation the end points infer (ties ->
                            direct) + TN of Eq. 3 on the chord lengths of the
                            21-point polylines (R16-R18); accept iff score <= thr;
                            dist = the score */
};

/*
 * seg_create_ex -- seg_create with a scoring mode in `flags` (SEG_MODE_EXACT or SEG_MODE_PAPER).
 * seg_create(...) is seg_create_ex(..., SEG_MODE_EXACT, out).  The cull, the discard cascade and
 * the closest-bundle rule are shared: every bound of the exact mode is a lower bound of the paper
 * score too (TN >= 0, and one orientation's maximum >= d_ME), so both modes are exact.
 * Errors as seg_create, plus SEG_EINVAL for unknown flag bits.
 */
int seg_create_ex(const float *centroids, const int32_t *bundle_id, int64_t M,
                  const float *thresh, int32_t B, int device, uint32_t flags, seg_atlas **out);

/*
 * seg_classify -- label N fibers (Alg. 1 over all fibers).
 *   fibers float32 [N][21][3]; label int32 [N]; dist float32 [N].
 *   Either all three pointers are device memory on the atlas's device (the call is
 *   then ASYNCHRONOUS on `stream`, a cudaStream_t; NULL = legacy default stream) -- label and dist
 *   may also be device memory of a PEER GPU the atlas's device can access (e.g. rank 0's result
 *   buffer mapped through CUDA IPC): the kernel's epilogue then stores each fiber's result straight
 *   into that GPU's memory over NVLink, which fuses the multi-GPU gather (SURVEY.md Sec. 8(e),
 *   PAPER.md:152 "no collision problems": one slot per fiber); the caller orders the completion
 *   (e.g. a stream-ordered collective after the call) before the peer reads -- or
 *   all three are host memory (pinned or pageable): the call then streams chunks
 *   host->device, classifies and copies the results back, overlapping the copies
 *   with the kernel, and returns after the results are in host memory.
 *   Internally a spatial-order prepass (Morton code of point 10) groups nearby fibers
 *   into the same warps; results are scattered back to the caller's order.
 *   Output is bitwise deterministic: independent of N, of the chunking, of the
 *   stream, of the GPU count and of the order of centroids in seg_create.
 *   Scratch is stream-ordered, from a memory pool the atlas owns (cached between calls, released by
 *   seg_destroy; the device's default pool is not touched).  fibers needs 4-byte alignment.
 *   Device-resident inputs run in slices of at most 2^23 fibers (bounded scratch: 16 B per fiber --
 *   Morton key, bucket rank, permutation, seed code -- plus 2 (T + 2) B per 256 fibers); fibers are independent, so the slicing changes no result.
 *   N = 0 is a no-op returning SEG_OK.
 * Errors: SEG_EINVAL (null atlas, null pointer with N > 0, N > 2^31 - 1, mixed host
 * and device pointers, fibers on another device, label / dist on a device the atlas's device
 * cannot access, misalignment),
 * SEG_ENOMEM, SEG_ECUDA (launch failure).  Asynchronous execution faults surface
 * at the caller's next synchronisation.
 */
int seg_classify(const seg_atlas *atlas, const float *fibers, int64_t N,
                 int32_t *label, float *dist, void *stream);

/* Number of counters written by seg_classify_stats. */
#define SEG_NSTATS 22
/*
 * seg_classify_stats -- seg_classify (device pointers only) with the kernel's
 * per-stage counters (SPEC.md:233-236 CascadeStats, extended), accumulated into the
 * HOST array stats[SEG_NSTATS] after a stream synchronisation:
 *   [0] fibers                [1] (warp, tile) pairs listed by the CTA pre-pass
 *   [2] (warp, tile) pairs computed (some lane passed the tile bound)
 *   [3] (lane, tile) pairs passing the tile bound    [4] lane midpoint tests (test1)
 *   [5] lane endpoint tests (test2)                  [6] lane orientation passes into test3/4
 *   [7] lane full 21-point completions               [8] best-distance updates (Alg. 1 l.15-16)
 *   [9] lane point-distance evaluations (Eq. 1, all stages and the bounds)
 *   [10] lane tile-bound tests (live, boxes)         [11] CTAs
 *   clock64 cycles summed over consumer warps: [12] tile loop, [13] waiting for a tile,
 *   [14] candidate selection (stack pushes, incl. the overflow rounds they trigger),
 *   [15] candidate rounds, [16] live tile-bound test, [17] fiber ingest (start -> first barrier)
 *   [18] candidate rounds run, [19] candidate lanes over those rounds, [20] fibers with a surviving
 *   orientation after test2 in a tile (stack pushes), [21] reserved (0)
 * A separate kernel instantiation; it computes the same labels and distances.
 */
int seg_classify_stats(const seg_atlas *atlas, const float *fibers, int64_t N,
                       int32_t *label, float *dist, uint64_t *stats, void *stream);

/*
 * seg_group_by_bundle -- row f3: the segmented bundles of a classified subject
 * (Fig. 1B).  From label[N] (and optionally dist[N]) as seg_classify writes them:
 *   order   int32 [N]   the fiber indices, STABLY partitioned by bundle: bundle 0's fibers in
 *                       increasing index, then bundle 1's, ..., then the unassigned ones (label -1,
 *                       or any label outside [0, B)) last
 *   offsets int64 [B+2] bundle b occupies order[offsets[b] .. offsets[b+1]); the unassigned ones
 *                       order[offsets[B] .. offsets[B+1]); offsets[B+1] = N
 *   dmin, dmax float [B], dsum double [B]  per-bundle min / max / sum of dist (dist >= 0 for every
 *                       labelled fiber, as seg_classify writes it); +inf / 0 / 0 for an empty
 *                       bundle.  Requested by a non-NULL dmin (then dmax, dsum and, for N > 0,
 *                       dist are required); all NULL = no summaries.
 *                       dsum is accumulated with floating-point atomics: its last bits may vary
 *                       between runs; order, offsets, dmin and dmax are bitwise deterministic.
 * All arrays are device memory on one device; ASYNCHRONOUS on `stream`; 1 <= B <= 4095.
 * Scratch comes from a stream-ordered pool the library keeps per device (cached between calls; the
 * device's default pool is not touched).
 * Errors: SEG_EINVAL (N < 0 or > 2^31-1, B out of range, null pointer, host memory, mixed devices),
 * SEG_ECUDA.
 */
int seg_group_by_bundle(const int32_t *label, const float *dist, int64_t N, int32_t B, int32_t *order,
                        int64_t *offsets, float *dmin, float *dmax, double *dsum, void *stream);

/*
 * seg_resample -- row f2: the step before the path.  Raw streamlines of any
 * length -> the 21-point fibers seg_classify takes ("resampled using 21 equidistant points",
 * PAPER.md:93): chord-length parameterisation with linear interpolation (reading R19,
 * SPEC.md:63-71).  Output point k is the polyline's point at arc length k * L / 20 (L = total chord
 * length), points 0 and 20 are the input end points exactly; arc lengths and interpolation in double,
 * each output coordinate rounded to FP32 once.
 *   points  float32 [P][3]; offsets int64 [N+1]: fiber f = points[offsets[f] .. offsets[f+1])
 *   out     float32 [N][21][3]
 * A fiber with fewer than 2 points, zero length (all points coincident) or non-finite points is
 * invalid input: its 63 outputs are NaN (seg_classify then labels it -1 / NaN).
 * All arrays device memory on one device; ASYNCHRONOUS on `stream`.  N = 0 is a no-op.
 * Errors: SEG_EINVAL (N out of range, null pointer with N > 0, host memory, mixed devices,
 * misalignment: points / out 4 B, offsets 8 B), SEG_ECUDA.
 */
int seg_resample(const float *points, const int64_t *offsets, int64_t N, float *out, void *stream);

/*
 * Row f4: atlas-sharded classification for atlases beyond one GPU's L2 / memory
 * or for more GPUs than subjects.  Each shard is an atlas built from a subset of the bundles (with
 * the global bundle count B, so labels stay global; the other bundles are empty).  seg_classify_keys
 * writes each fiber's best key over its shard; the element-wise MIN of the shards' keys (e.g. an
 * all_reduce MIN over int64) is the key of the whole atlas -- exact and deterministic, because a
 * key orders (value, bundle) lexicographically as Alg. 1's closest-bundle rule does (PAPER.md:129-133,
 * :163; ties -> lowest bundle).  seg_keys_to_labels decodes keys into seg_classify's label / dist.
 * Key space (all keys < 2^63, so signed and unsigned 64-bit MIN agree):
 *   (float bits of d^2 -- SEG_MODE_PAPER: of the score -- << 32) | bundle id,
 *   SEG_KEY_NONE (no bundle accepts the fiber), SEG_KEY_NONFINITE (non-finite fiber; every shard
 *   agrees).  Device pointers only, asynchronous on `stream`.  Errors as seg_classify (keys 8-B
 *   aligned); seg_keys_to_labels: SEG_EINVAL for an unknown mode.
 */
#define SEG_KEY_NONE 0x7fffffffffffffffULL
#define SEG_KEY_NONFINITE 0x7ffffffffffffffeULL
int seg_classify_keys(const seg_atlas *atlas, const float *fibers, int64_t N, uint64_t *keys, void *stream);
int seg_keys_to_labels(const uint64_t *keys, int64_t N, int32_t mode, int32_t *label, float *dist, void *stream);

/*
 * seg_classify_multi -- row f4's optional half: the original DWM multi-label
 * assignment the paper replaced by closest-bundle labelling.  For every fiber, bit b of
 * masks[n * words + b / 32] (bit b % 32) is set iff the bundle's minimum Eq. 2 distance is within its
 * threshold, D_b <= thr_b; words >= ceil(B / 32) (unused high words are written 0).  The cascade and cull
 * are the same, cut at each bundle's own threshold (no best-so-far across bundles); the closest-bundle
 * label of seg_classify is the argmin of D_b over the set bits.  A non-finite fiber gets an all-zero mask.
 * Exact-mode atlases with B <= 128.  Device pointers only, asynchronous on `stream`.
 * Errors: SEG_EINVAL (paper-mode atlas, B > 128, words out of range, N out of range, null or misaligned
 * (4 B) pointers, host memory or another device), SEG_ENOMEM, SEG_ECUDA.
 */
int seg_classify_multi(const seg_atlas *atlas, const float *fibers, int64_t N, uint32_t *masks, int32_t words,
                       void *stream);

/* Shape of a built atlas (for tests and the bench). */
typedef struct {
    int64_t n_centroids;  /* M */
    int32_t n_bundles;    /* B */
    int32_t n_tiles;      /* tiles of 32 centroids (bundle-aligned, padded) */
    int32_t tile_size;    /* 32 */
    int32_t device;       /* CUDA ordinal */
    int64_t device_bytes; /* device memory held by the context */
    int32_t mode;         /* SEG_MODE_EXACT or SEG_MODE_PAPER */
} seg_atlas_info;

int seg_get_atlas_info(const seg_atlas *atlas, seg_atlas_info *info);

/*
 * seg_plan_tiles -- the host half of seg_create, with no CUDA call: from HOST arrays
 * computes the tile plan.  For tile t (t < *n_tiles, at most max_tiles written):
 *   tile_bundle[t]          bundle id of the tile
 *   tile_members[t*32 + k]  index into the caller's centroids of slot k (padding slots
 *                           repeat a real member of the same bundle)
 *   tile_spheres[t*12 + 4*s + {0,1,2,3}]  centre xyz and radius of the bounding sphere of
 *                           point p_s over the tile's members, p = (0, 10, 20)
 * Lets host tests check the cull's soundness invariant without a GPU.
 * Errors: SEG_EINVAL as seg_create (host pointers only); SEG_ENOMEM.
 */
int seg_plan_tiles(const float *centroids, const int32_t *bundle_id, int64_t M, int32_t B,
                   int32_t max_tiles, int32_t *n_tiles, int32_t *tile_bundle,
                   int32_t *tile_members, float *tile_spheres);

/*
 * Profiling hook (bench.py only; NOT thread-safe, unlike the rest of the context):
 * after seg_profile_enable(atlas, cap) the first `cap` device-pointer seg_classify calls
 * on `atlas` (one record per slice of at most 2^23 fibers, see seg_classify) record CUDA
 * events on their stream before the spatial prepass, before the
 * tile-list kernel (k_cull), before the classify kernel and after it.  seg_profile_read
 * synchronises on those events and writes, per recorded call i < min(count, capacity),
 * prepass_ms[i], cull_ms[i] and classify_ms[i] (nullable host arrays);
 * *count receives the number of recorded calls.  cap = 0 disables and frees the events.
 * Errors: SEG_EINVAL (null atlas, cap < 0), SEG_ECUDA.
 */
int seg_profile_enable(seg_atlas *atlas, int32_t capacity);
int seg_profile_read(seg_atlas *atlas, float *prepass_ms, float *cull_ms, float *classify_ms,
                     int32_t capacity, int32_t *count);

/*
 * seg_debug_classify_seeded -- experiment hook (device pointers only): seg_classify with each
 * fiber's running best initialised from seed_keys[N] (device uint64, caller order), key =
 * (float bits of a squared distance << 32) | bundle id, or ~0 for none.  The result equals
 * seg_classify's whenever every seed is an upper bound of the fiber's true best key, e.g.
 * (d^2 rounded up, label) from an earlier run; it measures how much of the kernel's work a
 * perfect best-first order would save.  Errors as seg_classify.
 */
int seg_debug_classify_seeded(const seg_atlas *atlas, const float *fibers, int64_t N,
                              const uint64_t *seed_keys, int32_t *label, float *dist,
                              uint64_t *stats /* nullable host [SEG_NSTATS] */, void *stream);

/* Destroy a context (NULL-safe).  Must not race an in-flight seg_classify. */
void seg_destroy(seg_atlas *atlas);

/* Thread-local description of the last error ("" if none). */
const char *seg_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* SEG_H */
