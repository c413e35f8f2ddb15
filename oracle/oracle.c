/*
 * oracle.c -- plain, slow, double-precision CPU oracle for the segmentation hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke(), bench.py's
 * cpu_baseline / --impl reference legs and the committed scripts that cache oracle outputs
 * (scripts/oracle_full.py) may load this library.  The product path (paper_1912_11494_b200/)
 * never links, imports or executes it, and this file shares no code, header, table or
 * constant generator with the CUDA path.
 *
 * What it computes is the plain definition of the method's result (SURVEY.md
 * Sec. 8(c), steps 1-6); the method's discard cascade (test1..test4,
 * PAPER.md:97-99) is sound pruning and therefore reaches this same result, so the
 * plain oracle evaluates every (fiber, centroid) pair with no discarding, no blocking
 * and no reordering:
 *
 *   Eq. 1 (Sec. 2.3):  d_E(a_i, b_i) = || a_i - b_i ||_2
 *   Eq. 2 (Sec. 2.3):  d_ME(a, b) = min( max_i d_E(a_i, b_i),
 *                                                      max_i d_E(a_i, b_{N-i}) )
 *          with 0-based indices, b_{N-i} read as b_{20-i} (reading R1),
 *   labelling (Alg. 1 lines 13-16; "only the
 *          closest bundle"; PAPER.md:64 per-bundle threshold):
 *          label(a) = argmin_b { D_b(a) : D_b(a) <= thr_b },  D_b = min_{c in b} d_ME(a, c),
 *          ties -> lowest bundle id (Alg. 1 updates on strict '<' with j ascending,
 *          PAPER.md:130, reading R5), -1 when no bundle qualifies (reading R8).
 *
 * Arithmetic: every FP32 input is promoted to double; squared distances are
 * compared (monotone, so the argmin/threshold decisions equal those on distances);
 * dist = sqrt(D^2) of the winner, +inf when unlabelled, NaN for a non-finite fiber
 * (reading R12).
 *
 * Tie band (BASELINE.json north_star "1e-3 mm from its
 * threshold and from the runner-up bundle"): decidable[n] = 1 iff the fiber's label
 * is not within delta of a threshold or of a runner-up bundle; only decidable
 * fibers are held to exact label equality by the parity tests.
 *
 * Sound-discard variants (oracle_classify_sound, oracle_classify_paper_sound; SURVEY.md
 * Sec. 8(c) step 7): the paper's own Alg. 1 loop -- per fiber, every
 * centroid, discardCenter (test1, point 10), discardExtremes (test2, end points),
 * discardFourPoints (test3, points 3/7/13/17), discarded21points (test4, the rest) with an
 * early exit after every pairwise distance -- but cut at
 * (thr_b + 2 delta)^2 instead of thr_b^2.  Every value the labelling and the tie band read
 * (those up to thr_b + delta) is therefore computed exactly as the plain oracle computes it
 * (the same oracle_point_d2 values, and a maximum does not depend on the order it is taken
 * in), so label, dist and decidable are bitwise those of the plain definition; only values
 * beyond the cut, which no decision reads, are left out.  tests/test_oracle_sound.py pins
 * that equality.  These variants make full-size oracle runs affordable (configs 3-4).
 *
 * Parity pins: tests/test_oracle_pins.py, tests/test_oracle_paper_pins.py,
 * tests/test_oracle_sound.py (closed forms, SPEC worked examples under tests/golden/,
 * invariants, a library special case, brute force on tiny inputs, constructed tie-band
 * cases).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#define NPTS 21

/* Orientation band of reading R20 (paper mode): 2^-18 relative on the squared end-point
 * maxima, 32x the error of a FP32 evaluation of either maximum (<= 8 ulp relative). */
#define ORIENT_REL 0x1p-18

/* Eq. 1, squared: ||p - q||^2 in double. */
double oracle_point_d2(const float *p, const float *q)
{
    double dx = (double)p[0] - (double)q[0];
    double dy = (double)p[1] - (double)q[1];
    double dz = (double)p[2] - (double)q[2];
    return dx * dx + dy * dy + dz * dz;
}

/* One inner term of Eq. 2, squared: max_i d_E(a_i, b_i)^2 (inverse = 0) or
 * max_i d_E(a_i, b_{20-i})^2 (inverse = 1). */
double oracle_max_pointwise_d2(const float *a, const float *b, int inverse)
{
    double m = 0.0;
    for (int i = 0; i < NPTS; i++) {
        int j = inverse ? (NPTS - 1 - i) : i;
        double d2 = oracle_point_d2(a + 3 * i, b + 3 * j);
        if (d2 > m)
            m = d2;
    }
    return m;
}

/* Eq. 2, squared: min over the direct and the inverse orientation. */
double oracle_dme_d2(const float *a, const float *b)
{
    double dd = oracle_max_pointwise_d2(a, b, 0);
    double di = oracle_max_pointwise_d2(a, b, 1);
    return dd < di ? dd : di;
}

/* Eq. 2 in mm. */
double oracle_dme(const float *a, const float *b)
{
    return sqrt(oracle_dme_d2(a, b));
}

static int fiber_is_finite(const float *f)
{
    for (int i = 0; i < 3 * NPTS; i++)
        if (!isfinite(f[i]))
            return 0;
    return 1;
}

static int bundle_ids_valid(const int32_t *bundle_id, int64_t M, int32_t B)
{
    for (int64_t m = 0; m < M; m++)
        if (bundle_id[m] < 0 || bundle_id[m] >= B)
            return 0;
    return 1;
}

/* Steps 4-6 of SURVEY.md Sec. 8(c) on the per-bundle minima Db (squared, double). */
static void label_exact(const double *Db, const float *thresh, int32_t B, double delta,
                        int32_t *label, double *dist, uint8_t *decidable)
{
    /* step 4-5: accepted set {b : D_b^2 <= thr_b^2}; closest, ties -> lowest b */
    int32_t best = -1;
    for (int32_t b = 0; b < B; b++) {
        double t = (double)thresh[b];
        if (Db[b] <= t * t && (best < 0 || Db[b] < Db[best]))
            best = b;
    }
    *label = best;
    *dist = best < 0 ? INFINITY : sqrt(Db[best]);
    /* step 6: tie band.  P = {b : d_b <= thr_b + delta}; b* = argmin_P d_b;
     * decidable iff P empty, or d_b* < thr_b* - delta and every other b in P
     * has d_b > d_b* + delta. */
    int32_t bs = -1;
    for (int32_t b = 0; b < B; b++) {
        double d = sqrt(Db[b]);
        if (d <= (double)thresh[b] + delta && (bs < 0 || d < sqrt(Db[bs])))
            bs = b;
    }
    int ok = 1;
    if (bs >= 0) {
        double ds = sqrt(Db[bs]);
        if (!(ds < (double)thresh[bs] - delta))
            ok = 0;
        for (int32_t b = 0; b < B && ok; b++) {
            if (b == bs)
                continue;
            double d = sqrt(Db[b]);
            if (d <= (double)thresh[b] + delta && !(d > ds + delta))
                ok = 0;
        }
    }
    *decidable = (uint8_t)ok;
}

/*
 * Classify n fibers against the atlas by the plain definition.
 *   fibers     float [n][21][3]
 *   centroids  float [M][21][3], bundle_id int32 [M] in [0, B), thresh float [B]
 *   delta      tie-band half width in mm (1e-3 for the parity tests)
 * Outputs (caller-owned, length n): label int32, dist double, decidable uint8;
 *   d2b (nullable) double [n][B] = per-bundle minimum of d_ME^2 (+inf for an empty bundle).
 * Returns 0, or -1 on invalid arguments (a bundle id out of range).
 */
int oracle_classify(const float *fibers, int64_t n,
                    const float *centroids, const int32_t *bundle_id, int64_t M,
                    const float *thresh, int32_t B, double delta,
                    int32_t *label, double *dist, uint8_t *decidable, double *d2b)
{
    if (!bundle_ids_valid(bundle_id, M, B))
        return -1;
    double *Db = (double *)malloc(sizeof(double) * (size_t)B);
    if (!Db)
        return -1;
    for (int64_t f = 0; f < n; f++) {
        const float *a = fibers + (size_t)f * 3 * NPTS;
        /* step 2-3: per-bundle minimum of d_ME^2 over all centroids, no discarding */
        for (int32_t b = 0; b < B; b++)
            Db[b] = INFINITY;
        for (int64_t m = 0; m < M; m++) {
            double d2 = oracle_dme_d2(a, centroids + (size_t)m * 3 * NPTS);
            if (d2 < Db[bundle_id[m]])
                Db[bundle_id[m]] = d2;
        }
        if (d2b)
            for (int32_t b = 0; b < B; b++)
                d2b[(size_t)f * B + b] = Db[b];
        if (!fiber_is_finite(a)) {
            label[f] = -1;
            dist[f] = NAN;
            decidable[f] = 1;
            continue;
        }
        label_exact(Db, thresh, B, delta, &label[f], &dist[f], &decidable[f]);
    }
    free(Db);
    return 0;
}

/* A contiguous copy of every centroid's point 10 (float [M][3], the input values unchanged): test1
 * reads 12 B per centroid instead of a 252-B record, so the sound variants stream 0.5 MB, not the
 * whole atlas, per fiber.  A copy of the inputs, no change to any arithmetic. */
static float *midpoint_copy(const float *centroids, int64_t M)
{
    float *c10 = (float *)malloc(sizeof(float) * 3 * (size_t)(M > 0 ? M : 1));
    if (c10)
        for (int64_t m = 0; m < M; m++)
            for (int k = 0; k < 3; k++)
                c10[3 * m + k] = centroids[(size_t)m * 3 * NPTS + 30 + k];
    return c10;
}

/* test3 points first ("4 intermediate points", indices 3/7/13/17 after SPEC.md:230,
 * reading R7), then the remaining points of test4; 0, 10 and 20 are tests 1-2. */
static const int CASCADE_REST[NPTS - 3] = {3, 7, 13, 17, 1, 2, 4, 5, 6, 8, 9, 11, 12, 14, 15, 16, 18, 19};

/* Running maximum of d_E^2 over the test3/test4 points of one orientation, starting from r, with
 * the early exit "after each pairwise distance": returns the exact maximum when it
 * stays <= cut, else some value > cut. */
static double cascade_rest(const float *a, const float *c, int inverse, double r, double cut)
{
    for (int k = 0; k < NPTS - 3 && r <= cut; k++) {
        int i = CASCADE_REST[k];
        int j = inverse ? (NPTS - 1 - i) : i;
        double d2 = oracle_point_d2(a + 3 * i, c + 3 * j);
        if (d2 > r)
            r = d2;
    }
    return r;
}

/*
 * The sound-discard variant of oracle_classify (see the header): same arguments and outputs,
 * without d2b.  Bitwise the plain definition's label, dist and decidable.
 */
int oracle_classify_sound(const float *fibers, int64_t n,
                          const float *centroids, const int32_t *bundle_id, int64_t M,
                          const float *thresh, int32_t B, double delta,
                          int32_t *label, double *dist, uint8_t *decidable)
{
    if (!bundle_ids_valid(bundle_id, M, B))
        return -1;
    double *Db = (double *)malloc(sizeof(double) * (size_t)B);
    double *cut = (double *)malloc(sizeof(double) * (size_t)B);
    float *c10 = midpoint_copy(centroids, M);
    if (!Db || !cut || !c10) {
        free(Db);
        free(cut);
        free(c10);
        return -1;
    }
    for (int32_t b = 0; b < B; b++) {
        double t = (double)thresh[b] + 2.0 * delta;
        cut[b] = t * t;
    }
    for (int64_t f = 0; f < n; f++) {
        const float *a = fibers + (size_t)f * 3 * NPTS;
        if (!fiber_is_finite(a)) {
            label[f] = -1;
            dist[f] = NAN;
            decidable[f] = 1;
            continue;
        }
        for (int32_t b = 0; b < B; b++)
            Db[b] = INFINITY;
        for (int64_t m = 0; m < M; m++) {
            const float *c = centroids + (size_t)m * 3 * NPTS;
            const int32_t b = bundle_id[m];
            const double cb = cut[b];
            /* test1, discardCenter: point 10 pairs with itself in both orientations */
            double m10 = oracle_point_d2(a + 30, c10 + 3 * m);
            if (m10 > cb)
                continue;
            /* test2, discardExtremes: the end points, each orientation */
            double e00 = oracle_point_d2(a, c), e2020 = oracle_point_d2(a + 60, c + 60);
            double e020 = oracle_point_d2(a, c + 60), e200 = oracle_point_d2(a + 60, c);
            double rd = m10, ri = m10;
            if (e00 > rd) rd = e00;
            if (e2020 > rd) rd = e2020;
            if (e020 > ri) ri = e020;
            if (e200 > ri) ri = e200;
            if (rd > cb && ri > cb)
                continue;
            /* test3 + test4 with early exit, per orientation still alive */
            if (rd <= cb)
                rd = cascade_rest(a, c, 0, rd, cb);
            if (ri <= cb)
                ri = cascade_rest(a, c, 1, ri, cb);
            double d2 = rd < ri ? rd : ri;
            if (d2 <= cb && d2 < Db[b])
                Db[b] = d2;
        }
        label_exact(Db, thresh, B, delta, &label[f], &dist[f], &decidable[f]);
    }
    free(Db);
    free(cut);
    free(c10);
    return 0;
}

/* ======================================================================================
 * Paper-semantics mode: the paper's final classifier.
 *
 *   Eq. 3:  TN = ( |l_S - l_C| / max(l_S, l_C) + 1 )^2 - 1, added to d_ME:
 *          "the complete distance metric (d_ME + TN)".  Discarding a pair
 *          before TN when the distance already exceeds the threshold is sound
 *          because TN >= 0, so it does not change the result and the plain oracle omits it.
 *   Lengths: the chord length of the 21-point resampled polyline (reading R16,
 *          after SPEC.md:124).
 *   Orientation: the optimised algorithm "uses the distances computed in [the] second
 *          discarding stage to determine the direction of the fiber" and evaluates the later
 *          stages in that direction only: orientation = argmin of the two
 *          end-point maxima m_dir = max(d(a_0,c_0), d(a_20,c_20)), m_inv = max(d(a_0,c_20),
 *          d(a_20,c_0)), ties -> direct (reading R17, after SPEC.md:251), decided in double.
 *   Orientation band (reading R20): the paper fixes no precision for that decision, and an
 *          FP32 implementation can decide a near-tie either way.  A pair is orientation-
 *          ambiguous when |m_dir^2 - m_inv^2| <= ORIENT_REL * max(m_dir^2, m_inv^2); both of
 *          its orientations' scores are then correct answers for that pair.
 *   score(a, c) = max_i d_E(a_i, c_o(i)) + TN  in double, o the inferred orientation;
 *   label(a) = argmin_b { S_b(a) : S_b(a) <= thr_b },  S_b = min_{c in b} score(a, c),
 *          ties -> lowest bundle id, -1 when none qualifies; dist = S_label.
 *   Tie band: per bundle the interval [L_b, H_b] of the values S_b can take over every
 *          choice on the ambiguous pairs (L_b = min_c of the smaller possible score, H_b =
 *          min_c of the larger); L_b = H_b = S_b when no pair of b is ambiguous.  A fiber is
 *          decidable iff P = {b : L_b <= thr_b + delta} is empty, or its winner b* (argmin_P
 *          S_b) has L_b* = H_b* < thr_b* - delta and every other b in P has L_b > H_b* + delta.
 *          With no ambiguous pair this is exactly the exact mode's rule on S_b.
 * ====================================================================================== */

/* Chord length of a 21-point polyline, in mm (double). */
double oracle_polyline_length(const float *a)
{
    double l = 0.0;
    for (int i = 0; i + 1 < NPTS; i++)
        l += sqrt(oracle_point_d2(a + 3 * i, a + 3 * (i + 1)));
    return l;
}

/* Eq. 3. */
double oracle_tn(double ls, double lc)
{
    double mx = ls > lc ? ls : lc;
    double q = fabs(ls - lc) / mx + 1.0;
    return q * q - 1.0;
}

/* The squared end-point maxima of the direct and the inverse orientation (double). */
static void endpoint_maxima_d2(const float *a, const float *c, double *mdir, double *minv)
{
    const float *a0 = a, *a20 = a + 3 * (NPTS - 1), *c0 = c, *c20 = c + 3 * (NPTS - 1);
    double e00 = oracle_point_d2(a0, c0), e2020 = oracle_point_d2(a20, c20);
    double e020 = oracle_point_d2(a0, c20), e200 = oracle_point_d2(a20, c0);
    *mdir = e00 > e2020 ? e00 : e2020;
    *minv = e020 > e200 ? e020 : e200;
}

static int orientation_of(double mdir, double minv)
{
    return minv < mdir ? 1 : 0;
}

static int ambiguous_of(double mdir, double minv)
{
    double mx = mdir > minv ? mdir : minv;
    return fabs(mdir - minv) <= ORIENT_REL * mx;
}

/* 1 = inverse, 0 = direct: the argmin of the end-point maxima, ties -> direct (double). */
int oracle_endpoint_orientation(const float *a, const float *c)
{
    double mdir, minv;
    endpoint_maxima_d2(a, c, &mdir, &minv);
    return orientation_of(mdir, minv);
}

/* 1 iff the orientation decision of the pair lies inside the band of reading R20. */
int oracle_orientation_ambiguous(const float *a, const float *c)
{
    double mdir, minv;
    endpoint_maxima_d2(a, c, &mdir, &minv);
    return ambiguous_of(mdir, minv);
}

/* The complete metric of one pair in the inferred orientation, in mm. */
double oracle_paper_score(const float *a, const float *c)
{
    int o = oracle_endpoint_orientation(a, c);
    return sqrt(oracle_max_pointwise_d2(a, c, o)) + oracle_tn(oracle_polyline_length(a), oracle_polyline_length(c));
}

/* Alg. 1's closest-bundle labelling on the decided per-bundle scores S and the tie band on the
 * intervals [L_b, H_b] (all in mm); see the header of this section. */
static void label_paper(const double *S, const double *L, const double *H, const float *thresh, int32_t B,
                        double delta, int32_t *label, double *dist, uint8_t *decidable)
{
    int32_t best = -1;
    for (int32_t b = 0; b < B; b++)
        if (S[b] <= (double)thresh[b] && (best < 0 || S[b] < S[best]))
            best = b;
    *label = best;
    *dist = best < 0 ? INFINITY : S[best];
    int32_t bs = -1;
    for (int32_t b = 0; b < B; b++)
        if (L[b] <= (double)thresh[b] + delta && (bs < 0 || S[b] < S[bs]))
            bs = b;
    int ok = 1;
    if (bs >= 0) {
        if (!(L[bs] == H[bs] && H[bs] < (double)thresh[bs] - delta))
            ok = 0;
        for (int32_t b = 0; b < B && ok; b++)
            if (b != bs && L[b] <= (double)thresh[b] + delta && !(L[b] > H[bs] + delta))
                ok = 0;
    }
    *decidable = (uint8_t)ok;
}

static double *alloc_doubles(int64_t k)
{
    return (double *)malloc(sizeof(double) * (size_t)(k > 0 ? k : 1));
}

static double *centroid_lengths(const float *centroids, int64_t M)
{
    double *lc = alloc_doubles(M);
    if (lc)
        for (int64_t m = 0; m < M; m++)
            lc[m] = oracle_polyline_length(centroids + (size_t)m * 3 * NPTS);
    return lc;
}

/*
 * Classify n fibers by the paper's complete metric (plain definition, every pair, no
 * discarding).  Arguments and outputs as oracle_classify; dist = the winning score;
 * sb, sb_lo, sb_hi (each nullable) double [n][B] = per-bundle S_b, L_b, H_b (mm; +inf for an
 * empty bundle, NaN for a non-finite fiber).
 */
int oracle_classify_paper(const float *fibers, int64_t n,
                          const float *centroids, const int32_t *bundle_id, int64_t M,
                          const float *thresh, int32_t B, double delta,
                          int32_t *label, double *dist, uint8_t *decidable,
                          double *sb, double *sb_lo, double *sb_hi)
{
    if (!bundle_ids_valid(bundle_id, M, B))
        return -1;
    double *S = alloc_doubles(B), *L = alloc_doubles(B), *H = alloc_doubles(B);
    double *lc = centroid_lengths(centroids, M);
    if (!S || !L || !H || !lc) {
        free(S); free(L); free(H); free(lc);
        return -1;
    }
    for (int64_t f = 0; f < n; f++) {
        const float *a = fibers + (size_t)f * 3 * NPTS;
        if (!fiber_is_finite(a)) {
            label[f] = -1;
            dist[f] = NAN;
            decidable[f] = 1;
            for (int32_t b = 0; b < B; b++) {
                if (sb) sb[(size_t)f * B + b] = NAN;
                if (sb_lo) sb_lo[(size_t)f * B + b] = NAN;
                if (sb_hi) sb_hi[(size_t)f * B + b] = NAN;
            }
            continue;
        }
        for (int32_t b = 0; b < B; b++)
            S[b] = L[b] = H[b] = INFINITY;
        const double ls = oracle_polyline_length(a);
        for (int64_t m = 0; m < M; m++) {
            const float *c = centroids + (size_t)m * 3 * NPTS;
            const int32_t b = bundle_id[m];
            double mdir, minv;
            endpoint_maxima_d2(a, c, &mdir, &minv);
            const int o = orientation_of(mdir, minv);
            const double tn = oracle_tn(ls, lc[m]);
            const double s = sqrt(oracle_max_pointwise_d2(a, c, o)) + tn;
            double lo = s, hi = s;
            if (ambiguous_of(mdir, minv)) {
                const double s2 = sqrt(oracle_max_pointwise_d2(a, c, 1 - o)) + tn;
                lo = s < s2 ? s : s2;
                hi = s < s2 ? s2 : s;
            }
            if (s < S[b]) S[b] = s;
            if (lo < L[b]) L[b] = lo;
            if (hi < H[b]) H[b] = hi;
        }
        for (int32_t b = 0; b < B; b++) {
            if (sb) sb[(size_t)f * B + b] = S[b];
            if (sb_lo) sb_lo[(size_t)f * B + b] = L[b];
            if (sb_hi) sb_hi[(size_t)f * B + b] = H[b];
        }
        label_paper(S, L, H, thresh, B, delta, &label[f], &dist[f], &decidable[f]);
    }
    free(S); free(L); free(H); free(lc);
    return 0;
}

/*
 * The sound-discard variant of oracle_classify_paper (see the file header): Alg. 1's cascade
 * per evaluated orientation -- the inferred one, both for an ambiguous pair -- cut at
 * (thr_b + 2 delta)^2 on the running maximum (score >= that maximum since TN >= 0), TN only
 * for the survivors.  Bitwise the plain definition's label, dist, decidable.
 */
int oracle_classify_paper_sound(const float *fibers, int64_t n,
                                const float *centroids, const int32_t *bundle_id, int64_t M,
                                const float *thresh, int32_t B, double delta,
                                int32_t *label, double *dist, uint8_t *decidable)
{
    if (!bundle_ids_valid(bundle_id, M, B))
        return -1;
    double *S = alloc_doubles(B), *L = alloc_doubles(B), *H = alloc_doubles(B), *cut = alloc_doubles(B);
    double *lc = centroid_lengths(centroids, M);
    float *c10 = midpoint_copy(centroids, M);
    if (!S || !L || !H || !cut || !lc || !c10) {
        free(S); free(L); free(H); free(cut); free(lc); free(c10);
        return -1;
    }
    for (int32_t b = 0; b < B; b++) {
        double t = (double)thresh[b] + 2.0 * delta;
        cut[b] = t * t;
    }
    for (int64_t f = 0; f < n; f++) {
        const float *a = fibers + (size_t)f * 3 * NPTS;
        if (!fiber_is_finite(a)) {
            label[f] = -1;
            dist[f] = NAN;
            decidable[f] = 1;
            continue;
        }
        for (int32_t b = 0; b < B; b++)
            S[b] = L[b] = H[b] = INFINITY;
        const double ls = oracle_polyline_length(a);
        for (int64_t m = 0; m < M; m++) {
            const float *c = centroids + (size_t)m * 3 * NPTS;
            const int32_t b = bundle_id[m];
            const double cb = cut[b];
            /* test1: point 10 bounds either orientation's maximum */
            double m10 = oracle_point_d2(a + 30, c10 + 3 * m);
            if (m10 > cb)
                continue;
            /* test2: the end points decide the orientation (both when ambiguous) */
            double mdir, minv;
            endpoint_maxima_d2(a, c, &mdir, &minv);
            const int o = orientation_of(mdir, minv);
            const int amb = ambiguous_of(mdir, minv);
            double r[2] = {INFINITY, INFINITY};   /* running maximum per orientation, inf = not evaluated */
            for (int q = 0; q < 2; q++) {
                if (q != o && !amb)
                    continue;
                double rq = m10;
                double e = q ? minv : mdir;
                if (e > rq) rq = e;
                if (rq > cb)
                    continue;
                /* test3 + test4 with early exit */
                r[q] = cascade_rest(a, c, q, rq, cb);
            }
            double s[2];
            for (int q = 0; q < 2; q++)   /* TN only for the survivors */
                s[q] = r[q] <= cb ? sqrt(r[q]) + oracle_tn(ls, lc[m]) : INFINITY;
            const double sd = s[o];
            double lo = sd, hi = sd;
            if (amb) {
                lo = s[0] < s[1] ? s[0] : s[1];
                hi = s[0] < s[1] ? s[1] : s[0];
            }
            if (sd < S[b]) S[b] = sd;
            if (lo < L[b]) L[b] = lo;
            if (hi < H[b]) H[b] = hi;
        }
        label_paper(S, L, H, thresh, B, delta, &label[f], &dist[f], &decidable[f]);
    }
    free(S); free(L); free(H); free(cut); free(lc); free(c10);
    return 0;
}

/* ======================================================================================
 * Multi-label output (optional half): the original DWM behaviour the
 * paper replaced by closest-bundle labelling ("... a fiber could be assigned to
 * several bundles").  Plain definition: per fiber, bit b of the mask is set iff D_b <= thr_b
 * (D_b = min over the bundle's centroids of Eq. 2's d_ME, as in oracle_classify), B <= 32 * words.
 * amb (nullable) marks the bits the tie band leaves open: |d_b - thr_b| <= delta.  A non-finite
 * fiber gets an all-zero mask (reading R12: it is unassigned).
 * ====================================================================================== */
int oracle_classify_multi(const float *fibers, int64_t n,
                          const float *centroids, const int32_t *bundle_id, int64_t M,
                          const float *thresh, int32_t B, double delta, int32_t words,
                          uint32_t *mask, uint32_t *amb)
{
    if (!bundle_ids_valid(bundle_id, M, B) || words < 1 || B > 32 * words)
        return -1;
    double *Db = alloc_doubles(B);
    if (!Db)
        return -1;
    for (int64_t f = 0; f < n; f++) {
        const float *a = fibers + (size_t)f * 3 * NPTS;
        uint32_t *mf = mask + (size_t)f * words, *af = amb ? amb + (size_t)f * words : NULL;
        for (int32_t w = 0; w < words; w++) {
            mf[w] = 0;
            if (af) af[w] = 0;
        }
        if (!fiber_is_finite(a))
            continue;
        for (int32_t b = 0; b < B; b++)
            Db[b] = INFINITY;
        for (int64_t m = 0; m < M; m++) {
            double d2 = oracle_dme_d2(a, centroids + (size_t)m * 3 * NPTS);
            if (d2 < Db[bundle_id[m]])
                Db[bundle_id[m]] = d2;
        }
        for (int32_t b = 0; b < B; b++) {
            double t = (double)thresh[b];
            if (Db[b] <= t * t)
                mf[b >> 5] |= 1u << (b & 31);
            if (af && fabs(sqrt(Db[b]) - t) <= delta)
                af[b >> 5] |= 1u << (b & 31);
        }
    }
    free(Db);
    return 0;
}
