/*
 * lfp_oracle.c -- CPU ORACLE (test infrastructure only).
 *
 * A plain-C restatement of the reference's probe-grid tracer
 * (/root/reference/pkg/src/lfprobe/kernels.py, cited below as K:<line>) and
 * of its camera ray generation (render.py, cited as R:<line>). It exists to
 * CHECK the CUDA path: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load it. Nothing in the product
 * package links or calls it.
 *
 * Pinning: tests/golden/make_golden.py runs the reference itself (numba,
 * imported read-only in the build container) on seeded inputs and commits
 * its outputs; tests/test_oracle_golden.py checks this file against them
 * bit-for-bit (status, probe, texel, fetch count, radiance).
 *
 * Arithmetic: IEEE fp64 per operation in the reference's source order, no
 * FMA contraction (build with -ffp-contract=off). numba emits no FMA for
 * these kernels, so this reproduces its bits. Comparisons
 * are written in the reference's exact form (never fmin/fmax) so NaN and
 * tie behaviour match as well.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define MISS 0
#define HIT 1
#define UNKNOWN 2

typedef struct {
    const float *dist_hi;   /* (P, R, R)    */
    const float *dir_hi;    /* (P, R, R, 3) */
    const float *irr_hi;    /* (P, R, R, 3) */
    const float *dist_lo;   /* (P, r, r)    */
    const double *origins;  /* (P, 3)       */
    int64_t P;
    int64_t R;
    int64_t r;
} probes_t;

/* K:30-32 */
static inline double sign_nz(double v) { return v >= 0.0 ? 1.0 : -1.0; }

/* K:35-45 */
static void oct_encode_s(double x, double y, double z, double *u, double *v)
{
    double l1 = fabs(x) + fabs(y) + fabs(z);
    double px = x / l1;
    double pz = z / l1;
    if (y < 0.0) {
        double fx = sign_nz(px) * (1.0 - fabs(pz));
        double fz = sign_nz(pz) * (1.0 - fabs(px));
        px = fx;
        pz = fz;
    }
    *u = px * 0.5 + 0.5;
    *v = pz * 0.5 + 0.5;
}

/* K:48-59 */
static void oct_decode_s(double u, double v, double *ox, double *oy, double *oz)
{
    double fx = u * 2.0 - 1.0;
    double fz = v * 2.0 - 1.0;
    double y = 1.0 - fabs(fx) - fabs(fz);
    if (y < 0.0) {
        double ux = sign_nz(fx) * (1.0 - fabs(fz));
        double uz = sign_nz(fz) * (1.0 - fabs(fx));
        fx = ux;
        fz = uz;
    }
    double inv = 1.0 / sqrt(fx * fx + y * y + fz * fz);
    *ox = fx * inv;
    *oy = y * inv;
    *oz = fz * inv;
}

/* K:62-81 */
static double distance_to_intersection_s(double wx, double wy, double wz,
                                         double dx, double dy, double dz,
                                         double vx, double vy, double vz)
{
    double ax = wy * vz - wz * vy;
    double ay = wz * vx - wx * vz;
    double az = wx * vy - wy * vx;
    double bx = dy * vz - dz * vy;
    double by = dz * vx - dx * vz;
    double bz = dx * vy - dy * vx;
    double denom = bx * bx + by * by + bz * bz;
    if (denom < 1e-12)
        return sqrt(wx * wx + wy * wy + wz * wz);
    double t = -(ax * bx + ay * by + az * bz) / denom;
    double px = wx + t * dx;
    double py = wy + t * dy;
    double pz = wz + t * dz;
    return sqrt(px * px + py * py + pz * pz);
}

/* K:84-89 */
static inline double ray_radius(double wx, double wy, double wz,
                                double dx, double dy, double dz, double t)
{
    double px = wx + t * dx;
    double py = wy + t * dy;
    double pz = wz + t * dz;
    return sqrt(px * px + py * py + pz * pz);
}

/* K:92-99 */
static inline double s_to_t(double s, double l0, double l1, double a, double b)
{
    double denom = l1 + s * (l0 - l1);
    if (denom <= 0.0)
        return b;
    double tau = s * l0 / denom;
    return a + tau * (b - a);
}

/* K:102-129 */
static int compute_fold_boundaries(double wx, double wy, double wz,
                                   double dx, double dy, double dz,
                                   double t0, double t1, double *out)
{
    int n = 0;
    double tmp[3];
    double cw[3] = {wx, wy, wz};
    double cd[3] = {dx, dy, dz};
    for (int axis = 0; axis < 3; axis++) {
        double d = cd[axis];
        if (d != 0.0) {
            double tc = -cw[axis] / d;
            if (t0 < tc && tc < t1)
                tmp[n++] = tc;
        }
    }
    for (int i = 1; i < n; i++) {
        double key = tmp[i];
        int j = i - 1;
        while (j >= 0 && tmp[j] > key) {
            tmp[j + 1] = tmp[j];
            j--;
        }
        tmp[j + 1] = key;
    }
    out[0] = t0;
    for (int i = 0; i < n; i++)
        out[i + 1] = tmp[i];
    out[n + 1] = t1;
    return n + 2;
}

typedef struct {
    double p0u, p0v, p1u, p1v, l0, l1, aa, bb;
} chord_t;

/* K:132-154 */
static chord_t chord_setup(double wx, double wy, double wz,
                           double dx, double dy, double dz, double a, double b)
{
    chord_t c;
    double shrink = (b - a) * 1e-9 + 1e-12;
    double aa = a + shrink;
    double bb = b - shrink;
    if (bb < aa) {
        aa = a;
        bb = b;
    }
    double x0 = wx + aa * dx, y0 = wy + aa * dy, z0 = wz + aa * dz;
    double x1 = wx + bb * dx, y1 = wy + bb * dy, z1 = wz + bb * dz;
    c.l0 = fabs(x0) + fabs(y0) + fabs(z0);
    c.l1 = fabs(x1) + fabs(y1) + fabs(z1);
    double n0 = sqrt(x0 * x0 + y0 * y0 + z0 * z0);
    double n1 = sqrt(x1 * x1 + y1 * y1 + z1 * z1);
    oct_encode_s(x0 / n0, y0 / n0, z0 / n0, &c.p0u, &c.p0v);
    oct_encode_s(x1 / n1, y1 / n1, z1 / n1, &c.p1u, &c.p1v);
    c.aa = aa;
    c.bb = bb;
    return c;
}

/* numba's int(np.floor(q)) on x86-64: cvttsd2si, NaN/overflow -> INT64_MIN */
static inline int64_t floor_i64(double q)
{
    double f = floor(q);
    if (!(f >= -9.2e18 && f <= 9.2e18))
        return INT64_MIN;
    return (int64_t)f;
}

static inline int64_t trunc_i64(double q)
{
    if (!(q >= -9.2e18 && q <= 9.2e18))
        return INT64_MIN;
    return (int64_t)q;
}

typedef struct {
    int status;
    int64_t tx, ty, fetches, occ_x, occ_y;
} hscan_t;

/* K:157-267 */
static hscan_t high_res_scan(const float *dist_hi, const float *dir_hi,
                             int64_t res, const chord_t *c,
                             double s_begin, double s_end,
                             double wx, double wy, double wz,
                             double dx, double dy, double dz, double slack)
{
    hscan_t o;
    double du = c->p1u - c->p0u;
    double dv = c->p1v - c->p0v;
    const double eps_s = 1e-12;
    double s = s_begin;
    double qu = (c->p0u + s * du) * (double)res;
    double qv = (c->p0v + s * dv) * (double)res;
    int64_t ix = floor_i64(qu);
    int64_t iy = floor_i64(qv);
    if (ix < 0) ix = 0;
    if (ix > res - 1) ix = res - 1;
    if (iy < 0) iy = 0;
    if (iy > res - 1) iy = res - 1;
    double sdu = du * (double)res;
    double sdv = dv * (double)res;
    int64_t step_x = sdu > 0.0 ? 1 : -1;
    int64_t step_y = sdv > 0.0 ? 1 : -1;
    double t_max_x, t_dx, t_max_y, t_dy;
    if (sdu != 0.0) {
        int64_t nx = step_x > 0 ? ix + 1 : ix;
        t_max_x = s + ((double)nx - qu) / sdu;
        t_dx = fabs(1.0 / sdu);
    } else {
        t_max_x = INFINITY;
        t_dx = INFINITY;
    }
    if (sdv != 0.0) {
        int64_t ny = step_y > 0 ? iy + 1 : iy;
        t_max_y = s + ((double)ny - qv) / sdv;
        t_dy = fabs(1.0 / sdv);
    } else {
        t_max_y = INFINITY;
        t_dy = INFINITY;
    }
    int64_t fetches = 0, occ_x = -1, occ_y = -1;
    for (;;) {
        double stored = (double)dist_hi[iy * res + ix];
        fetches += 1;
        if (isfinite(stored)) {
            double s_hi = t_max_x < t_max_y ? t_max_x : t_max_y;
            if (s_hi > s_end) s_hi = s_end;
            if (s_hi > 1.0) s_hi = 1.0;
            double s_lo = s > 0.0 ? s : 0.0;
            double cu = ((double)ix + 0.5) / (double)res;
            double cv = ((double)iy + 0.5) / (double)res;
            double vx, vy, vz;
            oct_decode_s(cu, cv, &vx, &vy, &vz);
            double d2i = distance_to_intersection_s(wx, wy, wz, dx, dy, dz,
                                                    vx, vy, vz);
            double r_in = ray_radius(wx, wy, wz, dx, dy, dz,
                                     s_to_t(s_lo, c->l0, c->l1, c->aa, c->bb));
            double r_out = ray_radius(wx, wy, wz, dx, dy, dz,
                                      s_to_t(s_hi, c->l0, c->l1, c->aa, c->bb));
            double rmin = r_in < r_out ? r_in : r_out;
            if (d2i < rmin) rmin = d2i;
            double rmax = r_in > r_out ? r_in : r_out;
            if (d2i > rmax) rmax = d2i;
            double thick = 4.0 * (rmax - rmin) + slack * rmin;
            if (stored < rmin - thick) {
                occ_x = ix;
                occ_y = iy;
            } else if (stored < rmax * (1.0 + slack)) {
                const float *nv = dir_hi + (iy * res + ix) * 3;
                double nx_ = nv[0], ny_ = nv[1], nz_ = nv[2];
                o.tx = ix; o.ty = iy; o.fetches = fetches;
                o.occ_x = occ_x; o.occ_y = occ_y;
                o.status = (nx_ * dx + ny_ * dy + nz_ * dz > 0.0) ? HIT : UNKNOWN;
                return o;
            }
        }
        if (t_max_x < t_max_y) {
            s = t_max_x;
            t_max_x += t_dx;
            ix += step_x;
        } else {
            s = t_max_y;
            t_max_y += t_dy;
            iy += step_y;
        }
        if (s > s_end + eps_s || s > 1.0 ||
            ix < 0 || ix >= res || iy < 0 || iy >= res) {
            o.status = MISS; o.tx = ix; o.ty = iy; o.fetches = fetches;
            o.occ_x = occ_x; o.occ_y = occ_y;
            return o;
        }
    }
}

typedef struct {
    int status;
    int64_t tx, ty, fetches;
} seg_t;

/* K:373-480 */
static seg_t trace_segment(const float *dist_hi, const float *dir_hi,
                           const float *dist_lo, int64_t res_hi, int64_t res,
                           double wx, double wy, double wz,
                           double dx, double dy, double dz,
                           double a, double b, double slack)
{
    seg_t o;
    chord_t c = chord_setup(wx, wy, wz, dx, dy, dz, a, b);
    double du = c.p1u - c.p0u;
    double dv = c.p1v - c.p0v;
    double chord_len = sqrt(du * du + dv * dv);
    double margin;
    if (chord_len * (double)res_hi > 1e-9)
        margin = 2.0 / ((double)res_hi * chord_len);
    else
        margin = 2.0;
    double qu = c.p0u * (double)res;
    double qv = c.p0v * (double)res;
    int64_t ix = floor_i64(qu);
    int64_t iy = floor_i64(qv);
    if (ix < 0) ix = 0;
    if (ix > res - 1) ix = res - 1;
    if (iy < 0) iy = 0;
    if (iy > res - 1) iy = res - 1;
    double sdu = du * (double)res;
    double sdv = dv * (double)res;
    int64_t step_x = sdu > 0.0 ? 1 : -1;
    int64_t step_y = sdv > 0.0 ? 1 : -1;
    double t_max_x, t_dx, t_max_y, t_dy;
    if (sdu != 0.0) {
        int64_t nx = step_x > 0 ? ix + 1 : ix;
        t_max_x = ((double)nx - qu) / sdu;
        t_dx = fabs(1.0 / sdu);
    } else {
        t_max_x = INFINITY;
        t_dx = INFINITY;
    }
    if (sdv != 0.0) {
        int64_t ny = step_y > 0 ? iy + 1 : iy;
        t_max_y = ((double)ny - qv) / sdv;
        t_dy = fabs(1.0 / sdv);
    } else {
        t_max_y = INFINITY;
        t_dy = INFINITY;
    }
    int64_t fetches = 0, occ_x = -1, occ_y = -1;
    double s_in = 0.0;
    for (;;) {
        double s_out = t_max_x < t_max_y ? t_max_x : t_max_y;
        if (s_out > 1.0) s_out = 1.0;
        double m = INFINITY;
        for (int64_t jy = iy - 1; jy < iy + 2; jy++) {
            if (jy < 0 || jy >= res) continue;
            for (int64_t jx = ix - 1; jx < ix + 2; jx++) {
                if (jx < 0 || jx >= res) continue;
                double val = (double)dist_lo[jy * res + jx];
                fetches += 1;
                if (val < m) m = val;
            }
        }
        if (isfinite(m)) {
            double s_a = s_in - margin;
            if (s_a < 0.0) s_a = 0.0;
            double s_b = s_out + margin;
            if (s_b > 1.0) s_b = 1.0;
            double r_a = ray_radius(wx, wy, wz, dx, dy, dz,
                                    s_to_t(s_a, c.l0, c.l1, c.aa, c.bb));
            double r_b = ray_radius(wx, wy, wz, dx, dy, dz,
                                    s_to_t(s_b, c.l0, c.l1, c.aa, c.bb));
            double rmax = r_a > r_b ? r_a : r_b;
            if (m < rmax * (1.0 + slack)) {
                hscan_t h = high_res_scan(dist_hi, dir_hi, res_hi, &c, s_in,
                                          s_out, wx, wy, wz, dx, dy, dz, slack);
                fetches += h.fetches;
                if (h.occ_x >= 0) {
                    occ_x = h.occ_x;
                    occ_y = h.occ_y;
                }
                if (h.status != MISS) {
                    o.status = h.status; o.tx = h.tx; o.ty = h.ty;
                    o.fetches = fetches;
                    return o;
                }
            }
        }
        if (t_max_x < t_max_y) {
            s_in = t_max_x;
            t_max_x += t_dx;
            ix += step_x;
        } else {
            s_in = t_max_y;
            t_max_y += t_dy;
            iy += step_y;
        }
        if (s_in >= 1.0 || ix < 0 || ix >= res || iy < 0 || iy >= res) {
            o.fetches = fetches;
            if (occ_x >= 0) {
                o.status = UNKNOWN; o.tx = occ_x; o.ty = occ_y;
            } else {
                o.status = MISS; o.tx = -1; o.ty = -1;
            }
            return o;
        }
    }
}

/* K:483-494 */
static seg_t trace_segment_brute(const float *dist_hi, const float *dir_hi,
                                 int64_t res_hi, double wx, double wy,
                                 double wz, double dx, double dy, double dz,
                                 double a, double b, double slack)
{
    seg_t o;
    chord_t c = chord_setup(wx, wy, wz, dx, dy, dz, a, b);
    hscan_t h = high_res_scan(dist_hi, dir_hi, res_hi, &c, 0.0, 1.0,
                              wx, wy, wz, dx, dy, dz, slack);
    o.fetches = h.fetches;
    if (h.status == MISS && h.occ_x >= 0) {
        o.status = UNKNOWN; o.tx = h.occ_x; o.ty = h.occ_y;
        return o;
    }
    o.status = h.status; o.tx = h.tx; o.ty = h.ty;
    return o;
}

/* K:497-515 (brute=0) and K:518-534 (brute=1) */
static seg_t trace_probe_range(const probes_t *ps, int64_t p, int brute,
                               double wx, double wy, double wz,
                               double dx, double dy, double dz,
                               double t0, double t1, double slack)
{
    double bounds[5];
    int nb = compute_fold_boundaries(wx, wy, wz, dx, dy, dz, t0, t1, bounds);
    const int64_t R = ps->R, r = ps->r;
    const float *dh = ps->dist_hi + p * R * R;
    const float *nh = ps->dir_hi + p * R * R * 3;
    const float *dl = ps->dist_lo + p * r * r;
    int64_t fetches = 0;
    seg_t o;
    for (int i = 0; i < nb - 1; i++) {
        double a = bounds[i], b = bounds[i + 1];
        if (b - a < 1e-12) continue;
        seg_t s = brute ? trace_segment_brute(dh, nh, R, wx, wy, wz, dx, dy,
                                              dz, a, b, slack)
                        : trace_segment(dh, nh, dl, R, r, wx, wy, wz, dx, dy,
                                        dz, a, b, slack);
        fetches += s.fetches;
        if (s.status != MISS) {
            s.fetches = fetches;
            return s;
        }
    }
    o.status = MISS; o.tx = -1; o.ty = -1; o.fetches = fetches;
    return o;
}

/* K:537-564 */
static double exit_t(double ox, double oy, double oz, double dx, double dy,
                     double dz, const double *lo, const double *hi)
{
    double t_near = -INFINITY, t_far = INFINITY;
    double o3[3] = {ox, oy, oz}, d3[3] = {dx, dy, dz};
    for (int axis = 0; axis < 3; axis++) {
        double o = o3[axis], d = d3[axis];
        if (d == 0.0) {
            if (o < lo[axis] || o > hi[axis]) return -1.0;
        } else {
            double ta = (lo[axis] - o) / d;
            double tb = (hi[axis] - o) / d;
            if (ta > tb) { double t = ta; ta = tb; tb = t; }
            if (ta > t_near) t_near = ta;
            if (tb < t_far) t_far = tb;
        }
    }
    if (t_far < t_near || t_far < 0.0) return -1.0;
    return t_far;
}

typedef struct {
    int status;
    int64_t probe, tx, ty, fetches;
} ray_out_t;

/* K:599-650 */
static ray_out_t trace_probes_ordered(const probes_t *ps, const int64_t *order,
                                      int n_order, double ex, double ey,
                                      double ez, double dx, double dy,
                                      double dz, double t0, double t1,
                                      double eps_start, double eps_align,
                                      double slack, double *rgb_out)
{
    ray_out_t o;
    int64_t last_p = -1, last_tx = -1, last_ty = -1, fetches = 0;
    const int64_t R = ps->R;
    for (int oi = 0; oi < n_order; oi++) {
        int64_t p = order[oi];
        double wx = ex - ps->origins[p * 3 + 0];
        double wy = ey - ps->origins[p * 3 + 1];
        double wz = ez - ps->origins[p * 3 + 2];
        double wlen = sqrt(wx * wx + wy * wy + wz * wz);
        if (wlen < eps_align && t0 <= eps_start * 2.0) {
            double u, v;
            oct_encode_s(dx, dy, dz, &u, &v);
            int64_t tx = trunc_i64(u * (double)R);
            int64_t ty = trunc_i64(v * (double)R);
            if (tx > R - 1) tx = R - 1;
            if (ty > R - 1) ty = R - 1;
            double stored = (double)ps->dist_hi[(p * R + ty) * R + tx];
            fetches += 1;
            if (isfinite(stored) && stored <= t1 * (1.0 + slack)) {
                const float *c = ps->irr_hi + ((p * R + ty) * R + tx) * 3;
                rgb_out[0] = c[0]; rgb_out[1] = c[1]; rgb_out[2] = c[2];
                o.status = HIT; o.probe = p; o.tx = tx; o.ty = ty;
                o.fetches = fetches;
                return o;
            }
            continue;
        }
        seg_t s = trace_probe_range(ps, p, 0, wx, wy, wz, dx, dy, dz, t0, t1,
                                    slack);
        fetches += s.fetches;
        if (s.status == HIT) {
            const float *c = ps->irr_hi + ((p * R + s.ty) * R + s.tx) * 3;
            rgb_out[0] = c[0]; rgb_out[1] = c[1]; rgb_out[2] = c[2];
            o.status = HIT; o.probe = p; o.tx = s.tx; o.ty = s.ty;
            o.fetches = fetches;
            return o;
        }
        if (s.status == UNKNOWN) {
            last_p = p; last_tx = s.tx; last_ty = s.ty;
        }
    }
    o.fetches = fetches;
    if (last_p >= 0) {
        o.status = UNKNOWN; o.probe = last_p; o.tx = last_tx; o.ty = last_ty;
    } else {
        o.status = MISS; o.probe = -1; o.tx = -1; o.ty = -1;
    }
    return o;
}

typedef struct {
    double g0[3];
    double cell;
    int64_t nx, ny, nz;
    double eps_start, eps_align, slack;
} grid_t;

/* K:653-822 */
static ray_out_t trace_grid_ray(const probes_t *ps, const grid_t *g,
                                double ex, double ey, double ez,
                                double dx, double dy, double dz,
                                double *rgb_out)
{
    ray_out_t o;
    o.status = MISS; o.probe = -1; o.tx = -1; o.ty = -1; o.fetches = 0;
    const int64_t cx = g->nx - 1, cy = g->ny - 1, cz = g->nz - 1;
    const double cell = g->cell;
    const double gx0 = g->g0[0], gy0 = g->g0[1], gz0 = g->g0[2];
    double t_near = -INFINITY, t_far = INFINITY;
    for (int axis = 0; axis < 3; axis++) {
        double or_, d, lo, hi;
        if (axis == 0) { or_ = ex; d = dx; lo = gx0; hi = gx0 + (double)cx * cell; }
        else if (axis == 1) { or_ = ey; d = dy; lo = gy0; hi = gy0 + (double)cy * cell; }
        else { or_ = ez; d = dz; lo = gz0; hi = gz0 + (double)cz * cell; }
        if (d == 0.0) {
            if (or_ < lo || or_ > hi) return o;
        } else {
            double ta = (lo - or_) / d;
            double tb = (hi - or_) / d;
            if (ta > tb) { double t = ta; ta = tb; tb = t; }
            if (ta > t_near) t_near = ta;
            if (tb < t_far) t_far = tb;
        }
    }
    if (t_far < t_near || t_far <= 0.0) return o;
    double t_enter = t_near > 0.0 ? t_near : 0.0;

    double t_probe = t_enter + 1e-9;
    double px = (ex + t_probe * dx - gx0) / cell;
    double py = (ey + t_probe * dy - gy0) / cell;
    double pz = (ez + t_probe * dz - gz0) / cell;
    int64_t ci = floor_i64(px), cj = floor_i64(py), ck = floor_i64(pz);
    if (ci < 0) ci = 0;
    if (ci > cx - 1) ci = cx - 1;
    if (cj < 0) cj = 0;
    if (cj > cy - 1) cj = cy - 1;
    if (ck < 0) ck = 0;
    if (ck > cz - 1) ck = cz - 1;

    int64_t step_i = dx > 0.0 ? 1 : -1;
    int64_t step_j = dy > 0.0 ? 1 : -1;
    int64_t step_k = dz > 0.0 ? 1 : -1;
    double t_max_i, t_d_i, t_max_j, t_d_j, t_max_k, t_d_k;
    if (dx != 0.0) {
        double nb = gx0 + (double)(ci + (step_i > 0 ? 1 : 0)) * cell;
        t_max_i = (nb - ex) / dx;
        t_d_i = fabs(cell / dx);
    } else { t_max_i = INFINITY; t_d_i = INFINITY; }
    if (dy != 0.0) {
        double nb = gy0 + (double)(cj + (step_j > 0 ? 1 : 0)) * cell;
        t_max_j = (nb - ey) / dy;
        t_d_j = fabs(cell / dy);
    } else { t_max_j = INFINITY; t_d_j = INFINITY; }
    if (dz != 0.0) {
        double nb = gz0 + (double)(ck + (step_k > 0 ? 1 : 0)) * cell;
        t_max_k = (nb - ez) / dz;
        t_d_k = fabs(cell / dz);
    } else { t_max_k = INFINITY; t_d_k = INFINITY; }

    int64_t corner_idx[8], order[8], probe_order[8];
    double corner_d2[8];
    int64_t fetches = 0, best_p = -1, best_tx = -1, best_ty = -1;
    double t_cur = t_enter;
    for (;;) {
        double t_exit_cube = t_max_i;
        if (t_max_j < t_exit_cube) t_exit_cube = t_max_j;
        if (t_max_k < t_exit_cube) t_exit_cube = t_max_k;
        if (t_exit_cube > t_far) t_exit_cube = t_far;
        int c = 0;
        for (int di = 0; di < 2; di++)
            for (int dj = 0; dj < 2; dj++)
                for (int dk = 0; dk < 2; dk++) {
                    int64_t idx = ((ci + di) * g->ny + (cj + dj)) * g->nz + (ck + dk);
                    double ox = ps->origins[idx * 3 + 0] - ex;
                    double oy = ps->origins[idx * 3 + 1] - ey;
                    double oz = ps->origins[idx * 3 + 2] - ez;
                    corner_idx[c] = idx;
                    corner_d2[c] = ox * ox + oy * oy + oz * oz;
                    c++;
                }
        for (c = 0; c < 8; c++) order[c] = c;
        for (c = 1; c < 8; c++) {
            double key_d = corner_d2[order[c]];
            int64_t key_o = order[c];
            int j = c - 1;
            while (j >= 0 && corner_d2[order[j]] > key_d) {
                order[j + 1] = order[j];
                j--;
            }
            order[j + 1] = key_o;
        }
        for (c = 0; c < 8; c++) probe_order[c] = corner_idx[order[c]];
        double t0 = (0.0 > t_cur) ? 0.0 : t_cur;   /* numba max(t_cur, 0.0) */
        ray_out_t r = trace_probes_ordered(ps, probe_order, 8, ex, ey, ez,
                                           dx, dy, dz, t0, t_exit_cube,
                                           g->eps_start, g->eps_align,
                                           g->slack, rgb_out);
        fetches += r.fetches;
        if (r.status == HIT) {
            r.fetches = fetches;
            return r;
        }
        if (r.status == UNKNOWN) {
            best_p = r.probe; best_tx = r.tx; best_ty = r.ty;
        }
        if (t_max_i <= t_max_j && t_max_i <= t_max_k) {
            t_cur = t_max_i;
            t_max_i += t_d_i;
            ci += step_i;
            if (ci < 0 || ci >= cx) break;
        } else if (t_max_j <= t_max_k) {
            t_cur = t_max_j;
            t_max_j += t_d_j;
            cj += step_j;
            if (cj < 0 || cj >= cy) break;
        } else {
            t_cur = t_max_k;
            t_max_k += t_d_k;
            ck += step_k;
            if (ck < 0 || ck >= cz) break;
        }
        if (t_cur >= t_far) break;
    }
    o.status = MISS; o.probe = best_p; o.tx = best_tx; o.ty = best_ty;
    o.fetches = fetches;
    return o;
}

/* ------------------------------------------------------------------------ */
/* exported entry points (ctypes)                                           */
/* ------------------------------------------------------------------------ */

static probes_t mk_probes(const float *dist_hi, const float *dir_hi,
                          const float *irr_hi, const float *dist_lo,
                          const double *origins, int64_t P, int64_t R,
                          int64_t r)
{
    probes_t ps = {dist_hi, dir_hi, irr_hi, dist_lo, origins, P, R, r};
    return ps;
}

int lfpo_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void lfpo_set_num_threads(int n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* R:50-62: pixel-centre directions, row-major from the top-left pixel.
 * basis = (r, u, f) as computed by Camera.basis() (R:33-48). */
void lfpo_camera_dirs(const double *basis, double tan_v, double tan_h,
                      int64_t W, int64_t H, double *dirs)
{
    const double *rr = basis, *uu = basis + 3, *ff = basis + 6;
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < H; j++) {
        double y = (1.0 - ((double)j + 0.5) / (double)H * 2.0) * tan_v;
        for (int64_t i = 0; i < W; i++) {
            double x = (((double)i + 0.5) / (double)W * 2.0 - 1.0) * tan_h;
            double c0 = (ff[0] + x * rr[0]) + y * uu[0];
            double c1 = (ff[1] + x * rr[1]) + y * uu[1];
            double c2 = (ff[2] + x * rr[2]) + y * uu[2];
            double n = sqrt((c0 * c0 + c1 * c1) + c2 * c2);
            double *d = dirs + (j * W + i) * 3;
            d[0] = c0 / n;
            d[1] = c1 / n;
            d[2] = c2 / n;
        }
    }
}

/* Per-ray twin of K:653 over a batch. origins (N,3) or a single eye when
 * origin_stride == 0. Outputs are all per ray; rgb (N,3) is written only on
 * HIT (caller pre-zeroes), matching K:838-843. */
void lfpo_trace_rays(const float *dist_hi, const float *dir_hi,
                     const float *irr_hi, const float *dist_lo,
                     const double *origins, int64_t P, int64_t R, int64_t r,
                     const double *grid_origin, double cell, int64_t nx,
                     int64_t ny, int64_t nz, const double *ray_o,
                     int64_t origin_stride, const double *ray_d, int64_t n,
                     double eps_start, double eps_align, double slack,
                     uint8_t *out_status, int32_t *out_probe, int32_t *out_tx,
                     int32_t *out_ty, int64_t *out_fetch, double *out_rgb)
{
    probes_t ps = mk_probes(dist_hi, dir_hi, irr_hi, dist_lo, origins, P, R, r);
    grid_t g;
    g.g0[0] = grid_origin[0]; g.g0[1] = grid_origin[1]; g.g0[2] = grid_origin[2];
    g.cell = cell; g.nx = nx; g.ny = ny; g.nz = nz;
    g.eps_start = eps_start; g.eps_align = eps_align; g.slack = slack;
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t i = 0; i < n; i++) {
        const double *o = ray_o + i * origin_stride;
        const double *d = ray_d + i * 3;
        double rgb[3] = {0.0, 0.0, 0.0};
        ray_out_t res = trace_grid_ray(&ps, &g, o[0], o[1], o[2], d[0], d[1],
                                       d[2], rgb);
        out_status[i] = (uint8_t)res.status;
        if (out_probe) out_probe[i] = (int32_t)res.probe;
        if (out_tx) out_tx[i] = (int32_t)res.tx;
        if (out_ty) out_ty[i] = (int32_t)res.ty;
        if (out_fetch) out_fetch[i] = res.fetches;
        if (res.status == HIT && out_rgb) {
            out_rgb[i * 3 + 0] = rgb[0];
            out_rgb[i * 3 + 1] = rgb[1];
            out_rgb[i * 3 + 2] = rgb[2];
        }
    }
}

/* K:567-596 (render_single_probe): full marching against one probe. */
void lfpo_render_single_probe(const float *dist_hi, const float *dir_hi,
                              const float *irr_hi, const float *dist_lo,
                              int64_t R, int64_t r, const double *origin,
                              const double *eye, const double *dirs, int64_t n,
                              const double *blo, const double *bhi,
                              double eps_start, double slack,
                              uint8_t *out_status, double *out_rgb,
                              int64_t *out_fetch)
{
    probes_t ps = mk_probes(dist_hi, dir_hi, irr_hi, dist_lo, origin, 1, R, r);
    double wx = eye[0] - origin[0], wy = eye[1] - origin[1],
           wz = eye[2] - origin[2];
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t i = 0; i < n; i++) {
        double dx = dirs[i * 3], dy = dirs[i * 3 + 1], dz = dirs[i * 3 + 2];
        double t1 = exit_t(eye[0], eye[1], eye[2], dx, dy, dz, blo, bhi);
        if (t1 <= eps_start) {
            out_status[i] = MISS;
            out_fetch[i] = 0;
            continue;
        }
        seg_t s = trace_probe_range(&ps, 0, 0, wx, wy, wz, dx, dy, dz,
                                    eps_start, t1, slack);
        out_status[i] = (uint8_t)s.status;
        out_fetch[i] = s.fetches;
        if (s.status == HIT) {
            const float *c = irr_hi + (s.ty * R + s.tx) * 3;
            out_rgb[i * 3] = c[0]; out_rgb[i * 3 + 1] = c[1];
            out_rgb[i * 3 + 2] = c[2];
        }
    }
}

/* K:846-892 (render_few_probes): global nearest-first order, no cubes. */
void lfpo_render_few_probes(const float *dist_hi, const float *dir_hi,
                            const float *irr_hi, const float *dist_lo,
                            const double *origins, int64_t P, int64_t R,
                            int64_t r, const double *blo, const double *bhi,
                            const double *eye, const double *dirs, int64_t n,
                            double eps_start, double eps_align, double slack,
                            uint8_t *out_status, double *out_rgb,
                            int64_t *out_fetch)
{
    probes_t ps = mk_probes(dist_hi, dir_hi, irr_hi, dist_lo, origins, P, R, r);
    int64_t *order = (int64_t *)malloc(sizeof(int64_t) * (size_t)P);
    double *d2 = (double *)malloc(sizeof(double) * (size_t)P);
    for (int64_t p = 0; p < P; p++) {
        double ox = origins[p * 3] - eye[0], oy = origins[p * 3 + 1] - eye[1],
               oz = origins[p * 3 + 2] - eye[2];
        d2[p] = ox * ox + oy * oy + oz * oz;
        order[p] = p;
    }
    for (int64_t c = 1; c < P; c++) {
        double key_d = d2[order[c]];
        int64_t key_o = order[c];
        int64_t j = c - 1;
        while (j >= 0 && d2[order[j]] > key_d) {
            order[j + 1] = order[j];
            j--;
        }
        order[j + 1] = key_o;
    }
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t i = 0; i < n; i++) {
        double dx = dirs[i * 3], dy = dirs[i * 3 + 1], dz = dirs[i * 3 + 2];
        double t1 = exit_t(eye[0], eye[1], eye[2], dx, dy, dz, blo, bhi);
        if (t1 <= eps_start) {
            out_status[i] = MISS;
            out_fetch[i] = 0;
            continue;
        }
        double rgb[3] = {0, 0, 0};
        ray_out_t res = trace_probes_ordered(&ps, order, (int)P, eye[0],
                                             eye[1], eye[2], dx, dy, dz,
                                             eps_start, t1, eps_start,
                                             eps_align, slack, rgb);
        out_status[i] = (uint8_t)res.status;
        out_fetch[i] = res.fetches;
        if (res.status == HIT) {
            out_rgb[i * 3] = rgb[0]; out_rgb[i * 3 + 1] = rgb[1];
            out_rgb[i * 3 + 2] = rgb[2];
        }
    }
    free(order);
    free(d2);
}

/* ---- scalar known-answer hooks (tests only) ---- */
void lfpo_oct_encode(double x, double y, double z, double *uv)
{
    oct_encode_s(x, y, z, &uv[0], &uv[1]);
}

void lfpo_oct_decode(double u, double v, double *d)
{
    oct_decode_s(u, v, &d[0], &d[1], &d[2]);
}

double lfpo_distance_to_intersection(const double *w, const double *d,
                                     const double *v)
{
    return distance_to_intersection_s(w[0], w[1], w[2], d[0], d[1], d[2],
                                      v[0], v[1], v[2]);
}

int lfpo_fold_boundaries(const double *w, const double *d, double t0,
                         double t1, double *out)
{
    return compute_fold_boundaries(w[0], w[1], w[2], d[0], d[1], d[2], t0, t1,
                                   out);
}

/* one probe, one ray over [t0, t1]; brute != 0 selects K:518 */
void lfpo_trace_probe_range(const float *dist_hi, const float *dir_hi,
                            const float *dist_lo, int64_t R, int64_t r,
                            const double *w, const double *d, double t0,
                            double t1, double slack, int brute, int64_t *out4)
{
    double zero[3] = {0, 0, 0};
    probes_t ps = mk_probes(dist_hi, dir_hi, NULL, dist_lo, zero, 1, R, r);
    seg_t s = trace_probe_range(&ps, 0, brute, w[0], w[1], w[2], d[0], d[1],
                                d[2], t0, t1, slack);
    out4[0] = s.status; out4[1] = s.tx; out4[2] = s.ty; out4[3] = s.fetches;
}
