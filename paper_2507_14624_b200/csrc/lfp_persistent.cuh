// lfp_persistent.cuh -- persistent, flattened grid traversal (sm_100a).
//
// The nested traversal (lfp_trace.cuh: cube loop > probe loop > segment loop
// > low-res loop > high-res loop) keeps a warp busy until its slowest ray is
// done; with heavy-tailed per-ray cost (incoherent rays: fetch p99 ~8x p50)
// most lanes idle (ncu: 2.65 active threads / warp on C5). Here every lane
// runs an explicit state machine over the SAME steps and decisions
// (K:599-822, K:373-480, K:157-267 via the shared helpers in lfp_trace.cuh),
// and lanes whose ray is finished fetch a new ray from a global counter
// (warp-aggregated atomics), so warps stay full until the batch is done.
//
// Scheduling: a round = (1) transition phase: every lane that is not in a
// stepping state advances ray -> cube -> probe -> segment setup until it
// reaches a low-res step (or finishes its ray, emits it and fetches the next
// one); (2) stepping phase: low-res / high-res DDA steps while at least
// `min_active` lanes of the warp are stepping. Lanes whose segment ends
// during (2) wait for the next transition phase, so the expensive segment
// setup is executed by many lanes together.
#pragma once

#include "lfp_trace.cuh"

namespace lfp {

enum : int {
    S_FETCH = 0,   // needs a ray
    S_CUBE,        // set up the current cube (corner order)
    S_PROBE,       // next probe of the cube (or next cube)
    S_SEG,         // next fold-free segment of the probe range (or next probe)
    S_LO,          // stepping: low-res DDA
    S_HI,          // stepping: high-res DDA inside a flagged block
    S_EMIT,        // ray finished: write outputs
    S_EXIT         // no more rays
};

// Everything a lane carries between steps.
struct Lane {
    long long ray;          // ray id (slot) being traced
    double ex, ey, ez, dx, dy, dz;
    // cube walk (K:715-821)
    double t_max_i, t_max_j, t_max_k, t_d_i, t_d_j, t_d_k, t_cur, t_far;
    int ci, cj, ck, steps;  // steps: bit0..2 = (dx>0, dy>0, dz>0)
    int fetches, best_p, best_tx, best_ty;
    // cube: probe order and fall-through (K:599-650)
    unsigned order;
    int oi, base, last_p, last_tx, last_ty;
    double t0, t1;
    // probe range (K:497-515)
    int p, nb, seg_i;
    double wx, wy, wz, b1, b2, b3;
    // segment (K:373-480)
    Chord c;
    ChordF* cf;             // this lane's slot in shared memory
    Dda lo, hi;
    double margin, s_out, s_end, prev_s, prev_r;
    int occ_x, occ_y, hocc_x, hocc_y;
    // result
    int status, rp, rtx, rty;
};

// K:668-692: slab test of the ray against the lattice AABB; false when the
// ray misses it (or the lattice is degenerate, G:118-120).
__device__ __forceinline__ bool lattice_slab(const GridParams& g, double ex,
                                             double ey, double ez, double dx,
                                             double dy, double dz,
                                             double& t_near_out,
                                             double& t_far_out)
{
    const int cx = g.nx - 1, cy = g.ny - 1, cz = g.nz - 1;
    if (cx < 1 || cy < 1 || cz < 1) return false;
    const double cell = g.cell;
    double t_near = -CUDART_INF, t_far = CUDART_INF;
    const double oo[3] = {ex, ey, ez};
    const double dd[3] = {dx, dy, dz};
    const double hi3[3] = {g.g0[0] + (double)cx * cell, g.g0[1] + (double)cy * cell,
                           g.g0[2] + (double)cz * cell};
#pragma unroll
    for (int axis = 0; axis < 3; axis++) {
        const double or_ = oo[axis], d = dd[axis];
        const double lo = g.g0[axis], hi = hi3[axis];
        if (d == 0.0) {
            if (or_ < lo || or_ > hi) return false;
        } else {
            double ta = (lo - or_) / d;
            double tb = (hi - or_) / d;
            if (ta > tb) { double t = ta; ta = tb; tb = t; }
            if (ta > t_near) t_near = ta;
            if (tb < t_far) t_far = tb;
        }
    }
    if (t_far < t_near || t_far <= 0.0) return false;
    t_near_out = t_near;
    t_far_out = t_far;
    return true;
}

// K:653-738: lattice entry of the lane's ray; returns false for a ray that
// misses the lattice (MISS, 0 fetches).
__device__ __forceinline__ bool lane_ray_init(Lane& L, const GridParams& g)
{
    L.fetches = 0;
    L.best_p = L.best_tx = L.best_ty = -1;
    L.status = MISS; L.rp = -1; L.rtx = -1; L.rty = -1;
    const int cx = g.nx - 1, cy = g.ny - 1, cz = g.nz - 1;
    const double cell = g.cell;
    double t_near, t_far;
    if (!lattice_slab(g, L.ex, L.ey, L.ez, L.dx, L.dy, L.dz, t_near, t_far))
        return false;
    const double t_enter = t_near > 0.0 ? t_near : 0.0;
    const double t_probe = t_enter + 1e-9;
    L.ci = floor_clamp((L.ex + t_probe * L.dx - g.g0[0]) / cell, cx - 1);
    L.cj = floor_clamp((L.ey + t_probe * L.dy - g.g0[1]) / cell, cy - 1);
    L.ck = floor_clamp((L.ez + t_probe * L.dz - g.g0[2]) / cell, cz - 1);
    L.steps = (L.dx > 0.0 ? 1 : 0) | (L.dy > 0.0 ? 2 : 0) | (L.dz > 0.0 ? 4 : 0);
    if (L.dx != 0.0) {
        double nb = g.g0[0] + (double)(L.ci + (L.dx > 0.0 ? 1 : 0)) * cell;
        L.t_max_i = (nb - L.ex) / L.dx;
        L.t_d_i = fabs(cell / L.dx);
    } else { L.t_max_i = CUDART_INF; L.t_d_i = CUDART_INF; }
    if (L.dy != 0.0) {
        double nb = g.g0[1] + (double)(L.cj + (L.dy > 0.0 ? 1 : 0)) * cell;
        L.t_max_j = (nb - L.ey) / L.dy;
        L.t_d_j = fabs(cell / L.dy);
    } else { L.t_max_j = CUDART_INF; L.t_d_j = CUDART_INF; }
    if (L.dz != 0.0) {
        double nb = g.g0[2] + (double)(L.ck + (L.dz > 0.0 ? 1 : 0)) * cell;
        L.t_max_k = (nb - L.ez) / L.dz;
        L.t_d_k = fabs(cell / L.dz);
    } else { L.t_max_k = CUDART_INF; L.t_d_k = CUDART_INF; }
    L.t_cur = t_enter;
    L.t_far = t_far;
    return true;
}

// K:750-786: corner probes of the current cube in stable distance order
__device__ __forceinline__ void lane_cube(Lane& L, const DevProbes& ps,
                                          const GridParams& g)
{
    double t_exit_cube = L.t_max_i;
    if (L.t_max_j < t_exit_cube) t_exit_cube = L.t_max_j;
    if (L.t_max_k < t_exit_cube) t_exit_cube = L.t_max_k;
    if (t_exit_cube > L.t_far) t_exit_cube = L.t_far;
    const int ny = g.ny, nz = g.nz;
    L.base = (L.ci * ny + L.cj) * nz + L.ck;
    double d2[8];
#pragma unroll
    for (int c = 0; c < 8; c++) {
        const int idx = L.base + ((c >> 2) & 1) * ny * nz + ((c >> 1) & 1) * nz + (c & 1);
        LFP_BCHK(idx, ps.P, 201);
        const double ox = __ldg(ps.origins + 3 * idx + 0) - L.ex;
        const double oy = __ldg(ps.origins + 3 * idx + 1) - L.ey;
        const double oz = __ldg(ps.origins + 3 * idx + 2) - L.ez;
        d2[c] = ox * ox + oy * oy + oz * oz;
    }
    unsigned order = 0;
#pragma unroll
    for (int c = 0; c < 8; c++) {
        int rank = 0;
#pragma unroll
        for (int c2 = 0; c2 < 8; c2++) {
            if (c2 < c) rank += (d2[c2] > d2[c]) ? 0 : 1;
            else if (c2 > c) rank += (d2[c2] < d2[c]) ? 1 : 0;
        }
        order |= (unsigned)c << (4 * rank);
    }
    L.order = order;
    L.oi = 0;
    L.last_p = -1;
    L.t0 = (0.0 > L.t_cur) ? 0.0 : L.t_cur;   // numba max(t_cur, 0.0)
    L.t1 = t_exit_cube;
}

// K:801-821: next cube; false when the walk leaves the lattice
__device__ __forceinline__ bool lane_next_cube(Lane& L, const GridParams& g)
{
    const int cx = g.nx - 1, cy = g.ny - 1, cz = g.nz - 1;
    if (L.t_max_i <= L.t_max_j && L.t_max_i <= L.t_max_k) {
        L.t_cur = L.t_max_i;
        L.t_max_i += L.t_d_i;
        L.ci += (L.steps & 1) ? 1 : -1;
        if (L.ci < 0 || L.ci >= cx) return false;
    } else if (L.t_max_j <= L.t_max_k) {
        L.t_cur = L.t_max_j;
        L.t_max_j += L.t_d_j;
        L.cj += (L.steps & 2) ? 1 : -1;
        if (L.cj < 0 || L.cj >= cy) return false;
    } else {
        L.t_cur = L.t_max_k;
        L.t_max_k += L.t_d_k;
        L.ck += (L.steps & 4) ? 1 : -1;
        if (L.ck < 0 || L.ck >= cz) return false;
    }
    return !(L.t_cur >= L.t_far);
}

// K:102-129 fold boundaries of the probe range [t0, t1]
__device__ __forceinline__ void lane_fold(Lane& L)
{
    int n = 0;
    double tmp0 = 0.0, tmp1 = 0.0, tmp2 = 0.0;
    const double cw[3] = {L.wx, L.wy, L.wz};
    const double cd[3] = {L.dx, L.dy, L.dz};
#pragma unroll
    for (int axis = 0; axis < 3; axis++) {
        const double d = cd[axis];
        if (d != 0.0) {
            const double tc = -cw[axis] / d;
            if (L.t0 < tc && tc < L.t1) {
                if (n == 0) tmp0 = tc;
                else if (n == 1) tmp1 = tc;
                else tmp2 = tc;
                n++;
            }
        }
    }
    if (n >= 2 && tmp0 > tmp1) { double t = tmp0; tmp0 = tmp1; tmp1 = t; }
    if (n == 3 && tmp1 > tmp2) {
        const double key = tmp2;
        tmp2 = tmp1;
        if (tmp0 > key) { tmp1 = tmp0; tmp0 = key; }
        else tmp1 = key;
    }
    L.b1 = n > 0 ? tmp0 : L.t1;
    L.b2 = n > 1 ? tmp1 : L.t1;
    L.b3 = n > 2 ? tmp2 : L.t1;
    L.nb = n + 2;
    L.seg_i = 0;
}

// Transition phase: advance a non-stepping lane until it reaches a stepping
// state (S_LO), finishes its ray (S_EMIT) or has no ray (S_FETCH/S_EXIT).
template <int MODE>
__device__ __forceinline__ int lane_transition(Lane& L, int state,
                                               const DevProbes& ps,
                                               const GridParams& g, Diag& dg)
{
    const int R = ps.R;
#pragma unroll 1
    while (state == S_CUBE || state == S_PROBE || state == S_SEG) {
        if (state == S_CUBE) {
            lane_cube(L, ps, g);
            state = S_PROBE;
        } else if (state == S_PROBE) {
            if (L.oi == 8) {
                // K:795-799: the cube's last UNKNOWN is a diagnostic only
                if (L.last_p >= 0) {
                    L.best_p = L.last_p; L.best_tx = L.last_tx; L.best_ty = L.last_ty;
                }
                if (lane_next_cube(L, g)) {
                    state = S_CUBE;
                } else {
                    L.status = MISS; L.rp = L.best_p; L.rtx = L.best_tx;
                    L.rty = L.best_ty;
                    state = S_EMIT;
                }
                continue;
            }
            const int c = (L.order >> (4 * L.oi)) & 15;
            const int nyz = g.ny * g.nz;
            L.p = L.base + ((c >> 2) & 1) * nyz + ((c >> 1) & 1) * g.nz + (c & 1);
            LFP_BCHK(L.p, ps.P, 202);
            L.wx = L.ex - __ldg(ps.origins + 3 * L.p + 0);
            L.wy = L.ey - __ldg(ps.origins + 3 * L.p + 1);
            L.wz = L.ez - __ldg(ps.origins + 3 * L.p + 2);
            const double wlen = sqrt(L.wx * L.wx + L.wy * L.wy + L.wz * L.wz);
            if (wlen < g.eps_align && L.t0 <= g.eps_start * 2.0) {
                // K:617-634 eye-aligned single lookup
                double u, v;
                oct_encode_s(L.dx, L.dy, L.dz, u, v);
                int tx = (int)(u * (double)R);
                int ty = (int)(v * (double)R);
                if (tx > R - 1) tx = R - 1;
                if (ty > R - 1) ty = R - 1;
                LFP_BCHK(tx, R, 203); LFP_BCHK(ty, R, 204);
                const float st = __ldg(ps.dist_hi + (long long)L.p * R * R + tex_index(tx, ty, R, ps.ts_hi));
                L.fetches += 1;
                if (isfinite(st) && (double)st <= L.t1 * (1.0 + g.slack)) {
                    L.status = HIT; L.rp = L.p; L.rtx = tx; L.rty = ty;
                    state = S_EMIT;
                } else {
                    L.oi++;
                }
                continue;
            }
            lane_fold(L);
            state = S_SEG;
        } else {   // S_SEG
            if (L.seg_i >= L.nb - 1) {   // probe range exhausted: MISS
                L.oi++;
                state = S_PROBE;
                continue;
            }
            const int i = L.seg_i;
            const double a = i == 0 ? L.t0 : i == 1 ? L.b1 : i == 2 ? L.b2 : L.b3;
            const double b = i == 0 ? L.b1 : i == 1 ? L.b2 : i == 2 ? L.b3 : L.t1;
            if (b - a < 1e-12) {
                L.seg_i++;
                continue;
            }
            L.c = chord_setup(L.wx, L.wy, L.wz, L.dx, L.dy, L.dz, a, b);
            LFP_DIAG(dg.segs++);
            if (MODE >= 1) *L.cf = chord_f(L.c, L.wx, L.wy, L.wz, L.dx, L.dy, L.dz, g.slack);
            else L.cf->ok = false;
            L.margin = chord_margin(L.c, R);
            L.lo = dda_init(L.c, ps.r, 0.0, false);
            L.occ_x = L.occ_y = -1;
            state = S_LO;
        }
    }
    return state;
}

// End of a probe's segment (K:477-480) or probe result from a candidate:
// `seg_status` MISS -> next segment, UNKNOWN -> the probe returns UNKNOWN
// (K:513-514) and the fall-through continues (K:644-647), HIT -> ray done.
__device__ __forceinline__ int lane_segment_result(Lane& L, int seg_status,
                                                   int tx, int ty)
{
    if (seg_status == MISS) {
        L.seg_i++;
        return S_SEG;
    }
    if (seg_status == HIT) {
        L.status = HIT; L.rp = L.p; L.rtx = tx; L.rty = ty;
        return S_EMIT;
    }
    L.last_p = L.p; L.last_tx = tx; L.last_ty = ty;
    L.oi++;
    return S_PROBE;
}

// Advance the low-res walk after the current block (K:469-480).
__device__ __forceinline__ int lane_lo_advance(Lane& L, int res)
{
    dda_advance(L.lo);
    if (L.lo.s >= 1.0 || L.lo.ix < 0 || L.lo.ix >= res || L.lo.iy < 0 ||
        L.lo.iy >= res) {
        if (L.occ_x >= 0) return lane_segment_result(L, UNKNOWN, L.occ_x, L.occ_y);
        return lane_segment_result(L, MISS, -1, -1);
    }
    return S_LO;
}

// One low-res step (K:432-467): fetch, decide, maybe start a hi-res scan.
template <int MODE>
__device__ __forceinline__ int lane_lo_step(Lane& L, const DevProbes& ps,
                                            double slack, Diag& dg)
{
    const int res = ps.r;
    L.fetches += lo_fetches(L.lo.ix, L.lo.iy, res);
    LFP_BCHK(L.lo.ix, res, 205); LFP_BCHK(L.lo.iy, res, 206);
    const float m_f = __ldg(ps.dil_lo + (long long)L.p * res * res +
                            tex_index(L.lo.ix, L.lo.iy, res, ps.ts_lo));
    if (isfinite(m_f)) {
        double s_out = L.lo.t_max_x < L.lo.t_max_y ? L.lo.t_max_x : L.lo.t_max_y;
        if (s_out > 1.0) s_out = 1.0;
        if (lo_decide<MODE>(ps, L.c, *L.cf, m_f, L.lo.s, s_out, L.margin, L.wx, L.wy,
                            L.wz, L.dx, L.dy, L.dz, slack, dg)) {
            L.hi = dda_init_hi(L.c, ps.R, L.lo.s, L.lo, ps.inv_k);
            L.s_end = s_out;
            L.prev_s = CUDART_NAN;
            L.prev_r = 0.0;
            L.hocc_x = -1;
            return S_HI;
        }
    }
    return lane_lo_advance(L, res);
}

// One high-res step (K:214-267).
template <int MODE>
__device__ __forceinline__ int lane_hi_step(Lane& L, const DevProbes& ps,
                                            double slack, Diag& dg)
{
    const int res = ps.R;
    const long long pbase = (long long)L.p * res * res;
    const int ti = L.hi.iy * res + L.hi.ix;
    LFP_BCHK(L.hi.ix, res, 207); LFP_BCHK(L.hi.iy, res, 208);
    const float stored_f = __ldg(ps.dist_hi + pbase + tex_index(L.hi.ix, L.hi.iy, res, ps.ts_hi));
    L.fetches += 1;
    if (isfinite(stored_f)) {
        double s_hi = L.hi.t_max_x < L.hi.t_max_y ? L.hi.t_max_x : L.hi.t_max_y;
        if (s_hi > L.s_end) s_hi = L.s_end;
        if (s_hi > 1.0) s_hi = 1.0;
        const double s_lo = L.hi.s > 0.0 ? L.hi.s : 0.0;
        const int cls = hi_classify<MODE>(ps, L.c, *L.cf, stored_f, s_lo, s_hi, ti,
                                          L.wx, L.wy, L.wz, L.dx, L.dy, L.dz,
                                          slack, L.prev_s, L.prev_r, dg);
        if (cls == 1) {
            L.hocc_x = L.hi.ix;
            L.hocc_y = L.hi.iy;
        } else if (cls == 2) {
            // K:246-254 resolves the segment (and the probe range)
            const int st = candidate_status(ps, pbase + ti, L.dx, L.dy, L.dz);
            return lane_segment_result(L, st, L.hi.ix, L.hi.iy);
        }
    }
    dda_advance(L.hi);
    if (L.hi.s > L.s_end + 1e-12 || L.hi.s > 1.0 || L.hi.ix < 0 ||
        L.hi.ix >= res || L.hi.iy < 0 || L.hi.iy >= res) {
        // scan over the block ended without a candidate (K:462-467)
        if (L.hocc_x >= 0) {
            L.occ_x = L.hocc_x;
            L.occ_y = L.hocc_y;
        }
        return lane_lo_advance(L, ps.r);
    }
    return S_HI;
}

}  // namespace lfp
