// lfp_wave.cuh -- wavefront (probe-sorted) traversal of explicit ray
// batches (sm_100a).
//
// Incoherent rays (BASELINE config 5) defeat both one-thread-per-ray
// schedules: the nested traversal idles most lanes behind the warp's
// slowest ray, and the persistent state machine (lfp_persistent.cuh) keeps
// its lanes busy but in different phases (cube set-up, segment set-up,
// low-res step, high-res step), executed one after another, from a code
// footprint that misses the instruction cache.
//
// Here the unit of work is ONE probe trace of the reference's fall-through
// (K:603-647). Each iteration, every live ray traces the next probe of its
// current cube's order (K:758-785) over [max(t_cur, 0), t_exit_cube]; a HIT
// finishes the ray, a MISS / UNKNOWN moves on (the next corner, or the next
// cube of the walk, K:801-821) and the ray re-enters the queue keyed by
// (next probe, where its chord starts and ends on the probe's maps)
// (wave_key). The queue
// is radix-sorted by that key between iterations, so the 32 lanes of a
// warp trace the SAME probe map along nearly the same chord: one code path
// (probe range -> segments -> low-/high-res DDA), similar step counts,
// shared texels in L1. Per-ray decisions are the shared
// helpers of lfp_trace.cuh, so outputs are identical to the other schedules
// and to the reference; only the order of work changes.
//
// Ray state between iterations: ONE record per ray, indexed by input ray id
// (96 B for f32 rays, 128 B for f64 rays):
//   [0, R)        origin, direction (f32 x6 + pad / f64 x6 + pad), written
//                 once when the ray enters the lattice
//   [S-64, S-32)  double4 (t_max_i, t_max_j, t_max_k, t_cur)    K:715-738
//   [S-32, S-16)  int4 (ci | cj << 10 | ck << 20, corner order,
//                 oi | fetches << 4, best_p)                    K:758-799
//   [S-16, S-12)  best texel tx | ty << 16                      K:795-799, 822
//   [S-8, S)      t_far, the ray's exit from the lattice        K:668-692
// A re-queued ray is gathered by ray id (the queue is sorted by probe and
// chord, so the ids are random): with separate arrays for origins,
// directions and the three state parts that was five 64-byte DRAM fetches
// per ray and iteration, most of them for 4-16 useful bytes, plus partial-
// sector writes that L2 has to fill first -- the bulk of the wavefront's
// DRAM traffic (ncu: 955 B per probe trace, ~2x the algorithmic bytes). The
// packed record is two fetches and one 64-byte full-sector write-back; the
// input ray arrays are read once (coalesced) by the first iteration.
// The cube increment |cell / d| is recomputed (reference ops, bit-identical)
// only when a ray moves to the next cube.
#pragma once

#include "lfp_persistent.cuh"

namespace lfp {

struct WaveState {
    char* rec;      // [n][stride]
    int stride;     // 96 (f32 rays) or 128 (f64 rays)
};

// Ray state, ray inputs and queues are touched once per iteration and would
// otherwise push the probe maps out of L2 (C5: 2^26 rays x ~100 B per
// iteration vs a 71 MB distance working set): they are read / written with
// evict-first (.cs) hints; the maps are additionally pinned by an L2
// access-policy window on the launch (lfp_capi.cu, LFP_WAVE_L2_PERSIST).
#ifndef LFP_WAVE_STREAMING
#define LFP_WAVE_STREAMING 1
#endif
#if LFP_WAVE_STREAMING
#define LFP_LDCS(p) __ldcs(p)
#define LFP_STCS(p, v) __stcs((p), (v))
#else
#define LFP_LDCS(p) (*(p))
#define LFP_STCS(p, v) (*(p) = (v))
#endif

__device__ __forceinline__ double4 ld_state_cs(const double4* p)
{
    const double2* q = reinterpret_cast<const double2*>(p);
    const double2 a = LFP_LDCS(q), b = LFP_LDCS(q + 1);
    return make_double4(a.x, a.y, b.x, b.y);
}

__device__ __forceinline__ void st_state_cs(double4* p, double4 v)
{
    double2* q = reinterpret_cast<double2*>(p);
    LFP_STCS(q, make_double2(v.x, v.y));
    LFP_STCS(q + 1, make_double2(v.z, v.w));
}

__device__ __forceinline__ char* wave_rec(const WaveState& S, long long ray)
{
    return S.rec + ray * (long long)S.stride;
}
// the mutable 64 bytes of a record
__device__ __forceinline__ void wave_ld_mut(const char* r, int stride, double4& tm,
                                            int4& cw, int& bt, double& t_far)
{
    const char* m = r + stride - 64;
    tm = ld_state_cs(reinterpret_cast<const double4*>(m));
    const int4 a = LFP_LDCS(reinterpret_cast<const int4*>(m + 32));
    const int4 b = LFP_LDCS(reinterpret_cast<const int4*>(m + 48));
    cw = a;
    bt = b.x;
    t_far = __hiloint2double(b.w, b.z);
}
__device__ __forceinline__ void wave_st_mut(char* r, int stride, double4 tm, int4 cw,
                                            int bt, double t_far)
{
    char* m = r + stride - 64;
    st_state_cs(reinterpret_cast<double4*>(m), tm);
    LFP_STCS(reinterpret_cast<int4*>(m + 32), cw);
    LFP_STCS(reinterpret_cast<int4*>(m + 48),
             make_int4(bt, 0, __double2loint(t_far), __double2hiint(t_far)));
}

struct WaveRays {
    const void* ro;      // origins [n][3] (nullptr: shared eye)
    const void* rd;      // directions [n][3]
    double3 eye;
    int f32;
};

__device__ __forceinline__ void wave_load_ray(const WaveRays& rays, long long i,
                                              Lane& L)
{
    if (rays.f32) {
        const float* d = (const float*)rays.rd;
        L.dx = LFP_LDCS(d + 3 * i); L.dy = LFP_LDCS(d + 3 * i + 1);
        L.dz = LFP_LDCS(d + 3 * i + 2);
        if (rays.ro) {
            const float* o = (const float*)rays.ro;
            L.ex = LFP_LDCS(o + 3 * i); L.ey = LFP_LDCS(o + 3 * i + 1);
            L.ez = LFP_LDCS(o + 3 * i + 2);
        }
    } else {
        const double* d = (const double*)rays.rd;
        L.dx = LFP_LDCS(d + 3 * i); L.dy = LFP_LDCS(d + 3 * i + 1);
        L.dz = LFP_LDCS(d + 3 * i + 2);
        if (rays.ro) {
            const double* o = (const double*)rays.ro;
            L.ex = LFP_LDCS(o + 3 * i); L.ey = LFP_LDCS(o + 3 * i + 1);
            L.ez = LFP_LDCS(o + 3 * i + 2);
        }
    }
    if (!rays.ro) { L.ex = rays.eye.x; L.ey = rays.eye.y; L.ez = rays.eye.z; }
}

// origin / direction of a re-queued ray from its record (exact copies of the
// input values; f32 inputs are widened exactly as wave_load_ray does)
__device__ __forceinline__ void wave_ld_ray(const char* r, int f32, Lane& L)
{
    if (f32) {
        const float4 a = LFP_LDCS(reinterpret_cast<const float4*>(r));
        const float2 b = LFP_LDCS(reinterpret_cast<const float2*>(r + 16));
        L.ex = a.x; L.ey = a.y; L.ez = a.z; L.dx = a.w; L.dy = b.x; L.dz = b.y;
    } else {
        const double2 a = LFP_LDCS(reinterpret_cast<const double2*>(r));
        const double2 b = LFP_LDCS(reinterpret_cast<const double2*>(r + 16));
        const double2 c = LFP_LDCS(reinterpret_cast<const double2*>(r + 32));
        L.ex = a.x; L.ey = a.y; L.ez = b.x; L.dx = b.y; L.dy = c.x; L.dz = c.y;
    }
}
__device__ __forceinline__ void wave_st_ray(char* r, int f32, const Lane& L)
{
    if (f32) {
        LFP_STCS(reinterpret_cast<float4*>(r),
                 make_float4((float)L.ex, (float)L.ey, (float)L.ez, (float)L.dx));
        LFP_STCS(reinterpret_cast<float4*>(r + 16),
                 make_float4((float)L.dy, (float)L.dz, 0.0f, 0.0f));
    } else {
        LFP_STCS(reinterpret_cast<double2*>(r), make_double2(L.ex, L.ey));
        LFP_STCS(reinterpret_cast<double2*>(r + 16), make_double2(L.ez, L.dx));
        LFP_STCS(reinterpret_cast<double2*>(r + 32), make_double2(L.dy, L.dz));
        LFP_STCS(reinterpret_cast<double2*>(r + 48), make_double2(0.0, 0.0));
    }
}

// Sort key of a re-queued ray (scheduling only, never a result): the next
// probe p, then a 4-D Morton code of the octahedral cells (2^cbits per axis)
// of the directions from p's origin to the two ends of the ray's range in
// the current cube -- i.e. where the probe-space chord starts and ends on
// p's maps. Rays with nearby keys walk nearly the same texels, so a warp's
// lanes take similar numbers of steps over shared (L1-resident) texels.
__device__ __forceinline__ void wave_oct_cell(float x, float y, float z,
                                              float scale, int hi, int& cu,
                                              int& cv)
{
    const float l1 = fabsf(x) + fabsf(y) + fabsf(z);
    float px = __fdividef(x, l1), pz = __fdividef(z, l1);
    if (y < 0.0f) {
        const float fx = (px >= 0.0f ? 1.0f : -1.0f) * (1.0f - fabsf(pz));
        const float fz = (pz >= 0.0f ? 1.0f : -1.0f) * (1.0f - fabsf(px));
        px = fx;
        pz = fz;
    }
    int u = (int)floorf((px * 0.5f + 0.5f) * scale);
    int v = (int)floorf((pz * 0.5f + 0.5f) * scale);
    cu = u < 0 ? 0 : (u > hi ? hi : u);   // NaN (l1 == 0) -> 0
    cv = v < 0 ? 0 : (v > hi ? hi : v);
}

#ifndef LFP_WAVE_KEY_LEN
#define LFP_WAVE_KEY_LEN 0
#endif
#ifndef LFP_WAVE_KEY_NSEG
#define LFP_WAVE_KEY_NSEG 0
#endif
__device__ __forceinline__ unsigned wave_key(const Lane& L, const DevProbes& ps,
                                             int p, int cbits)
{
    const float ox = (float)__ldg(ps.origins + 3 * p + 0);
    const float oy = (float)__ldg(ps.origins + 3 * p + 1);
    const float oz = (float)__ldg(ps.origins + 3 * p + 2);
    const float ex = (float)L.ex - ox, ey = (float)L.ey - oy, ez = (float)L.ez - oz;
    const float dx = (float)L.dx, dy = (float)L.dy, dz = (float)L.dz;
    const float t0 = (float)L.t0, t1 = (float)L.t1;
    const float scale = (float)(1 << cbits);
    const int hi = (1 << cbits) - 1;
    int c[4];
    const float x0 = ex + t0 * dx, y0 = ey + t0 * dy, z0 = ez + t0 * dz;
    const float x1 = ex + t1 * dx, y1 = ey + t1 * dy, z1 = ez + t1 * dz;
    wave_oct_cell(x0, y0, z0, scale, hi, c[0], c[1]);
    wave_oct_cell(x1, y1, z1, scale, hi, c[2], c[3]);
    // 4-D Morton code: bit b of coordinate k lands at 4 b + (3 - k); each
    // coordinate (<= 8 bits) is spread by three shift-or-mask steps
    unsigned m = 0;
#pragma unroll
    for (int k = 0; k < 4; k++) {
        unsigned x = (unsigned)c[k] & 0xffu;
        x = (x | (x << 12)) & 0x000f000fu;
        x = (x | (x << 6)) & 0x03030303u;
        x = (x | (x << 3)) & 0x11111111u;
        m |= x << (3 - k);
    }
#if LFP_WAVE_KEY_LEN
    // chord length in cells (Manhattan, halved, 5 bits) above the cell code:
    // a warp's lanes then walk about the same number of low-res blocks
    {
        const int sh = cbits > 5 ? cbits - 5 : 0;   // measure at <= 32 cells/axis
        int len = (abs((c[2] >> sh) - (c[0] >> sh)) + abs((c[3] >> sh) - (c[1] >> sh)));
        len = len > 31 ? 31 : len;
        return ((((unsigned)p << 5) | (unsigned)len) << (4 * cbits)) | m;
    }
#elif LFP_WAVE_KEY_NSEG
    // fold crossings of the range (K:102-129: one per axis whose probe-space
    // coordinate changes sign) = segments - 1, above the cell code: a warp's
    // lanes then run the same number of segments (a probe range has 1-4; with
    // mixed lanes the warp runs the longest count with the others idle)
    const unsigned nx = (unsigned)((x0 < 0.0f) != (x1 < 0.0f)) +
                        (unsigned)((y0 < 0.0f) != (y1 < 0.0f)) +
                        (unsigned)((z0 < 0.0f) != (z1 < 0.0f));
    return ((((unsigned)p << 2) | nx) << (4 * cbits)) | m;
#else
    return ((unsigned)p << (4 * cbits)) | m;
#endif
}

__device__ __forceinline__ int wave_probe(const Lane& L, const GridParams& g)
{
    const int c = (L.order >> (4 * L.oi)) & 15;
    return L.base + ((c >> 2) & 1) * g.ny * g.nz + ((c >> 1) & 1) * g.nz + (c & 1);
}

#ifndef LFP_WAVE_RELOAD
#define LFP_WAVE_RELOAD 1
#endif
#ifndef LFP_WAVE_RELOAD_RAY
#define LFP_WAVE_RELOAD_RAY 1
#endif

// The walk state of a re-queued ray (K:715-738 increments recomputed with
// the reference's ops, bit-identical).
__device__ __forceinline__ void wave_restore(Lane& L, const GridParams& g,
                                             const double4 tm, const int4 cw,
                                             const int bt)
{
    L.t_max_i = tm.x; L.t_max_j = tm.y; L.t_max_k = tm.z; L.t_cur = tm.w;
    L.ci = cw.x & 1023; L.cj = (cw.x >> 10) & 1023; L.ck = (cw.x >> 20) & 1023;
    L.order = (unsigned)cw.y;
    L.oi = cw.z & 15;
    L.fetches = (int)((unsigned)cw.z >> 4);
    L.best_p = cw.w;
    L.best_tx = bt < 0 ? -1 : (bt & 0xFFFF);
    L.best_ty = bt < 0 ? -1 : (bt >> 16);
    L.base = (L.ci * g.ny + L.cj) * g.nz + L.ck;
}

// K:801-821 for a re-queued ray: the increment of the axis that steps
// (K:715-738, |cell / d|, the reference's own division) is formed here, once
// per cube change, instead of all three on every iteration.
__device__ __forceinline__ bool wave_next_cube(Lane& L, const GridParams& g)
{
    const int ax = (L.t_max_i <= L.t_max_j && L.t_max_i <= L.t_max_k) ? 0
                   : (L.t_max_j <= L.t_max_k ? 1 : 2);
    const double d = ax == 0 ? L.dx : (ax == 1 ? L.dy : L.dz);
    const double td = d != 0.0 ? fabs(g.cell / d) : CUDART_INF;
    L.t_d_i = td; L.t_d_j = td; L.t_d_k = td;
    return lane_next_cube(L, g);
}

// One iteration for the rays q_in[0..n_in) (q_in == nullptr: identity).
// `first`: the rays enter the lattice (K:653-713) and are queued for their
// first probe without tracing it (so that trace is sorted too). Live rays are
// appended to (key_out, q_out) at positions taken from *n_out; finished
// rays write their outputs (emit_fn) at their input index.
template <int MODE, int CFS, typename EmitFn>
__device__ __forceinline__ void wave_step(const DevProbes& ps, const GridParams& g,
                                          const WaveRays& rays, const WaveState& S,
                                          const int* __restrict__ q_in,
                                          long long n_in, int first,
                                          int sparse_shift,
                                          unsigned* __restrict__ key_out,
                                          int* __restrict__ q_out,
                                          unsigned long long* __restrict__ n_out,
                                          int cbits, ChordF* cfs, Chord* chs,
                                          Range* rgs, EmitFn emit_fn)
{
    const unsigned FULL = 0xffffffffu;
    // Small iterations (the batch's tail: a few thousand long rays) are
    // latency-bound on the serialised paths of each warp's lanes, with most
    // of the GPU idle: they run with 32 >> sparse_shift rays per warp, spread
    // over more warps.
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int lanes = 32 >> sparse_shift;
    const int lane_id = threadIdx.x & 31;
    const long long i = (t >> 5) * lanes + lane_id;
    const bool valid = lane_id < lanes && i < n_in;
    Diag dg = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, cfs};
    dg.chs = chs;
    dg.rgs = rgs;
    Lane L;
    int ray = 0;
    bool done = false, live = false;
    unsigned key = 0;
    if (valid) {
        ray = q_in ? LFP_LDCS(q_in + i) : (int)i;
        if (first) wave_load_ray(rays, ray, L);
        else wave_ld_ray(wave_rec(S, ray), rays.f32, L);
        L.steps = (L.dx > 0.0 ? 1 : 0) | (L.dy > 0.0 ? 2 : 0) | (L.dz > 0.0 ? 4 : 0);
        bool inside = true;
        if (first) {
            inside = lane_ray_init(L, g);
            if (inside) lane_cube(L, ps, g);
        } else {
            // Only what the probe trace needs is computed here (K:749-756,
            // K:603-605); the rest of the walk state is re-read after the
            // trace (LFP_WAVE_RELOAD) so it is not live -- spilled to local
            // memory -- across the trace's loops.
            double4 tm;
            int4 cw;
            int bt0;
            wave_ld_mut(wave_rec(S, ray), S.stride, tm, cw, bt0, L.t_far);
            L.ci = cw.x & 1023; L.cj = (cw.x >> 10) & 1023; L.ck = (cw.x >> 20) & 1023;
            L.order = (unsigned)cw.y;
            L.oi = cw.z & 15;
            L.base = (L.ci * g.ny + L.cj) * g.nz + L.ck;
            double t_exit_cube = tm.x;
            if (tm.y < t_exit_cube) t_exit_cube = tm.y;
            if (tm.z < t_exit_cube) t_exit_cube = tm.z;
            if (t_exit_cube > L.t_far) t_exit_cube = L.t_far;
            L.t0 = (0.0 > tm.w) ? 0.0 : tm.w;
            L.t1 = t_exit_cube;
#if !LFP_WAVE_RELOAD
            wave_restore(L, g, tm, cw, bt0);
#endif
        }
        bool requeue = false;
        if (!inside) {
            done = true;   // misses the lattice: MISS, 0 fetches
        } else if (first) {
            requeue = true;   // entered the lattice: sort before tracing
        } else {
            // K:603-647: the next probe of the cube's fall-through
            L.p = wave_probe(L, g);
            const SegResult s = trace_one_probe<MODE, CFS>(
                ps, L.p, L.ex, L.ey, L.ez, L.dx, L.dy, L.dz, L.t0, L.t1,
                g.eps_start, g.eps_align, g.slack, dg);
#if LFP_WAVE_RELOAD
            {
                // opaque copies that depend on the trace's result: the
                // compiler can neither reuse the loads above nor hoist these
                // above the trace
                const char* rp = wave_rec(S, ray);
                asm volatile("" : "+l"(rp) : "r"(s.status), "r"(s.fetches));
                double4 tm2;
                int4 cw2;
                int bt2;
                // last reads of this iteration: evict-first
                wave_ld_mut(rp, S.stride, tm2, cw2, bt2, L.t_far);
                wave_restore(L, g, tm2, cw2, bt2);
#if LFP_WAVE_RELOAD_RAY
                wave_ld_ray(rp, rays.f32, L);
#endif
            }
#endif
            L.fetches += s.fetches;
            if (s.status == HIT) {
                L.status = HIT; L.rp = L.p; L.rtx = s.tx; L.rty = s.ty;
                done = true;
            } else {
                // the latest UNKNOWN is the walk's diagnostic (K:795-799, 822)
                if (s.status == UNKNOWN) {
                    L.best_p = L.p; L.best_tx = s.tx; L.best_ty = s.ty;
                }
                L.oi++;
                if (L.oi == 8) {
                    if (wave_next_cube(L, g)) {
                        lane_cube(L, ps, g);
                    } else {
                        L.status = MISS; L.rp = L.best_p; L.rtx = L.best_tx;
                        L.rty = L.best_ty;
                        done = true;
                    }
                }
                requeue = !done;
            }
        }
        if (requeue) {
            live = true;
            key = wave_key(L, ps, wave_probe(L, g), cbits);
            char* rp = wave_rec(S, ray);
            if (first) wave_st_ray(rp, rays.f32, L);
            wave_st_mut(rp, S.stride,
                        make_double4(L.t_max_i, L.t_max_j, L.t_max_k, L.t_cur),
                        make_int4(L.ci | (L.cj << 10) | (L.ck << 20), (int)L.order,
                                  (int)(((unsigned)L.fetches << 4) | (unsigned)L.oi),
                                  L.best_p),
                        L.best_tx < 0 ? -1 : (L.best_tx | (L.best_ty << 16)),
                        L.t_far);
        }
    }
    // queue the live rays (warp-aggregated slot allocation)
    const unsigned m = __ballot_sync(FULL, live);
    if (m) {
        const int lane = threadIdx.x & 31;
        unsigned long long base = 0;
        const int leader = __ffs(m) - 1;
        if (lane == leader) base = atomicAdd(n_out, (unsigned long long)__popc(m));
        base = __shfl_sync(FULL, base, leader);
        if (live) {
            const unsigned long long pos = base + __popc(m & ((1u << lane) - 1u));
            LFP_BCHK(pos, n_in, 401);
            LFP_STCS(key_out + pos, key);
            LFP_STCS(q_out + pos, ray);
        }
    }
    emit_fn(valid && done, ray, L, dg);
}

// Tail of a batch: once few rays are left (a few thousand long ones, each
// with dozens of probe traces to go) a wavefront iteration costs its launch,
// sort and host round trip for almost no work. wave_finish traces each
// remaining ray to its end in one launch: the same probe-by-probe steps
// (K:603-647, 801-821), looped in the thread, from the ray's record.
template <int MODE, int CFS, typename EmitFn>
__device__ __forceinline__ void wave_finish(const DevProbes& ps, const GridParams& g,
                                            int f32, const WaveState& S,
                                            const int* __restrict__ q_in,
                                            long long n_in, int sparse_shift,
                                            ChordF* cfs, Chord* chs, Range* rgs,
                                            EmitFn emit_fn)
{
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int lanes = 32 >> sparse_shift;
    const int lane_id = threadIdx.x & 31;
    const long long i = (t >> 5) * lanes + lane_id;
    const bool valid = lane_id < lanes && i < n_in;
    Diag dg = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, cfs};
    dg.chs = chs;
    dg.rgs = rgs;
    Lane L;
    int ray = 0;
    if (valid) {
        ray = LFP_LDCS(q_in + i);
        const char* rp = wave_rec(S, ray);
        wave_ld_ray(rp, f32, L);
        L.steps = (L.dx > 0.0 ? 1 : 0) | (L.dy > 0.0 ? 2 : 0) | (L.dz > 0.0 ? 4 : 0);
        double4 tm;
        int4 cw;
        int bt;
        wave_ld_mut(rp, S.stride, tm, cw, bt, L.t_far);
        wave_restore(L, g, tm, cw, bt);
        // the range inside the current cube (K:749-756, 603-605), as the
        // wavefront iteration forms it
        double t_exit_cube = L.t_max_i;
        if (L.t_max_j < t_exit_cube) t_exit_cube = L.t_max_j;
        if (L.t_max_k < t_exit_cube) t_exit_cube = L.t_max_k;
        if (t_exit_cube > L.t_far) t_exit_cube = L.t_far;
        L.t0 = (0.0 > L.t_cur) ? 0.0 : L.t_cur;
        L.t1 = t_exit_cube;
#pragma unroll 1
        for (;;) {
            L.p = wave_probe(L, g);
            const SegResult s = trace_one_probe<MODE, CFS>(
                ps, L.p, L.ex, L.ey, L.ez, L.dx, L.dy, L.dz, L.t0, L.t1,
                g.eps_start, g.eps_align, g.slack, dg);
            L.fetches += s.fetches;
            if (s.status == HIT) {
                L.status = HIT; L.rp = L.p; L.rtx = s.tx; L.rty = s.ty;
                break;
            }
            if (s.status == UNKNOWN) {
                L.best_p = L.p; L.best_tx = s.tx; L.best_ty = s.ty;
            }
            L.oi++;
            if (L.oi == 8) {
                if (wave_next_cube(L, g)) {
                    lane_cube(L, ps, g);   // order, oi = 0, t0 / t1 of the new cube
                } else {
                    L.status = MISS; L.rp = L.best_p; L.rtx = L.best_tx;
                    L.rty = L.best_ty;
                    break;
                }
            }
        }
    }
    emit_fn(valid, ray, L, dg);
}

}  // namespace lfp
