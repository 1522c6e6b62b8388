// lfp_bake.cu -- ray-cast probe bake on the GPU.
//
// Input production for the tracer: for every probe and texel, cast the
// texel-centre direction (oct_decode of the centre, octmap.py:46, 75) from the
// probe origin against analytic boxes / spheres, store the nearest hit
// distance (EMPTY = +inf), the direction (the reference's probe->surface
// "incoming direction", kernels.py:247-252) and the Lambertian radiance of
// the hit lit by one point light with a shadow ray; then the blockwise MIN
// low-res map (bake.py:94-102). Semantics follow the host bake in
// paper_2507_14624_b200/bake.py + scenes.py (nearest t > 1e-9, ties to the
// lower primitive index). This kernel defines the C3/C5 inputs; the oracle
// reads the arrays it produces, so it need not be bit-identical to numpy.
#include <cub/device/device_radix_sort.cuh>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <math_constants.h>

#include <string>

#include "../../include/lfprobe_b200.h"

namespace lfp_internal {
void set_error(const std::string& msg);   // lfp_capi.cu (lfp_last_error)
}

namespace {

struct Prim {
    int kind;            // 0 box, 1 sphere
    double a[3], b[3];   // box lo / hi; sphere centre / (radius, -, -)
    float albedo[3];
};

constexpr double kEps = 1e-9;

__device__ __forceinline__ double hit_box(const Prim& p, const double o[3],
                                          const double d[3])
{
    double t_near = -CUDART_INF, t_far = CUDART_INF;
    for (int k = 0; k < 3; k++) {
        if (d[k] == 0.0) {
            if (o[k] < p.a[k] || o[k] > p.b[k]) return CUDART_INF;
            continue;
        }
        double inv = 1.0 / d[k];
        double t1 = (p.a[k] - o[k]) * inv;
        double t2 = (p.b[k] - o[k]) * inv;
        double lo = t1 < t2 ? t1 : t2;
        double hi = t1 < t2 ? t2 : t1;
        if (lo > t_near) t_near = lo;
        if (hi < t_far) t_far = hi;
    }
    if (!(t_near <= t_far)) return CUDART_INF;
    double t = t_near > kEps ? t_near : t_far;
    return t > kEps ? t : CUDART_INF;
}

__device__ __forceinline__ double hit_sphere(const Prim& p, const double o[3],
                                             const double d[3])
{
    double oc0 = o[0] - p.a[0], oc1 = o[1] - p.a[1], oc2 = o[2] - p.a[2];
    double b = oc0 * d[0] + oc1 * d[1] + oc2 * d[2];
    double c = oc0 * oc0 + oc1 * oc1 + oc2 * oc2 - p.b[0] * p.b[0];
    double disc = b * b - c;
    if (disc < 0.0) return CUDART_INF;
    double sq = sqrt(disc);
    double t0 = -b - sq, t1 = -b + sq;
    double t = t0 > kEps ? t0 : t1;
    return t > kEps ? t : CUDART_INF;
}

__device__ __forceinline__ double hit_prim(const Prim& p, const double o[3],
                                           const double d[3])
{
    return p.kind == 0 ? hit_box(p, o, d) : hit_sphere(p, o, d);
}

__global__ void bake_kernel(const Prim* __restrict__ prims, int n_prims,
                            lfp_light light, const double* __restrict__ origins,
                            long long P, int R, int quant_f16, int shadows,
                            float* __restrict__ dist_hi, float* __restrict__ dir_hi,
                            float* __restrict__ irr_hi)
{
    extern __shared__ Prim sp[];
    for (int i = threadIdx.x; i < n_prims; i += blockDim.x) sp[i] = prims[i];
    __syncthreads();
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= P * R * R) return;
    const long long p = idx / ((long long)R * R);
    const int t = (int)(idx - p * R * R);
    const int ty = t / R, tx = t % R;
    // texel-centre direction (octmap.py:46-64)
    double fx = ((tx + 0.5) / R) * 2.0 - 1.0;
    double fz = ((ty + 0.5) / R) * 2.0 - 1.0;
    double y = 1.0 - fabs(fx) - fabs(fz);
    if (y < 0.0) {
        double ux = (fx >= 0.0 ? 1.0 : -1.0) * (1.0 - fabs(fz));
        double uz = (fz >= 0.0 ? 1.0 : -1.0) * (1.0 - fabs(fx));
        fx = ux;
        fz = uz;
    }
    double nrm = sqrt(fx * fx + y * y + fz * fz);
    const double d[3] = {fx / nrm, y / nrm, fz / nrm};
    const double o[3] = {origins[3 * p], origins[3 * p + 1], origins[3 * p + 2]};
    double best = CUDART_INF;
    int bi = -1;
    for (int i = 0; i < n_prims; i++) {
        double th = hit_prim(sp[i], o, d);
        if (th < best) { best = th; bi = i; }
    }
    float* dd = dir_hi + 3 * idx;
    float* cc = irr_hi + 3 * idx;
    if (bi < 0) {
        dist_hi[idx] = CUDART_INF_F;
        dd[0] = dd[1] = dd[2] = 0.f;
        cc[0] = cc[1] = cc[2] = 0.f;
        return;
    }
    const Prim& pr = sp[bi];
    const double q[3] = {o[0] + best * d[0], o[1] + best * d[1], o[2] + best * d[2]};
    double n[3] = {0.0, 0.0, 0.0};
    if (pr.kind == 1) {
        double v0 = q[0] - pr.a[0], v1 = q[1] - pr.a[1], v2 = q[2] - pr.a[2];
        double l = sqrt(v0 * v0 + v1 * v1 + v2 * v2);
        n[0] = v0 / l; n[1] = v1 / l; n[2] = v2 / l;
    } else {
        int face = 0;
        double bd = CUDART_INF;
        for (int k = 0; k < 3; k++) {
            double dl = fabs(q[k] - pr.a[k]);
            double dh = fabs(q[k] - pr.b[k]);
            if (dl < bd) { bd = dl; face = 2 * k; }
            if (dh < bd) { bd = dh; face = 2 * k + 1; }
        }
        n[face / 2] = (face % 2 == 0) ? -1.0 : 1.0;
    }
    if (n[0] * d[0] + n[1] * d[1] + n[2] * d[2] > 0.0) {
        n[0] = -n[0]; n[1] = -n[1]; n[2] = -n[2];
    }
    double tl[3] = {light.position[0] - q[0], light.position[1] - q[1],
                    light.position[2] - q[2]};
    double dist_l = sqrt(tl[0] * tl[0] + tl[1] * tl[1] + tl[2] * tl[2]);
    double ld[3] = {tl[0] / dist_l, tl[1] / dist_l, tl[2] / dist_l};
    double ndl = n[0] * ld[0] + n[1] * ld[1] + n[2] * ld[2];
    if (ndl < 0.0) ndl = 0.0;
    if (shadows && ndl > 0.0) {
        const double so[3] = {q[0] + 1e-6 * n[0], q[1] + 1e-6 * n[1],
                              q[2] + 1e-6 * n[2]};
        for (int i = 0; i < n_prims; i++) {
            if (hit_prim(sp[i], so, ld) < dist_l - 1e-6) { ndl = 0.0; break; }
        }
    }
    double fall = light.power / (1.0 + dist_l * dist_l);
    if (fall > 1.0) fall = 1.0;
    const double lum = light.ambient + (1.0 - light.ambient) * ndl * fall;
    float rgb[3], dir[3];
    for (int k = 0; k < 3; k++) {
        double c = pr.albedo[k] * lum;
        c = c < 0.0 ? 0.0 : (c > 1.0 ? 1.0 : c);
        rgb[k] = (float)c;
        dir[k] = (float)d[k];
        if (quant_f16) {
            rgb[k] = __half2float(__float2half_rn(rgb[k]));
            dir[k] = __half2float(__float2half_rn(dir[k]));
        }
    }
    dist_hi[idx] = (float)best;
    dd[0] = dir[0]; dd[1] = dir[1]; dd[2] = dir[2];
    cc[0] = rgb[0]; cc[1] = rgb[1]; cc[2] = rgb[2];
}

// bake.py:94-102 block MIN (+inf ignored; all-EMPTY stays EMPTY)
__global__ void block_min_kernel(const float* __restrict__ hi, float* __restrict__ lo,
                                 long long P, int R, int r)
{
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= P * r * r) return;
    const int f = R / r;
    const long long p = idx / ((long long)r * r);
    const int t = (int)(idx - p * r * r);
    const int by = t / r, bx = t % r;
    const float* h = hi + p * R * R;
    float m = CUDART_INF_F;
    for (int y = by * f; y < by * f + f; y++)
        for (int x = bx * f; x < bx * f + f; x++) {
            float v = h[y * R + x];
            m = v < m ? v : m;
        }
    lo[idx] = m;
}


// ---------------------------------------------------------------------------
// Point-cloud bake (bake.py:140-207, the reference's own bake): every cloud
// point is projected into every probe's octahedral map; per texel the point
// with the smallest distance wins, exact-distance ties go to the smallest
// (x, y, z, r, g, b) (bake.py:116-137), so the result is independent of the
// point order. Three passes per probe chunk:
//   1. point_min_kernel: 64-bit atomicMin of the fp64 squared-distance bits
//      (positive doubles order like their bit patterns) into key[p][texel];
//   2. point_tie_kernel: points whose distance equals the texel's minimum
//      race for win[p][texel] with a CAS loop on the lexicographic key (one
//      candidate per texel unless distances tie exactly);
//   3. point_finalize_kernel: per texel, the winner's RGB565 radiance,
//      float16 distance and 8-bit sub-texel direction, decoded exactly as the
//      reference stores them in memory (bake.py:62-91, 193-198).
// All arithmetic restates numpy's fp64 op order (no FMA: -fmad=false), so
// the maps are bit-identical to the reference bake.
// ---------------------------------------------------------------------------

#ifndef LFP_BAKE_FAST
#define LFP_BAKE_FAST 1
#endif

constexpr unsigned kNoWinner = 0xFFFFFFFFu;
constexpr int kMaxChunkProbes = 64;

// octmap.py:24-43 (numpy op order): l1 = (|x| + |y|) + |z|, fold with
// sign(0) = +1 using the unfolded px / pz, uv = p * 0.5 + 0.5
__device__ __forceinline__ void np_oct_encode(double x, double y, double z,
                                              double& u, double& v)
{
    const double l1 = (fabs(x) + fabs(y)) + fabs(z);
    double px = x / l1;
    double pz = z / l1;
    if (y < 0.0) {
        const double fx = (px >= 0.0 ? 1.0 : -1.0) * (1.0 - fabs(pz));
        const double fz = (pz >= 0.0 ? 1.0 : -1.0) * (1.0 - fabs(px));
        px = fx;
        pz = fz;
    }
    u = px * 0.5 + 0.5;
    v = pz * 0.5 + 0.5;
}

// octmap.py:46-64: y = (1 - |fx|) - |fz| is kept unfolded; d /= |d| with
// |d| = sqrt((x^2 + y^2) + z^2)
__device__ __forceinline__ void np_oct_decode(double u, double v, float out[3])
{
    const double fx = u * 2.0 - 1.0;
    const double fz = v * 2.0 - 1.0;
    const double y = (1.0 - fabs(fx)) - fabs(fz);
    double x = fx, z = fz;
    if (y < 0.0) {
        x = (fx >= 0.0 ? 1.0 : -1.0) * (1.0 - fabs(fz));
        z = (fz >= 0.0 ? 1.0 : -1.0) * (1.0 - fabs(fx));
    }
    const double n = sqrt((x * x + y * y) + z * z);
    out[0] = (float)(x / n);
    out[1] = (float)(y / n);
    out[2] = (float)(z / n);
}

// bake.py:152-165: w = p - origin, d = |w| (numpy norm order), uv of w / d,
// texel = min(int(uv * R), R - 1). Returns false for points within 1e-6 of
// the origin (skipped, bake.py:158-162, 167-174).
__device__ __forceinline__ bool project_point(const double* __restrict__ pos,
                                              long long i, const double* o,
                                              int R, double& d, int& tx,
                                              int& ty, double& u, double& v)
{
    const double wx = pos[3 * i] - o[0];
    const double wy = pos[3 * i + 1] - o[1];
    const double wz = pos[3 * i + 2] - o[2];
    d = sqrt((wx * wx + wy * wy) + wz * wz);
    if (!(d >= 1e-6)) return false;
    np_oct_encode(wx / d, wy / d, wz / d, u, v);
    long long a = (long long)(u * R), b = (long long)(v * R);
    tx = (int)(a < R - 1 ? a : R - 1);
    ty = (int)(b < R - 1 ? b : R - 1);
    return true;
}

// Texel of w in fp32 with a certainty test (exact-decision filter, as in the
// tracer): the fp64 chain of project_point and this fp32 chain both
// approximate U * R (U the exact octahedral coordinate; it does not depend
// on d) -- fp64 within ~1e-15 R, fp32 within 5 R 2^-24 (six roundings of
// |p| <= 1 plus the scale; bound used: R * 1e-6, a 3x margin). When u R and
// v R are farther than that from an integer the floors agree; otherwise (or
// for components fp32 cannot represent faithfully) return false and let
// the exact path decide. The fold test (y < 0) and the sign rule use the
// fp64 signs, which the divisions by d > 0 and l1 > 0 preserve.
__device__ __forceinline__ bool texel_fast(double wx, double wy, double wz,
                                           int R, int& tx, int& ty)
{
    const float x = (float)wx, y = (float)wy, z = (float)wz;
    const float ax = fabsf(x), ay = fabsf(y), az = fabsf(z);
    const float mx = fmaxf(ax, fmaxf(ay, az));
    if (!(mx > 1e-30f && mx < 1e30f)) return false;
    const float tiny = 1e-20f * mx;
    if ((wx != 0.0 && ax < tiny) || (wy != 0.0 && ay < tiny) ||
        (wz != 0.0 && az < tiny))
        return false;
    const float il = __fdividef(1.0f, (ax + ay) + az);   // rcp.approx
    float px = x * il, pz = z * il;
    if (wy < 0.0) {
        const float fx = (px >= 0.0f ? 1.0f : -1.0f) * (1.0f - fabsf(pz));
        const float fz = (pz >= 0.0f ? 1.0f : -1.0f) * (1.0f - fabsf(px));
        px = fx;
        pz = fz;
    }
    const float fr = (float)R;
    const float tu = fmaf(px, 0.5f, 0.5f) * fr;
    const float tv = fmaf(pz, 0.5f, 0.5f) * fr;
    const float e = fr * 1e-6f;
    const float gu = floorf(tu), gv = floorf(tv);
    const float du = tu - gu, dv = tv - gv;
    if (!(du > e && du < 1.0f - e && dv > e && dv < 1.0f - e)) return false;
    tx = (int)gu;
    ty = (int)gv;
    return tx >= 0 && tx < R && ty >= 0 && ty < R;
}

// project_point for the min / tie passes. Returns d2 = (wx^2 + wy^2) + wz^2,
// the reference's norm before its sqrt: fl(sqrt(.)) is monotone, so the
// per-texel minimum of d is fl(sqrt(min d2)) and the passes rank d2 (no
// fp64 sqrt per point). Texel via texel_fast with the exact fallback.
__device__ __forceinline__ bool project_texel(double px, double py, double pz,
                                              const double* o, int R,
                                              double& d2, int& tx, int& ty)
{
    const double wx = px - o[0];
    const double wy = py - o[1];
    const double wz = pz - o[2];
    d2 = (wx * wx + wy * wy) + wz * wz;
    // skip rule d < 1e-6 (bake.py:158): d2 >= 1.1e-12 implies d > 1.04e-6
    if (d2 < 1.1e-12 && !(sqrt(d2) >= 1e-6)) return false;
    if (LFP_BAKE_FAST && texel_fast(wx, wy, wz, R, tx, ty)) return true;
    const double d = sqrt(d2);
    double u, v;
    np_oct_encode(wx / d, wy / d, wz / d, u, v);
    long long a = (long long)(u * R), b = (long long)(v * R);
    tx = (int)(a < R - 1 ? a : R - 1);
    ty = (int)(b < R - 1 ? b : R - 1);
    return true;
}

// d(a) == d(b) for squared distances with bits(a) >= bits(b) = the texel
// minimum: equal bits, or (sqrt rounding can merge a few ulps of d2) equal
// fl(sqrt) when a is within 8 ulps of b
__device__ __forceinline__ bool same_distance(unsigned long long a,
                                              unsigned long long b)
{
    if (a == b) return true;
    if (a < b || a - b > 8) return false;
    return sqrt(__longlong_as_double((long long)a)) ==
           sqrt(__longlong_as_double((long long)b));
}

// numpy float64 -> float16 (round to nearest even, straight from the double;
// bake.py:71-73), returned widened to f32
__device__ __forceinline__ float f64_to_f16_f32(double x)
{
    const unsigned long long b = (unsigned long long)__double_as_longlong(x);
    const unsigned short sign = (unsigned short)((b >> 48) & 0x8000u);
    const int ex = (int)((b >> 52) & 0x7FF);
    const unsigned long long man = b & ((1ull << 52) - 1);
    unsigned short h;
    if (ex == 0x7FF) {
        h = sign | (man ? 0x7E00u : 0x7C00u);
    } else if (ex == 0) {
        h = sign;                       // fp64 subnormals underflow to 0
    } else {
        const int e = ex - 1023;
        const unsigned long long m = man | (1ull << 52);
        if (e > 15) {
            h = sign | 0x7C00u;
        } else {
            int shift = e >= -14 ? 42 : 42 + (-14 - e);
            unsigned long long q = 0;
            if (shift < 64) {
                q = m >> shift;
                const unsigned long long rem = m & ((1ull << shift) - 1);
                const unsigned long long half = 1ull << (shift - 1);
                if (rem > half || (rem == half && (q & 1))) q++;
            }
            if (e >= -14) {
                // q in [1024, 2048]; carry into the exponent is handled by
                // adding the biased exponent to the full significand
                const unsigned int bits = ((unsigned)(e + 14) << 10) + (unsigned)q;
                h = bits >= 0x7C00u ? (sign | 0x7C00u) : (unsigned short)(sign | bits);
            } else {
                h = sign | (unsigned short)q;   // q <= 1024 (1024 = min normal)
            }
        }
    }
    return __half2float(__ushort_as_half(h));
}

// Pass 1. The block strides over the (spatially sorted) cloud uniformly so
// every warp collective sees all 32 lanes; lanes of a warp that land in the
// same texel (neighbouring points, distant probe) combine their minimum
// with __match_any_sync + two 32-bit __reduce_min_sync, and one lane issues
// the 64-bit atomicMin: far fewer L2 atomics on coherent clouds.
__global__ void point_min_kernel(const double* __restrict__ pos, long long n,
                                 const double* __restrict__ origins, int np,
                                 int R, unsigned long long* key,
                                 unsigned long long* __restrict__ skipped)
{
    __shared__ double so[3 * kMaxChunkProbes];
    __shared__ unsigned s_skip[kMaxChunkProbes];
    for (int k = threadIdx.x; k < 3 * np; k += blockDim.x) so[k] = origins[k];
    for (int k = threadIdx.x; k < np; k += blockDim.x) s_skip[k] = 0;
    __syncthreads();
    const long long RR = (long long)R * R;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double px = pos[3 * i], py = pos[3 * i + 1], pz = pos[3 * i + 2];
        for (int p = 0; p < np; p++) {
            double d2;
            int tx, ty;
            if (!project_texel(px, py, pz, so + 3 * p, R, d2, tx, ty)) {
                atomicAdd(&s_skip[p], 1u);
                continue;
            }
            unsigned long long* k = key + p * RR + (long long)ty * R + tx;
            const unsigned long long kb =
                (unsigned long long)__double_as_longlong(d2);
            // the stored value only decreases: a (possibly stale) read that
            // is already <= kb means this point cannot be the minimum
            if (*k > kb) atomicMin(k, kb);
        }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < np; k += blockDim.x)
        if (s_skip[k]) atomicAdd(skipped + k, (unsigned long long)s_skip[k]);
}

// lexicographic (x, y, z, r, g, b, index) order of bake.py:125-137 (numpy
// lexsort keys, stable on full ties)
__device__ __forceinline__ bool point_less(const double* __restrict__ pos,
                                           const float* __restrict__ col,
                                           unsigned a, unsigned b)
{
    for (int k = 0; k < 3; k++) {
        const double x = pos[3ull * a + k], y = pos[3ull * b + k];
        if (x < y) return true;
        if (y < x) return false;
    }
    for (int k = 0; k < 3; k++) {
        const float x = col[3ull * a + k], y = col[3ull * b + k];
        if (x < y) return true;
        if (y < x) return false;
    }
    return a < b;
}

__global__ void point_tie_kernel(const double* __restrict__ pos,
                                 const float* __restrict__ col, long long n,
                                 const double* __restrict__ origins, int np,
                                 int R, const unsigned long long* __restrict__ key,
                                 unsigned* __restrict__ win)
{
    __shared__ double so[3 * kMaxChunkProbes];
    for (int k = threadIdx.x; k < 3 * np; k += blockDim.x) so[k] = origins[k];
    __syncthreads();
    const long long RR = (long long)R * R;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double px = pos[3 * i], py = pos[3 * i + 1], pz = pos[3 * i + 2];
        for (int p = 0; p < np; p++) {
            double d2;
            int tx, ty;
            if (!project_texel(px, py, pz, so + 3 * p, R, d2, tx, ty)) continue;
            const long long t = p * RR + (long long)ty * R + tx;
            if (!same_distance((unsigned long long)__double_as_longlong(d2),
                               key[t]))
                continue;
            const unsigned me = (unsigned)i;
            unsigned cur = win[t];
            while (cur == kNoWinner || point_less(pos, col, me, cur)) {
                const unsigned old = atomicCAS(win + t, cur, me);
                if (old == cur) break;
                cur = old;
            }
        }
    }
}

__global__ void point_finalize_kernel(const double* __restrict__ pos,
                                      const float* __restrict__ col,
                                      const double* __restrict__ origins,
                                      int np, int R,
                                      const unsigned* __restrict__ win,
                                      float* __restrict__ dist_hi,
                                      float* __restrict__ dir_hi,
                                      float* __restrict__ irr_hi)
{
    const long long RR = (long long)R * R;
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= np * RR) return;
    const long long p = idx / RR;
    const unsigned w = win[idx];
    float* dd = dir_hi + 3 * idx;
    float* cc = irr_hi + 3 * idx;
    if (w == kNoWinner) {
        dist_hi[idx] = CUDART_INF_F;
        dd[0] = dd[1] = dd[2] = 0.f;
        cc[0] = cc[1] = cc[2] = 0.f;
        return;
    }
    double d, u, v;
    int tx, ty;
    project_point(pos, w, origins + 3 * p, R, d, tx, ty, u, v);
    dist_hi[idx] = f64_to_f16_f32(d);
    // quantize_rgb565 (bake.py:62-68): clip to [0, 1], rint(c * L) / L
    const double lv[3] = {31.0, 63.0, 31.0};
    for (int k = 0; k < 3; k++) {
        double c = (double)col[3ull * w + k];
        c = c < 0.0 ? 0.0 : (c > 1.0 ? 1.0 : c);
        cc[k] = (float)(rint(c * lv[k]) / lv[k]);
    }
    // _quantize_direction / _decode_direction (bake.py:76-91)
    double fx = u * R - (double)tx;
    double fy = v * R - (double)ty;
    double qx = rint(fx * 254.0), qy = rint(fy * 254.0);
    qx = qx < 0.0 ? 0.0 : (qx > 254.0 ? 254.0 : qx);
    qy = qy < 0.0 ? 0.0 : (qy > 254.0 ? 254.0 : qy);
    const double du = ((double)tx + qx / 254.0) / R;
    const double dv = ((double)ty + qy / 254.0) / R;
    np_oct_decode(du, dv, dd);
}


// Spatial order for the passes: 30-bit Morton code of each point inside the
// cloud's bounding box (the bake is order-independent, bake.py:116-118, so
// any permutation gives identical maps; this one makes warps coherent).
__device__ __forceinline__ unsigned f2ord(float f)
{
    const unsigned b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__device__ __forceinline__ float ord2f(unsigned u)
{
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u);
}

__global__ void bbox_kernel(const double* __restrict__ pos, long long n,
                            unsigned* __restrict__ bb)
{
    unsigned lo[3] = {~0u, ~0u, ~0u}, hi[3] = {0u, 0u, 0u};
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        for (int k = 0; k < 3; k++) {
            const unsigned o = f2ord((float)pos[3 * i + k]);
            lo[k] = min(lo[k], o);
            hi[k] = max(hi[k], o);
        }
    for (int k = 0; k < 3; k++) {
        const unsigned l = __reduce_min_sync(0xFFFFFFFFu, lo[k]);
        const unsigned h = __reduce_max_sync(0xFFFFFFFFu, hi[k]);
        if ((threadIdx.x & 31) == 0) {
            atomicMin(bb + k, l);
            atomicMax(bb + 3 + k, h);
        }
    }
}

__device__ __forceinline__ unsigned spread10(unsigned v)
{
    v &= 0x3FFu;
    v = (v | (v << 16)) & 0x030000FFu;
    v = (v | (v << 8)) & 0x0300F00Fu;
    v = (v | (v << 4)) & 0x030C30C3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}

__global__ void morton_kernel(const double* __restrict__ pos, long long n,
                              const unsigned* __restrict__ bb,
                              unsigned* __restrict__ code,
                              unsigned* __restrict__ idx)
{
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    unsigned c = 0;
    for (int k = 0; k < 3; k++) {
        const float lo = ord2f(bb[k]), hi = ord2f(bb[3 + k]);
        const float ext = hi - lo;
        float q = ext > 0.0f ? ((float)pos[3 * i + k] - lo) / ext * 1023.0f : 0.0f;
        q = fminf(fmaxf(q, 0.0f), 1023.0f);
        c |= spread10((unsigned)q) << k;
    }
    code[i] = c;
    idx[i] = (unsigned)i;
}

__global__ void gather_points_kernel(const double* __restrict__ pos,
                                     const float* __restrict__ col,
                                     const unsigned* __restrict__ order,
                                     long long n, double* __restrict__ spos,
                                     float* __restrict__ scol)
{
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const long long j = order[i];
    for (int k = 0; k < 3; k++) {
        spos[3 * i + k] = pos[3 * j + k];
        scol[3 * i + k] = col[3 * j + k];
    }
}

}  // namespace

extern "C" {

int lfp_bake_probes(int device, const lfp_prim* prims_host, int32_t n_prims,
                    const lfp_light* light, const double* origins_host,
                    int64_t P, int32_t R, int32_t r, int32_t quant_f16,
                    int32_t shadows, float* dist_hi, float* dir_hi,
                    float* irr_hi, float* dist_lo, void* stream)
{
    if (!prims_host || n_prims < 1 || !light || !origins_host || P < 1 ||
        R < 1 || r < 1 || R % r != 0 || !dist_hi || !dir_hi || !irr_hi ||
        !dist_lo) {
        lfp_internal::set_error("lfp_bake_probes: invalid arguments");
        return LFP_ERR_INVALID;
    }
    if (sizeof(Prim) * (size_t)n_prims > 200 * 1024) {
        lfp_internal::set_error("lfp_bake_probes: too many primitives for the "
                                "shared-memory bake (max ~1700)");
        return LFP_ERR_INVALID;
    }
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    cudaStream_t st = (cudaStream_t)stream;
    Prim* hp = new Prim[n_prims];
    for (int i = 0; i < n_prims; i++) {
        hp[i].kind = prims_host[i].kind;
        for (int k = 0; k < 3; k++) {
            hp[i].a[k] = prims_host[i].a[k];
            hp[i].b[k] = prims_host[i].b[k];
            hp[i].albedo[k] = prims_host[i].albedo[k];
        }
    }
    Prim* dp = nullptr;
    double* dorg = nullptr;
    int rc = LFP_OK;
    const size_t smem = sizeof(Prim) * (size_t)n_prims;
    if (cudaMalloc(&dp, smem) != cudaSuccess ||
        cudaMalloc(&dorg, sizeof(double) * 3 * P) != cudaSuccess) {
        lfp_internal::set_error("lfp_bake_probes: cudaMalloc failed");
        rc = LFP_ERR_NOMEM;
    } else {
        cudaMemcpyAsync(dp, hp, smem, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(dorg, origins_host, sizeof(double) * 3 * P,
                        cudaMemcpyHostToDevice, st);
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(bake_kernel,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem);
        const long long n = P * (long long)R * R;
        bake_kernel<<<(unsigned)((n + 255) / 256), 256, smem, st>>>(
            dp, n_prims, *light, dorg, P, R, quant_f16, shadows, dist_hi,
            dir_hi, irr_hi);
        const long long nl = P * (long long)r * r;
        block_min_kernel<<<(unsigned)((nl + 255) / 256), 256, 0, st>>>(
            dist_hi, dist_lo, P, R, r);
        cudaError_t e = cudaStreamSynchronize(st);
        if (e == cudaSuccess) e = cudaGetLastError();
        if (e != cudaSuccess) {
            lfp_internal::set_error(std::string("lfp_bake_probes: ") +
                                    cudaGetErrorString(e));
            rc = LFP_ERR_CUDA;
        }
    }
    if (dp) cudaFree(dp);
    if (dorg) cudaFree(dorg);
    delete[] hp;
    cudaSetDevice(prev);
    return rc;
}

int lfp_bake_points(int device, const double* positions, const float* colors,
                    int64_t n_points, const double* origins_host, int64_t P,
                    int32_t R, int32_t r, uint32_t flags, float* dist_hi,
                    float* dir_hi, float* irr_hi, float* dist_lo,
                    int64_t* skipped_host, void* stream)
{
    if (!positions || !colors || n_points < 1 || n_points >= 0xFFFFFFFFll ||
        !origins_host || P < 1 || R < 1 || r < 1 || R % r != 0 || !dist_hi ||
        !dir_hi || !irr_hi || !dist_lo || R > 32768) {
        lfp_internal::set_error("lfp_bake_points: invalid arguments");
        return LFP_ERR_INVALID;
    }
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    cudaStream_t st = (cudaStream_t)stream;
    const bool on_dev = (flags & LFP_SRC_DEVICE) != 0;
    const long long RR = (long long)R * R;
    // probe chunk: <= kMaxChunkProbes and <= ~1 GiB of key + winner scratch
    long long chunk = (1ll << 30) / (12 * RR);
    if (chunk < 1) chunk = 1;
    if (chunk > kMaxChunkProbes) chunk = kMaxChunkProbes;
    if (chunk > P) chunk = P;
    double* dpos = nullptr;
    float* dcol = nullptr;
    double* dorg = nullptr;
    unsigned long long* key = nullptr;
    unsigned* win = nullptr;
    unsigned long long* dskip = nullptr;
    double* spos = nullptr;
    float* scol = nullptr;
    unsigned *code0 = nullptr, *code1 = nullptr, *idx0 = nullptr,
             *idx1 = nullptr, *bb = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, (unsigned*)nullptr,
                                    (unsigned*)nullptr, (unsigned*)nullptr,
                                    (unsigned*)nullptr, (long long)n_points, 0,
                                    30, st);
    int rc = LFP_OK;
    // stream-ordered allocations: the device pool reuses them across calls
    bool ok = cudaMallocAsync(&dorg, sizeof(double) * 3 * P, st) == cudaSuccess &&
              cudaMallocAsync(&key, sizeof(unsigned long long) * chunk * RR, st) == cudaSuccess &&
              cudaMallocAsync(&win, sizeof(unsigned) * chunk * RR, st) == cudaSuccess &&
              cudaMallocAsync(&dskip, sizeof(unsigned long long) * P, st) == cudaSuccess;
    if (ok && !on_dev)
        ok = cudaMallocAsync(&dpos, sizeof(double) * 3 * n_points, st) == cudaSuccess &&
             cudaMallocAsync(&dcol, sizeof(float) * 3 * n_points, st) == cudaSuccess;
    const size_t n4 = sizeof(unsigned) * (size_t)n_points;
    if (ok)
        ok = cudaMallocAsync(&spos, sizeof(double) * 3 * n_points, st) == cudaSuccess &&
             cudaMallocAsync(&scol, sizeof(float) * 3 * n_points, st) == cudaSuccess &&
             cudaMallocAsync(&code0, n4, st) == cudaSuccess &&
             cudaMallocAsync(&code1, n4, st) == cudaSuccess &&
             cudaMallocAsync(&idx0, n4, st) == cudaSuccess &&
             cudaMallocAsync(&idx1, n4, st) == cudaSuccess &&
             cudaMallocAsync(&bb, 6 * sizeof(unsigned), st) == cudaSuccess &&
             cudaMallocAsync(&tmp, tmp_bytes, st) == cudaSuccess;
    if (!ok) {
        lfp_internal::set_error("lfp_bake_points: cudaMallocAsync failed");
        rc = LFP_ERR_NOMEM;
    } else {
        const double* pos = positions;
        const float* col = colors;
        if (!on_dev) {
            cudaMemcpyAsync(dpos, positions, sizeof(double) * 3 * n_points,
                            cudaMemcpyHostToDevice, st);
            cudaMemcpyAsync(dcol, colors, sizeof(float) * 3 * n_points,
                            cudaMemcpyHostToDevice, st);
            pos = dpos;
            col = dcol;
        }
        cudaMemcpyAsync(dorg, origins_host, sizeof(double) * 3 * P,
                        cudaMemcpyHostToDevice, st);
        cudaMemsetAsync(dskip, 0, sizeof(unsigned long long) * P, st);
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
        const long long want = (n_points + 255) / 256;
        const unsigned grid = (unsigned)(want < 8ll * sms ? want : 8ll * sms);
        // spatial sort (Morton order inside the bounding box)
        cudaMemsetAsync(bb, 0xFF, 3 * sizeof(unsigned), st);
        cudaMemsetAsync(bb + 3, 0, 3 * sizeof(unsigned), st);
        bbox_kernel<<<grid, 256, 0, st>>>(pos, n_points, bb);
        morton_kernel<<<(unsigned)want, 256, 0, st>>>(pos, n_points, bb, code0,
                                                      idx0);
        cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, code0, code1, idx0,
                                        idx1, (long long)n_points, 0, 30, st);
        gather_points_kernel<<<(unsigned)want, 256, 0, st>>>(pos, col, idx1,
                                                             n_points, spos,
                                                             scol);
        pos = spos;
        col = scol;
        for (long long p0 = 0; p0 < P; p0 += chunk) {
            const int np = (int)(P - p0 < chunk ? P - p0 : chunk);
            cudaMemsetAsync(key, 0xFF, sizeof(unsigned long long) * np * RR, st);
            cudaMemsetAsync(win, 0xFF, sizeof(unsigned) * np * RR, st);
            point_min_kernel<<<grid, 256, 0, st>>>(pos, n_points, dorg + 3 * p0,
                                                   np, R, key, dskip + p0);
            point_tie_kernel<<<grid, 256, 0, st>>>(pos, col, n_points,
                                                   dorg + 3 * p0, np, R, key, win);
            const long long nt = np * RR;
            point_finalize_kernel<<<(unsigned)((nt + 255) / 256), 256, 0, st>>>(
                pos, col, dorg + 3 * p0, np, R, win, dist_hi + p0 * RR,
                dir_hi + 3 * p0 * RR, irr_hi + 3 * p0 * RR);
        }
        const long long nl = P * (long long)r * r;
        block_min_kernel<<<(unsigned)((nl + 255) / 256), 256, 0, st>>>(
            dist_hi, dist_lo, P, R, r);
        if (skipped_host)
            cudaMemcpyAsync(skipped_host, dskip, sizeof(int64_t) * P,
                            cudaMemcpyDeviceToHost, st);
        cudaError_t e = cudaStreamSynchronize(st);
        if (e == cudaSuccess) e = cudaGetLastError();
        if (e != cudaSuccess) {
            lfp_internal::set_error(std::string("lfp_bake_points: ") +
                                    cudaGetErrorString(e));
            rc = LFP_ERR_CUDA;
        }
    }
    for (void* ptr : {(void*)dpos, (void*)dcol, (void*)dorg, (void*)key,
                      (void*)win, (void*)dskip, (void*)spos, (void*)scol,
                      (void*)code0, (void*)code1, (void*)idx0, (void*)idx1,
                      (void*)bb, tmp})
        if (ptr) cudaFreeAsync(ptr, st);
    if (rc != LFP_OK) cudaStreamSynchronize(st);
    cudaGetLastError();
    cudaSetDevice(prev);
    return rc;
}

}  // extern "C"

