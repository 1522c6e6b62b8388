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

}  // extern "C"
