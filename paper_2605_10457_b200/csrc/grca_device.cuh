// grca_device.cuh -- device math of the GRCA hot path (sm_100a).
//
// Rows of SURVEY.md 8(a) implemented here:
//   A1  triangle load (fused "K1": coalesced float4 gathers, indexed or not)
//   A2  range cull          (Step 1.3; delta_min per Ericson)
//   A3  elevation interval -> channel range   (Obs. 2)
//   A4  azimuth arc -> ray range              (g(j,i) 760-763)
//   A6  certified edge-function ray-triangle test + closest-hit key
//       (Moller-Trumbore 756; f_sort 2340-2356)
//
// Precision contract: every cull is conservative (outward
// padding larger than the fp32 error bound), every fp32 hit/miss decision is
// certified by an a-priori error bound, and uncertain candidates are decided in
// fp64 -- so the result equals the exact-arithmetic closest hit of the fp32 ray
// table up to the 1e-16-relative fp64 boundary cases the parity contract excuses.
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

namespace grca {

// Bounds-checked build (-DGRCA_CHECK; tools/check_build.py): every global index of the hot path is checked
// against its buffer's extent; a violation sets bit `site` of g_check_err and the access is redirected to
// index 0 (no fault), and grca_cast reports the mask.  The product build compiles the checks away.
#ifdef GRCA_CHECK
__device__ unsigned g_check_err;
__device__ __forceinline__ long long chk_idx(long long i, long long n, int site) {
    if (i < 0 || i >= n) {
        atomicOr(&g_check_err, 1u << site);
        return 0;
    }
    return i;
}
#else
__device__ __forceinline__ long long chk_idx(long long i, long long, int) { return i; }
#endif
enum { CHK_SURV_WRITE = 0, CHK_RAY = 1, CHK_VERTEX = 2, CHK_SURV_READ = 3, CHK_LARGE = 4, CHK_CHUNK = 5,
       CHK_TRI = 6 };

constexpr float kU = 5.9604644775390625e-8f;   // 2^-24, unit roundoff of fp32
constexpr float kPadS = 4e-6f;                 // sin(elevation) padding (>> 3u ray rounding)
constexpr float kPadTheta = 5e-5f;             // azimuth padding in radians
constexpr float kNearAxis2 = 1e-3f;            // |x_h|^2 < 1e-3 |x|^2 -> full azimuth (general frames)
constexpr float kNearAxisLevel2 = 1e-10f;      // level frames: x_h has no cancellation (cull_pair)
constexpr float kChordSmall2 = 4e-2f;          // chord^2 below which the L^2/8 edge pad is used
constexpr float kTRel = 4.5e-6f;               // certified relative error of fp32 t
#ifndef GRCA_COLMAX
#define GRCA_COLMAX 128   // K4 chain = one chunk: 128 rays = 4 steps of 32 (measured: 1024 -> 128 took K4 0.046 -> 0.031 ms at C4)
#endif
constexpr int kColMax = GRCA_COLMAX;           // max columns per chunk row segment

// Per-emitter record (device + shared memory).  A = M^-1 with M = [f r u] (fp64 inverse,
// rounded): x = A (p - o) are the coordinates in which ray (j,i) is exactly
// (cos th cos phi, sin th cos phi, sin phi) -- so the cull is exact for any given frame.
struct EmDev {
    float o[3];
    float A[9];
    float theta0, dtheta, inv_dtheta;
    float dmax_lo, dmax_hi;   // certified accept / reject bounds around D_max (+inf if none)
    double dmax;              // fp64 D_max for the fallback (+inf if none)
    int gamma, chi, hfov, ray_base, sin_base, pole_lo, pole_hi, noisy;   // noisy: perturbed theta*_i
    int level;                // A = [[a0 a1 0] [a3 a4 0] [0 0 1]] exactly (level frame): x_u = a_z
};

// Phase-A (K2) view of an emitter: just what the elevation pre-test needs.
struct EmLite {
    float o[3];
    float Au[3];     // up row of A = M^-1: x_u = Au . (p - o)
    float G[6];      // Gram matrix A^T A (G00, G11, G22, G01, G02, G12) for |x| when !ortho
    float lim;       // range-cull limit D_max * (1 + 1e-5), +inf if none
    float pad0;      // kPadS + frame non-orthonormality allowance
    int gamma, sin_base, lut_base, ortho;
};
constexpr int kLutBins = 2048;   // O(1) channel lookup: u8 bins over sin(elevation) in [-1, 1]

struct f3 {
    float x, y, z;
};
struct d3 {
    double x, y, z;
};

__device__ __forceinline__ f3 mk(float4 a) { return {a.x, a.y, a.z}; }
// Fixed operation order (no contraction freedom): bit-identical wherever inlined.
__device__ __forceinline__ f3 subf(f3 a, f3 b) { return {__fsub_rn(a.x, b.x), __fsub_rn(a.y, b.y), __fsub_rn(a.z, b.z)}; }
__device__ __forceinline__ float dotf(f3 a, f3 b) {
    return __fmaf_rn(a.z, b.z, __fmaf_rn(a.y, b.y, __fmul_rn(a.x, b.x)));
}
__device__ __forceinline__ f3 crossf(f3 a, f3 b) {
    return {__fmaf_rn(a.y, b.z, -__fmul_rn(a.z, b.y)), __fmaf_rn(a.z, b.x, -__fmul_rn(a.x, b.z)),
            __fmaf_rn(a.x, b.y, -__fmul_rn(a.y, b.x))};
}
__device__ __forceinline__ f3 scalef(f3 a, float s) { return {__fmul_rn(a.x, s), __fmul_rn(a.y, s), __fmul_rn(a.z, s)}; }
__device__ __forceinline__ d3 tod(f3 a) { return {(double)a.x, (double)a.y, (double)a.z}; }
__device__ __forceinline__ d3 subd(d3 a, d3 b) { return {__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y), __dsub_rn(a.z, b.z)}; }
__device__ __forceinline__ double dotd(d3 a, d3 b) {
    return __fma_rn(a.z, b.z, __fma_rn(a.y, b.y, __dmul_rn(a.x, b.x)));
}
__device__ __forceinline__ d3 crossd(d3 a, d3 b) {
    return {__fma_rn(a.y, b.z, -__dmul_rn(a.z, b.y)), __fma_rn(a.z, b.x, -__dmul_rn(a.x, b.z)),
            __fma_rn(a.x, b.y, -__dmul_rn(a.y, b.x))};
}
// Lexicographic order of fp32 points: the canonical edge direction (watertightness).
__device__ __forceinline__ bool lexless(f3 p, f3 q) {
    const bool lx = p.x < q.x, ex = p.x == q.x, ly = p.y < q.y, ey = p.y == q.y, lz = p.z < q.z;
    return lx | (ex & (ly | (ey & lz)));
}
__device__ __forceinline__ bool finite3(f3 a) { return isfinite(a.x) && isfinite(a.y) && isfinite(a.z); }
// sqrt.approx.ftz (MUFU, relative error ~2^-22, no slow-path call): used only inside conservative
// pads / tolerances of the culls, never in a certified decision
__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// atan2 with |error| <= 2.0e-6 rad (odd degree-11 least-max polynomial on [0, 1] after octant
// reduction; bound checked on 2M points by tests/test_abi_cpu.py through grca_debug_fast_atan2,
// the host build).  The device build divides with __fdividef (<= 2 ulp in z, <= 1.2e-7 rad more).
// Used for vertex azimuths, whose cull pad (kPadTheta = 5e-5) budgets 2.5e-6 for it.
__host__ __device__ __forceinline__ float fast_atan2(float y, float x) {
    const float ax = fabsf(x), ay = fabsf(y);
    const float mx = fmaxf(ax, ay), mn = fminf(ax, ay);
#ifdef __CUDA_ARCH__
    const float z = mx > 0.f ? __fdividef(mn, mx) : 0.f;
#else
    const float z = mx > 0.f ? mn / mx : 0.f;
#endif
    const float z2 = z * z;
    float p = -0.011710336431860924f;
    p = p * z2 + 0.05262540653347969f;
    p = p * z2 - 0.11640699207782745f;
    p = p * z2 + 0.1935330331325531f;
    p = p * z2 - 0.3326217532157898f;
    p = p * z2 + 0.999977171421051f;
    float a = p * z;
    if (ay > ax) a = 1.5707963267948966f - a;
    if (x < 0.f) a = 3.141592653589793f - a;
    return copysignf(a, y);
}

// atan(z) for |z| <= 1 with the same polynomial (|error| <= 2e-6 rad), odd symmetric
__host__ __device__ __forceinline__ float poly_atan(float z) {
    const float az = fabsf(z), z2 = az * az;
    float p = -0.011710336431860924f;
    p = p * z2 + 0.05262540653347969f;
    p = p * z2 - 0.11640699207782745f;
    p = p * z2 + 0.1935330331325531f;
    p = p * z2 - 0.3326217532157898f;
    p = p * z2 + 0.999977171421051f;
    return copysignf(p * az, z);
}

// ----------------------------------------------------------------- A1 load --
struct TriSrc {
    const float4 *va;      // part A (grca_update_scene): triangles [0, n_a) as float4 triplets, then
    long long n_a;         // part B = the source below for triangles [n_a, n) (n_a = 0: B only)
    const float4 *v;       // float4 vertices (w ignored), or
    const float *v3;       // non-NULL: packed float3 vertices (12 B each; grca_update_triangles_f3)
    const uint32_t *idx;   // NULL -> non-indexed triplets
    const int32_t *ids;    // NULL -> id_base + local (global triangle index, parts A and B alike)
    int32_t id_base;
    long long n_v;         // vertices of part B (bounds-checked build only)
    long long n_t;         // triangles of parts A + B (+ C) (bounds-checked build only)
    // part C (grca_update_instances): triangles [n_c0, n_t) are rigid instances of one local mesh: triangle
    // n_c0 + i * c_faces + f is face f of instance i, its local vertices mapped by the instance's 3x4 matrix
    long long n_c0;        // first triangle of part C (LLONG_MAX: no part C)
    const float *cv;       // local vertices, packed float3 (object space)
    const uint32_t *cidx;  // local faces, 3 indices each
    const float4 *cpose;   // per instance 3 float4 rows (m00 m01 m02 m03), (m10 ...), (m20 ...)
    long long c_faces, c_nv, c_ninst;
    float c_inv_faces;     // 1 / c_faces (instance estimate, corrected exactly)
};
__device__ __forceinline__ f3 ldcs3(const float *p) { return {__ldcs(p), __ldcs(p + 1), __ldcs(p + 2)}; }
// Streaming (evict-first) loads: the ~1 GB triangle stream must not evict the L2-resident ray
// table (67 MB at C4) and hit buffer (33.5 MB) that the intersection kernels gather from.
// world = M [v; 1] with every product and sum rounded, in this order (no FMA contraction): a host evaluating
// ((m0 x + m1 y) + m2 z) + m3 in IEEE fp32 reproduces it bit for bit (include/grca.h grca_update_instances)
__device__ __forceinline__ float pose_row(float4 m, f3 p) {
    return __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(m.x, p.x), __fmul_rn(m.y, p.y)), __fmul_rn(m.z, p.z)), m.w);
}
#ifndef GRCA_INST_INLINE
#define GRCA_INST_INLINE 1   // inline: only the kC = true instantiations carry it (measured: out of line, the
                             // instanced C4 frame took 1.120 ms against 1.063 inline)
#endif
#if GRCA_INST_INLINE
__device__ __forceinline__
#else
__device__ __noinline__
#endif
void load_instance_tri(const TriSrc &T, long long u, f3 v[3]) {
    long long i = (long long)__float2ll_rz(__ll2float_rn(u) * T.c_inv_faces);
    long long f = u - i * T.c_faces;
    while (f < 0) { --i; f += T.c_faces; }
    while (f >= T.c_faces) { ++i; f -= T.c_faces; }
#ifdef GRCA_CHECK
    i = chk_idx(i, T.c_ninst, CHK_TRI);
#endif
    const float4 r0 = __ldg(T.cpose + 3 * i), r1 = __ldg(T.cpose + 3 * i + 1), r2 = __ldg(T.cpose + 3 * i + 2);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const long long vi = chk_idx(__ldg(T.cidx + 3 * f + k), T.c_nv, CHK_VERTEX);
        const f3 p = {__ldg(T.cv + 3 * vi), __ldg(T.cv + 3 * vi + 1), __ldg(T.cv + 3 * vi + 2)};
        v[k] = {pose_row(r0, p), pose_row(r1, p), pose_row(r2, p)};
    }
}

// kC: the set may have part C (instances).  The hot kernels (K2, the fused kernel) are instantiated with
// kC = false for sets without instances, so their triangle loads carry no part-C branch at all.
template <bool kC = true>
__device__ __forceinline__ void load_tri(const TriSrc &T, long long t, f3 v[3]) {
#ifdef GRCA_CHECK
    t = chk_idx(t, T.n_t, CHK_TRI);
#endif
    if (kC && t >= T.n_c0) {   // part C: a rigid instance of the local mesh (grca_update_instances)
        load_instance_tri(T, t - T.n_c0, v);
        return;
    }
    if (t < T.n_a) {   // part A: float4 triplets, no indirection (static scenery)
        v[0] = mk(__ldcs(T.va + 3 * t));
        v[1] = mk(__ldcs(T.va + 3 * t + 1));
        v[2] = mk(__ldcs(T.va + 3 * t + 2));
        return;
    }
    t -= T.n_a;
    if (T.idx) {
#ifdef GRCA_CHECK
        const uint32_t i0 = (uint32_t)chk_idx(__ldcs(T.idx + 3 * t), T.n_v, CHK_VERTEX),
                       i1 = (uint32_t)chk_idx(__ldcs(T.idx + 3 * t + 1), T.n_v, CHK_VERTEX),
                       i2 = (uint32_t)chk_idx(__ldcs(T.idx + 3 * t + 2), T.n_v, CHK_VERTEX);
#else
        const uint32_t i0 = __ldcs(T.idx + 3 * t), i1 = __ldcs(T.idx + 3 * t + 1), i2 = __ldcs(T.idx + 3 * t + 2);
#endif
        if (T.v3) {
            v[0] = ldcs3(T.v3 + 3ll * i0);
            v[1] = ldcs3(T.v3 + 3ll * i1);
            v[2] = ldcs3(T.v3 + 3ll * i2);
        } else {
            v[0] = mk(__ldcs(T.v + i0));
            v[1] = mk(__ldcs(T.v + i1));
            v[2] = mk(__ldcs(T.v + i2));
        }
    } else if (T.v3) {
        v[0] = ldcs3(T.v3 + 9 * t);
        v[1] = ldcs3(T.v3 + 9 * t + 3);
        v[2] = ldcs3(T.v3 + 9 * t + 6);
    } else {
        v[0] = mk(__ldcs(T.v + 3 * t));
        v[1] = mk(__ldcs(T.v + 3 * t + 1));
        v[2] = mk(__ldcs(T.v + 3 * t + 2));
    }
}
__device__ __forceinline__ uint32_t tri_id(const TriSrc &T, long long t) {
    return T.ids ? (uint32_t)__ldg(T.ids + t) : (uint32_t)(T.id_base + (int32_t)t);
}

// -------------------------------------------------------- A2 range (delta_min) --
// Closest distance from the origin (0) to the closed triangle a0,a1,a2 (relative coords),
// Ericson-style: plane distance when the projection is inside, else nearest edge.
__device__ __forceinline__ float seg_dist2(f3 a, f3 b) {
    f3 e = subf(b, a);
    float ee = dotf(e, e);
    float t = ee > 0.f ? fminf(fmaxf(__fdividef(-dotf(a, e), ee), 0.f), 1.f) : 0.f;   // ~2 ulp: 2nd-order in dist
    f3 p = {a.x + t * e.x, a.y + t * e.y, a.z + t * e.z};
    return dotf(p, p);
}
__device__ float tri_dist(const f3 a[3]) {
    f3 N = crossf(subf(a[1], a[0]), subf(a[2], a[0]));
    float w0 = dotf(crossf(a[0], a[1]), N), w1 = dotf(crossf(a[1], a[2]), N), w2 = dotf(crossf(a[2], a[0]), N);
    float nn = dotf(N, N);
    if (nn > 0.f && ((w0 >= 0.f && w1 >= 0.f && w2 >= 0.f) || (w0 <= 0.f && w1 <= 0.f && w2 <= 0.f)))
        return fabsf(dotf(N, a[0])) * rsqrtf(nn);
    float d2 = fminf(seg_dist2(a[0], a[1]), fminf(seg_dist2(a[1], a[2]), seg_dist2(a[2], a[0])));
    return sqrt_approx(d2);   // compared against D_max (1 + 1e-5): far above the 2^-22 error
}

// ------------------------------------------------------ A3/A4 angular bounds --
struct Rect {
    int c_from, c_to;   // channel range (inclusive)
    int r_lo, r_len;    // ray range start (mod chi) and length; r_len == chi -> full
    int pole_rows;      // 1 if the range touches pole channels (full-azimuth rows)
};

enum { CULL_KEEP = 0, CULL_RANGE = 1, CULL_CHANNEL = 2, CULL_AZIMUTH = 3, CULL_DEGENERATE = 4, CULL_AREA = 5 };

__device__ __forceinline__ int lower_bound_f(const float *t, int n, float x) {   // first j: t[j] >= x
    int lo = 0, hi = n;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (t[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}
__device__ __forceinline__ int upper_bound_f(const float *t, int n, float x) {   // first j: t[j] > x
    int lo = 0, hi = n;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (t[mid] <= x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// First channel j with sin_j >= x: LUT start (an under-estimate) + short linear advance over
// the sentinel-terminated table (sinT[gamma] = +inf), or a binary search without a LUT.
__device__ __forceinline__ int first_channel_ge(const float *sinT, int gamma, const unsigned char *lut, float x) {
    if (!lut) return lower_bound_f(sinT, gamma, x);
    int b = (int)((x + 1.f) * (0.5f * kLutBins));
    b = min(max(b, 0), kLutBins - 1);
    int j = lut[b];
    while (sinT[j] < x) ++j;
    return j;
}

// First channel j with sin_j > x (upper bound), same scheme.
__device__ __forceinline__ int first_channel_gt(const float *sinT, int gamma, const unsigned char *lut, float x) {
    if (!lut) return upper_bound_f(sinT, gamma, x);
    int b = (int)((x + 1.f) * (0.5f * kLutBins));
    b = min(max(b, 0), kLutBins - 1);
    int j = lut[b];
    while (sinT[j] <= x) ++j;
    return j;
}

// Does direction T lie on the great-circle arc from p to q (normal m = p x q)?  Tolerant
// (returns true when unsure) -- including an extreme that is not attained is conservative.
__device__ __forceinline__ bool on_arc(f3 p, f3 q, f3 m, f3 T) {
    float q1 = dotf(crossf(p, T), m), q2 = dotf(crossf(T, q), m);
    float tol = 1e-4f * sqrt_approx(dotf(p, p) * dotf(T, T)) * sqrt_approx(dotf(m, m));
    float tol2 = 1e-4f * sqrt_approx(dotf(q, q) * dotf(T, T)) * sqrt_approx(dotf(m, m));
    return q1 >= -tol && q2 >= -tol2;
}

// Conservative (channel, ray) rectangle of triangle v seen from emitter E.
// kLevel: every emitter's frame is level (EmDev.level for all; the host picks the instantiation)
template <bool kLevel = false>
__device__ int cull_pair(const f3 v[3], const EmDev &E, const float *sinTab, const unsigned char *lut, bool nocull,
                         Rect &R) {
    const f3 o = {E.o[0], E.o[1], E.o[2]};
    f3 a[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) a[k] = subf(v[k], o);
    {   // non-finite input (inf / NaN coordinates) -> degenerate: inf and NaN propagate through the
        // sum (inf - inf = NaN), so one test covers all nine values (finite sums cannot reach inf
        // below |coordinates| ~ 3.8e37)
        const float sum = ((a[0].x + a[0].y) + (a[0].z + a[1].x)) + ((a[1].y + a[1].z) + (a[2].x + a[2].y)) + a[2].z;
        if (!(fabsf(sum) < CUDART_INF_F)) return CULL_DEGENERATE;
    }
    if (nocull) {
        R.c_from = 0; R.c_to = E.gamma - 1; R.r_lo = 0; R.r_len = E.chi; R.pole_rows = 0;
        return CULL_KEEP;
    }
    // A2: Step 1.3 range cull (delta_min > D_max), exact per-ray t <= D_max is in the test.
    if (E.dmax_hi < CUDART_INF_F) {
        const float lim = E.dmax_hi * (1.f + 1e-5f);
        float m2 = fminf(dotf(a[0], a[0]), fminf(dotf(a[1], a[1]), dotf(a[2], a[2])));
        if (m2 > lim * lim && tri_dist(a) > lim) return CULL_RANGE;
    }
    // sensor coordinates x = A a  (x = (x_f, x_r, x_u))
    f3 x[3];
    float r2[3], inv[3], s[3];
    if (kLevel || E.level) {   // level frame: the zero / unit entries of A dropped (same values up to the sign of 0)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            x[k].x = E.A[0] * a[k].x + E.A[1] * a[k].y;
            x[k].y = E.A[3] * a[k].x + E.A[4] * a[k].y;
            x[k].z = a[k].z;
            r2[k] = x[k].x * x[k].x + x[k].y * x[k].y + x[k].z * x[k].z;
        }
    } else {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            x[k].x = E.A[0] * a[k].x + E.A[1] * a[k].y + E.A[2] * a[k].z;
            x[k].y = E.A[3] * a[k].x + E.A[4] * a[k].y + E.A[5] * a[k].z;
            x[k].z = E.A[6] * a[k].x + E.A[7] * a[k].y + E.A[8] * a[k].z;
            r2[k] = x[k].x * x[k].x + x[k].y * x[k].y + x[k].z * x[k].z;
        }
    }
    if (!(r2[0] > 0.f && r2[1] > 0.f && r2[2] > 0.f)) return CULL_DEGENERATE;   // o is a vertex: Vol = 0
    float xn[3];   // |x_k|
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        inv[k] = rsqrtf(r2[k]);
        s[k] = x[k].z * inv[k];
        xn[k] = r2[k] * inv[k];
    }
    float slo = fminf(s[0], fminf(s[1], s[2])), shi = fmaxf(s[0], fmaxf(s[1], s[2]));
    // Near the spin axis the azimuths (and the pole test below) need x_h = (x_f, x_r) accurate
    // relative to |x_h|.  In a general frame x_h carries absolute errors ~u|x| from the cancellation
    // of the a_z terms, so within ~1.8 deg of the axis the row is taken whole.  In a level frame x_h
    // is a 2-D rotation of (a_x, a_y) alone (errors <= 4.25u |x_h| per component, no cancellation):
    // azimuth error <= 6u + the 2e-6 of fast_atan2, inside kPadTheta, at any |x_h| > 0, so only a
    // vertex on the axis itself (|x_h| < 1e-5 |x|) forces the full row.
    bool near_axis = false;
    float h2[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        h2[k] = x[k].x * x[k].x + x[k].y * x[k].y;
        near_axis |= h2[k] < ((kLevel || E.level) ? kNearAxisLevel2 : kNearAxis2) * r2[k];
    }
    // Fast path (most survivors: far, small triangles).  In sensor coordinates every point of T is
    // within diam of each vertex, so with rlb = max|x_k| - diam > 2 diam every chord subtends <= q =
    // diam / rlb: edge interiors exceed the vertex elevations by <= q^2/8 and a pole inside T would
    // force every |s_k| >= cos q >= 1 - q^2/2 (the K2 argument, now in x-space).
    float e2m = 0.f;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const f3 ev = subf(x[(k + 1) % 3], x[k]);
        e2m = fmaxf(e2m, dotf(ev, ev));
    }
    const float diam = (e2m > 0.f ? e2m * rsqrtf(e2m) : 0.f) * (1.f + 1e-5f);
    const float rlb_x = fmaxf(xn[0], fmaxf(xn[1], xn[2])) - diam;
    bool fast = false;
    float q2f = 0.f;
    if (rlb_x > 2.f * diam && !near_axis) {
        const float q = __fdividef(diam, rlb_x);   // ~2 ulp: the 0.13 q^2 pad has 4 % slack over q^2/8
        q2f = q * q;
        fast = fmaxf(fabsf(s[0]), fmaxf(fabsf(s[1]), fabsf(s[2]))) < 1.f - 0.51f * q2f - 1e-5f;
    }
    bool pole = false;
    float pad_e = 0.f;
    bool longedge = false;
    if (fast) {
        pad_e = 0.13f * q2f;
    } else {
    // pole containment: does the spin axis pass through T?  (2-D winding in the x_f x_r plane)
    // Bound of the computed winding's error: general frames 9u |x_k||x_k1| (x_h errors ~u|x|);
    // level frames 16u |x_h,k||x_h,k1| (x_h errors <= 4.25u|x_h| each + 2u for the cross product
    // = 10.5u, margin 1.5x), so a near-axis triangle still gets a decided pole test.
    bool pos = false, neg = false;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const int k1 = (k + 1) % 3;
        float w = x[k].x * x[k1].y - x[k].y * x[k1].x;
        float eps = (kLevel || E.level) ? 16.f * kU * (sqrt_approx(h2[k]) * sqrt_approx(h2[k1]))
                                        : 9.f * kU * xn[k] * xn[k1];
        pos |= (w > eps);
        neg |= (w < -eps);
    }
    // The axis can only meet T if T's horizontal projection straddles it on both coordinates
    // (this rejects degenerate, e.g. radial vertical, projections whose windings all round to ~0).
    const float tolb = 17.f * kU * fmaxf(xn[0], fmaxf(xn[1], xn[2]));
    const bool straddle = fminf(x[0].x, fminf(x[1].x, x[2].x)) <= tolb && fmaxf(x[0].x, fmaxf(x[1].x, x[2].x)) >= -tolb &&
                          fminf(x[0].y, fminf(x[1].y, x[2].y)) <= tolb && fmaxf(x[0].y, fmaxf(x[1].y, x[2].y)) >= -tolb;
    pole = straddle && !(pos && neg);
    if (pole) {
        if (shi > 0.f) shi = 1.f;
        if (slo < 0.f) slo = -1.f;
    }
    // interior extremes of edges: small arcs -> L^2/8 pad, long arcs -> great-circle extreme
    f3 xh[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) xh[k] = scalef(x[k], inv[k]);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const int k1 = (k + 1) % 3;
        f3 dv = subf(xh[k], xh[k1]);
        float c2 = dotf(dv, dv);
        if (c2 <= kChordSmall2) {
            pad_e = fmaxf(pad_e, 0.31f * c2);
        } else {
            longedge = true;
            f3 m = crossf(x[k], x[k1]);
            float mh2 = m.x * m.x + m.y * m.y;
            float mm = mh2 + m.z * m.z;
            if (!(mm > 0.f)) { shi = fmaxf(shi, 1.f); slo = fminf(slo, -1.f); continue; }
            float S = sqrt_approx(__fdividef(mh2, mm));   // ~1e-7 rel., inside the long-edge pad 1e-5
            f3 T = {-m.z * m.x, -m.z * m.y, mh2};   // top of the great circle (u - (u.m)m) * mm
            if (on_arc(x[k], x[k1], m, T)) shi = fmaxf(shi, S);
            f3 Tb = {-T.x, -T.y, -T.z};
            if (on_arc(x[k], x[k1], m, Tb)) slo = fminf(slo, -S);
        }
    }
    }   // !fast
    const float pad = kPadS + pad_e + (longedge ? 1e-5f : 0.f);
    R.c_from = first_channel_ge(sinTab, E.gamma, lut, slo - pad);
    R.c_to = min(first_channel_gt(sinTab, E.gamma, lut, shi + pad), E.gamma) - 1;
    if (R.c_from > R.c_to) return CULL_CHANNEL;
    // A4: azimuth arc -> ray index range
    const bool full = pole || near_axis;
    if (full) {
        R.r_lo = 0; R.r_len = E.chi; R.pole_rows = 0;
        return CULL_KEEP;
    }
    float start, len;
    bool arc_done = false;
    if (fast) {   // arc from the centroid azimuth and the vertices' small angular offsets
        const float cx = x[0].x + x[1].x + x[2].x, cy = x[0].y + x[1].y + x[2].y;
        float zmin = 0.f, zmax = 0.f;
        bool ok = true;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const float cr = cx * x[k].y - cy * x[k].x, dt = cx * x[k].x + cy * x[k].y;
            ok = ok && dt > 0.f && fabsf(cr) < dt;
            const float z = __fdividef(cr, dt);
            zmin = k ? fminf(zmin, z) : z;
            zmax = k ? fmaxf(zmax, z) : z;
        }
        // atan (and its polynomial, increasing on [-1, 1]) is monotone: the extremes of the three offsets
        // are the offsets of the extreme tangents -- two evaluations instead of three, same values
        const float dmin = poly_atan(zmin), dmax = poly_atan(zmax);
        if (ok) {
            start = fast_atan2(cy, cx) + dmin;
            len = dmax - dmin;
            arc_done = true;
        }
    }
    if (!arc_done) {
    float th[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) th[k] = fast_atan2(x[k].y, x[k].x);
    // sort 3 angles
    float t0 = fminf(th[0], fminf(th[1], th[2]));
    float t2 = fmaxf(th[0], fmaxf(th[1], th[2]));
    float t1 = th[0] + th[1] + th[2] - t0 - t2;
    t1 = fminf(fmaxf(t1, t0), t2);
    const float TWO_PI = 6.283185307179586f;
    float g01 = t1 - t0, g12 = t2 - t1, g20 = t0 + TWO_PI - t2;
    if (g20 >= g01 && g20 >= g12) { start = t0; len = t2 - t0; }
    else if (g01 >= g12) { start = t1; len = (t0 + TWO_PI) - t1; }
    else { start = t2; len = (t1 + TWO_PI) - t2; }
    }   // !arc_done
    if (len > 3.1f) {   // arc near pi with the axis outside T only by rounding: be safe
        R.r_lo = 0; R.r_len = E.chi; R.pole_rows = 0;
        return CULL_KEEP;
    }
    // perturbed azimuths (noise model): |theta*_i - theta_i| < dtheta -> one more ray each side
    const float padth = kPadTheta + (E.noisy ? E.dtheta : 0.f);
    float xlo = (start - padth - E.theta0) * E.inv_dtheta;
    float xhi = (start + len + padth - E.theta0) * E.inv_dtheta;
    int ilo = (int)ceilf(xlo), ihi = (int)floorf(xhi);
    if (E.hfov == 360) {
        int n = ihi - ilo + 1;
        if (n <= 0) return CULL_AZIMUTH;
        if (n >= E.chi) { R.r_lo = 0; R.r_len = E.chi; }
        else {   // ilo is within ~[-1, chi + 1]: wrap without an integer division
            int r = ilo;
            while (r < 0) r += E.chi;
            while (r >= E.chi) r -= E.chi;
            R.r_lo = r;
            R.r_len = n;
        }
    } else {
        // 180 deg: valid indices [0, chi-1]; the arc may also appear one period (2 chi) lower.
        int lo = INT_MAX, hi = INT_MIN;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            int a0 = ilo - c * 2 * E.chi, a1 = ihi - c * 2 * E.chi;
            a0 = max(a0, 0);
            a1 = min(a1, E.chi - 1);
            if (a0 <= a1) { lo = min(lo, a0); hi = max(hi, a1); }
        }
        if (lo > hi) return CULL_AZIMUTH;
        R.r_lo = lo; R.r_len = hi - lo + 1;
    }
    R.pole_rows = (R.r_len < E.chi) && (R.c_from < E.pole_lo || R.c_to > E.gamma - 1 - E.pole_hi);
    return CULL_KEEP;
}

// number of candidate (channel, ray) items of a rectangle (pole rows take all chi rays)
__device__ __forceinline__ long long rect_items(const Rect &R, const EmDev &E) {
    long long rows = R.c_to - R.c_from + 1;
    if (!R.pole_rows) return rows * R.r_len;
    int plo = max(0, min(R.c_to, E.pole_lo - 1) - R.c_from + 1);
    int phi = max(0, R.c_to - max(R.c_from, E.gamma - E.pole_hi) + 1);
    return (long long)(plo + phi) * E.chi + (rows - plo - phi) * R.r_len;
}

// K2 phase A: cheap conservative elevation pre-test of one (triangle, emitter) pair.
// Bounds: every point of T is within emax (= T's diameter) of each vertex,
// so |p - o| >= r_lb = max_k |a_k| - emax; the angle L subtended by any chord of T is <= q =
// emax / r_lb; the elevation excess of an edge interior over its endpoints is <= L^2/8 and a pole
// inside T forces every |s_k| >= cos L >= 1 - L^2/2.  Returns CULL_KEEP (-> K2b) or the cull.
__device__ __forceinline__ int quick_cull(const f3 v[3], float emax, const EmLite &L, const float *sinT,
                                          const unsigned char *lut) {
    const f3 o = {L.o[0], L.o[1], L.o[2]};
    float s[3], r[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const f3 a = {v[k].x - o.x, v[k].y - o.y, v[k].z - o.z};
        const float w2 = a.x * a.x + a.y * a.y + a.z * a.z;
        const float xu = L.Au[0] * a.x + L.Au[1] * a.y + L.Au[2] * a.z;
        const float iw = rsqrtf(w2);
        r[k] = w2 * iw;   // |a_k| (world)
        if (L.ortho) {
            s[k] = xu * iw;
        } else {
            const float x2 = L.G[0] * a.x * a.x + L.G[1] * a.y * a.y + L.G[2] * a.z * a.z +
                             2.f * (L.G[3] * a.x * a.y + L.G[4] * a.x * a.z + L.G[5] * a.y * a.z);
            s[k] = xu * rsqrtf(x2);
        }
    }
    const float rmax = fmaxf(r[0], fmaxf(r[1], r[2]));
    // branch-free: every pair evaluates the whole test (early returns only cost reconvergence)
    const float rlb = rmax - emax;
    const bool range = rlb > L.lim;
    const bool near = !(rlb > 2.f * emax);   // near (or degenerate / non-finite): exact path in K2b
    const float q = __fdividef(emax, rlb);   // garbage when rlb <= 0, but then near = true
    const float q2 = q * q;
    const float smax = fmaxf(fabsf(s[0]), fmaxf(fabsf(s[1]), fabsf(s[2])));
    const bool pole = smax >= 1.f - 0.51f * q2 - 1e-5f;   // a pole may lie inside T
    const float pad = L.pad0 + 0.13f * q2;
    const float lo = fminf(s[0], fminf(s[1], s[2])) - pad;
    const float hi = fmaxf(s[0], fmaxf(s[1], s[2])) + pad;
    float vj;   // sin of the first channel >= lo
    if (lut) {
        int b = (int)((lo + 1.f) * (0.5f * kLutBins));
        b = min(max(b, 0), kLutBins - 1);
        int j = lut[b];
        const float v0 = sinT[j], v1 = sinT[j + 1];   // two +inf sentinels: j + 1 <= gamma + 1
        vj = v0 >= lo ? v0 : v1;
        if (v1 < lo) {   // rare: > 2 channels in one bin (near the poles)
            j += 2;
            while (sinT[j] < lo) ++j;
            vj = sinT[j];
        }
    } else {
        vj = sinT[lower_bound_f(sinT, L.gamma, lo)];
    }
    const bool keep = near || pole || vj <= hi;
    return range ? CULL_RANGE : (keep ? CULL_KEEP : CULL_CHANNEL);
}

// ------------------------------------------------ A7 per-channel ray range --
// Late-pass Steps 1-2 made exact: the points of T whose elevation sine lies in
// the band [s_lo, s_hi] (the channel's rays, widened by the fp32 pad) form a region whose azimuth
// extremes are boundary points: crossings of T's edges with the two bounding cones (per-edge
// quadratic; plane case P:518-528 when s = 0) and vertices inside the band.
// Each cone meets a ray from the apex at most once, so with no pole in T the region's azimuths
// form one interval between those extremes, measured along T's arc (SURVEY 8(a) A7 rules).
// Returns the number of boundary points; dmin/dmax are their azimuths relative to th_ref.
__device__ __forceinline__ void a7_add(double px, double py, float th_ref, int &cnt, float &dmin, float &dmax) {
    float d = fast_atan2((float)py, (float)px) - th_ref;
    if (d >= 3.14159265f) d -= 6.28318531f;
    if (d < -3.14159265f) d += 6.28318531f;
    dmin = fminf(dmin, d);
    dmax = fmaxf(dmax, d);
    ++cnt;
}

// sk[k]: the vertices' elevation sines x_k.z / |x_k| (row-independent: computed once per pair by the caller)
__device__ __noinline__ int refine_row(const d3 x[3], const double sk[3], double s_lo, double s_hi, float th_ref,
                                       float &dmin, float &dmax) {
    int cnt = 0;
    dmin = CUDART_INF_F;
    dmax = -CUDART_INF_F;
#pragma unroll
    for (int k = 0; k < 3; ++k)
        if (sk[k] >= s_lo && sk[k] <= s_hi) a7_add(x[k].x, x[k].y, th_ref, cnt, dmin, dmax);
    for (int c = 0; c < 2; ++c) {
        const double sc = c ? s_hi : s_lo;
        const double s2 = sc * sc;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const d3 p = x[k];
            const d3 q = x[(k + 1) % 3];
            const d3 e = subd(q, p);
            const double a2 = e.z * e.z - s2 * dotd(e, e);
            const double a1 = 2.0 * (e.z * p.z - s2 * dotd(p, e));
            const double a0 = p.z * p.z - s2 * dotd(p, p);
            double lam[2];
            int nl = 0;
            const double scale = fabs(a2) + fabs(a1) + fabs(a0);
            if (!(scale > 0.0)) {   // the whole edge lies on the cone
                lam[nl++] = 0.0;
                lam[nl++] = 1.0;
            } else if (fabs(a2) <= 1e-14 * scale) {   // linear
                if (fabs(a1) > 1e-300) lam[nl++] = -a0 / a1;
            } else {
                double disc = a1 * a1 - 4.0 * a2 * a0;
                if (disc < 0.0 && disc > -1e-12 * a1 * a1) disc = 0.0;   // tangency within rounding
                if (disc >= 0.0) {
                    const double sq = sqrt(disc);
                    const double qq = -0.5 * (a1 + (a1 >= 0.0 ? sq : -sq));
                    if (qq != 0.0) {   // roots qq / a2 and a0 / qq through one division (a few ulp)
                        const double inv = 1.0 / (a2 * qq);
                        lam[nl++] = qq * qq * inv;
                        lam[nl++] = a0 * a2 * inv;
                    } else {
                        lam[nl++] = -a1 / (2.0 * a2);
                    }
                }
            }
            for (int m = 0; m < nl; ++m) {
                const double l = lam[m];
                if (!(l >= -1e-9 && l <= 1.0 + 1e-9)) continue;
                const double px = p.x + l * e.x, py = p.y + l * e.y, pz = p.z + l * e.z;
                if (sc != 0.0 && pz * sc < -1e-12 * (px * px + py * py + pz * pz)) continue;   // mirror nappe
                a7_add(px, py, th_ref, cnt, dmin, dmax);
            }
        }
    }
    return cnt;
}

// Two emitters at once with packed fp32x2 arithmetic (sm_100 FADD2/FMUL2/FFMA2: two fp32 lanes
// per FMA-pipe issue).  Same test, same bounds as quick_cull; used when both frames are orthonormal.
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

__device__ __forceinline__ int quick_tail(const float s[3], float rmax, float emax, const EmLite &L, const float *sinT,
                                          const unsigned char *lut) {
    const float rlb = rmax - emax;
    const bool range = rlb > L.lim;
    const bool near = !(rlb > 2.f * emax);
    const float q = __fdividef(emax, rlb);
    const float q2 = q * q;
    const float smax = fmaxf(fabsf(s[0]), fmaxf(fabsf(s[1]), fabsf(s[2])));
    const bool pole = smax >= 1.f - 0.51f * q2 - 1e-5f;
    const float pad = L.pad0 + 0.13f * q2;
    const float lo = fminf(s[0], fminf(s[1], s[2])) - pad;
    const float hi = fmaxf(s[0], fmaxf(s[1], s[2])) + pad;
    float vj;
    if (lut) {
        int b = (int)((lo + 1.f) * (0.5f * kLutBins));
        b = min(max(b, 0), kLutBins - 1);
        int j = lut[b];
        const float v0 = sinT[j], v1 = sinT[j + 1];
        vj = v0 >= lo ? v0 : v1;
        if (v1 < lo) {
            j += 2;
            while (sinT[j] < lo) ++j;
            vj = sinT[j];
        }
    } else {
        vj = sinT[lower_bound_f(sinT, L.gamma, lo)];
    }
    const bool keep = near || pole || vj <= hi;
    return range ? CULL_RANGE : (keep ? CULL_KEEP : CULL_CHANNEL);
}

#ifndef K2_TAIL_SEL
#define K2_TAIL_SEL 1   // K2 packed path: mask bits by selects (measured: C4 K2 0.455 -> 0.437 ms; NE = 4 0.286 -> 0.280)
#endif
#ifndef K2_FOLD_NEAR
#define K2_FOLD_NEAR 1   // K2: the near test folded into the pole bound (measured: C4 K2 0.461 -> 0.457 ms, K2 survivors
                         // +0.07 %, exact survivors and hits unchanged)
#endif
#ifndef K2_BIN_U32
#define K2_BIN_U32 1   // LUT bin by a float-to-unsigned conversion (saturating) instead of a clamp (measured: C4 K2
                       // 0.468 -> 0.461 ms; sin tables at a fixed stride for compile-time offsets on top: no gain)
#endif
#ifndef K2_TAIL_FMA
#define K2_TAIL_FMA 1   // K2 pre-test tail: range and pole bounds as single FMAs, LUT bin clamped in float
                        // (measured: C4 K2 0.482 -> 0.467 ms, same survivors; 0 = the two-step forms)
#endif
// LUT bin of lo (sin units; lo < 1 - 4e-6 since lo = min s - pad, s <= 1 + 2u, pad >= kPadS).
#ifndef K2_FADD_BIN
#define K2_FADD_BIN 0
#endif
__device__ __forceinline__ int lut_bin(float lo) {
#if K2_FADD_BIN
    // floor((lo' + 1) * 1024) or one less, lo' = max(lo, -1), without F2I (an XU-pipe op) or integer clamps:
    // y - 1/2 = lo' * 1024 + 1023.5 (one rounding, <= 2^-14), then + 1.5 * 2^23 rounds it to an integer (ties to
    // even).  The result is in [0, 2047]; it exceeds floor(y) only when y lies within 2^-14 (6e-8 in sin units)
    // below an integer, i.e. inside the LUT's 1e-6 under-estimate margin; one less only starts the scan earlier.
    return __float_as_int(__fadd_rn(__fmaf_rn(fmaxf(lo, -1.f), 0.5f * kLutBins, 0.5f * kLutBins - 0.5f), 12582912.f)) -
           0x4B400000;
#else
    // one rounding (<= 2.4e-7 in sin units) against the LUT's 1e-6 under-estimate margin
    return min(max(__float2int_rz(__fmaf_rn(lo, 0.5f * kLutBins, 0.5f * kLutBins)), 0), kLutBins - 1);
#endif
}

// Fixed-kernel variants (k_cull_fixed, NE <= 8; LUT always present).  Same bounds as quick_tail;
// differences: (i) no scan past the second LUT channel -- when a bin holds more channels below lo
// the pair is kept (v1 < lo <= hi), which is conservative since K2b/cull_pair recomputes the exact
// channel range; (ii) the result is two bits (1 = keep, 2 = range-culled) instead of a code.
__device__ __forceinline__ unsigned quick_tail_lut(const float s[3], float miw, float emax, const EmLite &L,
                                                   const float *sinT, const unsigned char *lut) {
    // x = emax / max_k |a_k| (miw = min_k 1/|a_k| from the rsqrt already taken).  rlb = max|a_k| -
    // emax > 2 emax  <=>  x < 1/3 (0.33: margin for the rsqrt error); then q = x / (1 - x) gives
    // q^2 <= 2.25 x^2, so the pads of quick_cull become 0.13 q^2 <= 0.2925 x^2 and the pole bound
    // 0.51 q^2 <= 1.1475 x^2 (x^2 ~ 1e-6 for typical triangles: no measurable loss of culling).
    // Range: rlb > lim  <=>  max|a_k| > lim + emax  <=>  miw (lim + emax) < 1.
    const float x = emax * miw;
    const float x2 = x * x;
#if K2_TAIL_FMA
    // range: miw (lim + emax) = miw lim + x, one FMA; pole bound (1 - 1e-5) - 1.1475 x^2, one FMA (both within
    // an ulp of the two-step forms, far inside the 1e-5 slacks of lim and of the pole bound)
    const bool range = __fmaf_rn(miw, L.lim, x) < 1.f;
    const float smax = fmaxf(fabsf(s[0]), fmaxf(fabsf(s[1]), fabsf(s[2])));
#if K2_FOLD_NEAR
    // near (x >= 0.33) folded into the pole test: with 9.2 x^2 instead of 1.1475 x^2 the bound is <= 0 <= smax
    // for every x >= 0.33 (9.2 * 0.1089 > 0.99999), and lower (more conservative) below it
    const bool near = false;
    const bool pole = smax >= __fmaf_rn(x2, -9.2f, 0.99999f);
#else
    const bool near = !(x < 0.33f);
    const bool pole = smax >= __fmaf_rn(x2, -1.1475f, 0.99999f);
#endif
    const float pad = L.pad0 + 0.2925f * x2;
    const float lo = fminf(s[0], fminf(s[1], s[2])) - pad;
    const float hi = fmaxf(s[0], fmaxf(s[1], s[2])) + pad;
    // lo >= -1 after one FMNMX; lo < 1 - 3e-6 (s <= 1 + dev + 2u, pad >= kPadS + 4 dev): no upper clamp
#if K2_BIN_U32   // the float-to-unsigned conversion saturates negatives (and NaN) to 0: no clamp at all
    const int b = (int)__float2uint_rz(__fmaf_rn(lo, 0.5f * kLutBins, 0.5f * kLutBins));
#else
    const int b = __float2int_rz(__fmaf_rn(fmaxf(lo, -1.f), 0.5f * kLutBins, 0.5f * kLutBins));
#endif
#else
    const bool range = miw * (L.lim + emax) < 1.f;
    const bool near = !(x < 0.33f);
    const float smax = fmaxf(fabsf(s[0]), fmaxf(fabsf(s[1]), fabsf(s[2])));
    const bool pole = smax >= 1.f - 1.1475f * x2 - 1e-5f;
    const float pad = L.pad0 + 0.2925f * x2;
    const float lo = fminf(s[0], fminf(s[1], s[2])) - pad;
    const float hi = fmaxf(s[0], fmaxf(s[1], s[2])) + pad;
    const int b = lut_bin(lo);
#endif
    const float *sj = sinT + lut[b];
    const float v0 = sj[0], v1 = sj[1];   // two +inf sentinels: j + 1 <= gamma + 1
    const float vj = v0 >= lo ? v0 : v1;
    const bool keep = near || pole || vj <= hi;
    return range ? 2u : (keep ? 1u : 0u);
}

// scalar pre-test (any frame) with the fixed-kernel LUT tail; returns 1 = keep, 2 = range-culled.
// kLevel: the frame's up row is exactly (0, 0, 1), so x_u = a_z (bit for bit what the dot gives).
template <bool kLevel = false>
__device__ __forceinline__ unsigned quick_cull_lut(const f3 v[3], float emax, const EmLite &L, const float *sinT,
                                                   const unsigned char *lut) {
    float s[3], iw[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const f3 a = {v[k].x - L.o[0], v[k].y - L.o[1], v[k].z - L.o[2]};
        const float w2 = a.x * a.x + a.y * a.y + a.z * a.z;
        const float xu = kLevel ? a.z : L.Au[0] * a.x + L.Au[1] * a.y + L.Au[2] * a.z;
        iw[k] = rsqrtf(w2);
        if (L.ortho) {
            s[k] = xu * iw[k];
        } else {
            const float x2 = L.G[0] * a.x * a.x + L.G[1] * a.y * a.y + L.G[2] * a.z * a.z +
                             2.f * (L.G[3] * a.x * a.y + L.G[4] * a.x * a.z + L.G[5] * a.y * a.z);
            s[k] = xu * rsqrtf(x2);
        }
    }
    return quick_tail_lut(s, fminf(iw[0], fminf(iw[1], iw[2])), emax, L, sinT, lut);
}

// Predicate forms of quick_tail_lut / quick_cull_lut / quick_pair_lut (same tests, same bounds; K2_PRED): keep
// and range as booleans that k2_tri ORs into its masks with compile-time shifts (no 2-bit code packing), and
// the LUT bin clamped in float (lo >= -1 after one FMNMX; lo <= max s - pad < 1 - 2^-11 needs no upper clamp:
// s <= 1 + 2u and pad >= 4e-6) instead of two integer clamps.
__device__ __forceinline__ void quick_tail_pred(const float s[3], float miw, float emax, const EmLite &L,
                                                const float *sinT, const unsigned char *lut, bool &keep, bool &range) {
    const float x = emax * miw;
    const float x2 = x * x;
#if K2_TAIL_FMA
    range = __fmaf_rn(miw, L.lim, x) < 1.f;
    const float smax = fmaxf(fabsf(s[0]), fmaxf(fabsf(s[1]), fabsf(s[2])));
#if K2_FOLD_NEAR
    const bool near = false;
    const bool pole = smax >= __fmaf_rn(x2, -9.2f, 0.99999f);
#else
    const bool near = !(x < 0.33f);
    const bool pole = smax >= __fmaf_rn(x2, -1.1475f, 0.99999f);
#endif
#else
    range = miw * (L.lim + emax) < 1.f;
    const bool near = !(x < 0.33f);
    const float smax = fmaxf(fabsf(s[0]), fmaxf(fabsf(s[1]), fabsf(s[2])));
    const bool pole = smax >= 1.f - 1.1475f * x2 - 1e-5f;
#endif
    const float pad = L.pad0 + 0.2925f * x2;
    const float lo = fminf(s[0], fminf(s[1], s[2])) - pad;
    const float hi = fmaxf(s[0], fmaxf(s[1], s[2])) + pad;
#if K2_TAIL_FMA && K2_BIN_U32
    const int b = (int)__float2uint_rz(__fmaf_rn(lo, 0.5f * kLutBins, 0.5f * kLutBins));
#elif K2_TAIL_FMA
    const int b = __float2int_rz(__fmaf_rn(fmaxf(lo, -1.f), 0.5f * kLutBins, 0.5f * kLutBins));
#else
    const int b = lut_bin(lo);
#endif
    const float *sj = sinT + lut[b];
    const float v0 = sj[0], v1 = sj[1];
    const float vj = v0 >= lo ? v0 : v1;
    keep = !range && (near || pole || vj <= hi);
}

template <bool kLevel = false>
__device__ __forceinline__ void quick_cull_pred(const f3 v[3], float emax, const EmLite &L, const float *sinT,
                                                const unsigned char *lut, bool &keep, bool &range) {
    float s[3], iw[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const f3 a = {v[k].x - L.o[0], v[k].y - L.o[1], v[k].z - L.o[2]};
        const float w2 = a.x * a.x + a.y * a.y + a.z * a.z;
        const float xu = kLevel ? a.z : L.Au[0] * a.x + L.Au[1] * a.y + L.Au[2] * a.z;
        iw[k] = rsqrtf(w2);
        if (L.ortho) {
            s[k] = xu * iw[k];
        } else {
            const float x2 = L.G[0] * a.x * a.x + L.G[1] * a.y * a.y + L.G[2] * a.z * a.z +
                             2.f * (L.G[3] * a.x * a.y + L.G[4] * a.x * a.z + L.G[5] * a.y * a.z);
            s[k] = xu * rsqrtf(x2);
        }
    }
    quick_tail_pred(s, fminf(iw[0], fminf(iw[1], iw[2])), emax, L, sinT, lut, keep, range);
}

// interleaved constants of emitters (2p, 2p+1) for the packed path: one 64-bit constant load each
struct EmPair {
    float2 no[3];   // (-o_x), (-o_y), (-o_z)
    float2 u[3];    // Au_x, Au_y, Au_z
};

// two emitters at once; returns bits (keep0, keep1) | (range0, range1) << 2.  kLevel: both frames
// level (up row of M^-1 exactly (0, 0, 1), checked on the host), so x_u = a_z -- the same value
// the general dot product gives for that row, bit for bit.
template <bool kLevel = false>
__device__ __forceinline__ unsigned quick_pair_lut(const f3 v[3], float emax, const EmPair &PR, const EmLite &L0,
                                                   const EmLite &L1, const float *sinT0, const float *sinT1,
                                                   const unsigned char *lut0, const unsigned char *lut1) {
    float s0[3], s1[3], m0 = CUDART_INF_F, m1 = CUDART_INF_F;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const float2 ax = __fadd2_rn(f2(v[k].x, v[k].x), PR.no[0]);
        const float2 ay = __fadd2_rn(f2(v[k].y, v[k].y), PR.no[1]);
        const float2 az = __fadd2_rn(f2(v[k].z, v[k].z), PR.no[2]);
        const float2 w2 = __ffma2_rn(az, az, __ffma2_rn(ay, ay, __fmul2_rn(ax, ax)));
        const float2 xu = kLevel ? az : __ffma2_rn(PR.u[2], az, __ffma2_rn(PR.u[1], ay, __fmul2_rn(PR.u[0], ax)));
        const float2 iw = f2(rsqrtf(w2.x), rsqrtf(w2.y));
        const float2 ss = __fmul2_rn(xu, iw);
        s0[k] = ss.x;
        s1[k] = ss.y;
        m0 = fminf(m0, iw.x);
        m1 = fminf(m1, iw.y);
    }
    const unsigned a = quick_tail_lut(s0, m0, emax, L0, sinT0, lut0);
    const unsigned b = quick_tail_lut(s1, m1, emax, L1, sinT1, lut1);
    return (a & 1u) | ((b & 1u) << 1) | ((a & 2u) << 1) | ((b & 2u) << 2);
}

#if K2_TAIL_SEL
// quick_pair_lut with the per-emitter results as ready-made mask bits (keep ? bit : 0, range ? bit : 0) instead of a
// 4-bit code that k2_tri unpacks: two selects per emitter, one OR per pair of emitters for each mask
template <bool kLevel = false>
__device__ __forceinline__ void quick_pair_sel(const f3 v[3], float emax, const EmPair &PR, const EmLite &L0,
                                               const EmLite &L1, const float *sinT0, const float *sinT1,
                                               const unsigned char *lut0, const unsigned char *lut1, unsigned bit0,
                                               unsigned &kb, unsigned &rb) {
    float s0[3], s1[3], m0 = CUDART_INF_F, m1 = CUDART_INF_F;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const float2 ax = __fadd2_rn(f2(v[k].x, v[k].x), PR.no[0]);
        const float2 ay = __fadd2_rn(f2(v[k].y, v[k].y), PR.no[1]);
        const float2 az = __fadd2_rn(f2(v[k].z, v[k].z), PR.no[2]);
        const float2 w2 = __ffma2_rn(az, az, __ffma2_rn(ay, ay, __fmul2_rn(ax, ax)));
        const float2 xu = kLevel ? az : __ffma2_rn(PR.u[2], az, __ffma2_rn(PR.u[1], ay, __fmul2_rn(PR.u[0], ax)));
        const float2 iw = f2(rsqrtf(w2.x), rsqrtf(w2.y));
        const float2 ss = __fmul2_rn(xu, iw);
        s0[k] = ss.x;
        s1[k] = ss.y;
        m0 = fminf(m0, iw.x);
        m1 = fminf(m1, iw.y);
    }
    const unsigned a = quick_tail_lut(s0, m0, emax, L0, sinT0, lut0);
    const unsigned b = quick_tail_lut(s1, m1, emax, L1, sinT1, lut1);
    kb |= (a == 1u ? bit0 : 0u) | (b == 1u ? bit0 << 1 : 0u);
    rb |= (a == 2u ? bit0 : 0u) | (b == 2u ? bit0 << 1 : 0u);
}
#endif

template <bool kLevel = false>
__device__ __forceinline__ void quick_pair_pred(const f3 v[3], float emax, const EmPair &PR, const EmLite &L0,
                                                const EmLite &L1, const float *sinT0, const float *sinT1,
                                                const unsigned char *lut0, const unsigned char *lut1, bool &k0, bool &r0,
                                                bool &k1, bool &r1) {
    float s0[3], s1[3], m0 = CUDART_INF_F, m1 = CUDART_INF_F;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const float2 ax = __fadd2_rn(f2(v[k].x, v[k].x), PR.no[0]);
        const float2 ay = __fadd2_rn(f2(v[k].y, v[k].y), PR.no[1]);
        const float2 az = __fadd2_rn(f2(v[k].z, v[k].z), PR.no[2]);
        const float2 w2 = __ffma2_rn(az, az, __ffma2_rn(ay, ay, __fmul2_rn(ax, ax)));
        const float2 xu = kLevel ? az : __ffma2_rn(PR.u[2], az, __ffma2_rn(PR.u[1], ay, __fmul2_rn(PR.u[0], ax)));
        const float2 iw = f2(rsqrtf(w2.x), rsqrtf(w2.y));
        const float2 ss = __fmul2_rn(xu, iw);
        s0[k] = ss.x;
        s1[k] = ss.y;
        m0 = fminf(m0, iw.x);
        m1 = fminf(m1, iw.y);
    }
    quick_tail_pred(s0, m0, emax, L0, sinT0, lut0, k0, r0);
    quick_tail_pred(s1, m1, emax, L1, sinT1, lut1, k1, r1);
}

__device__ __forceinline__ void quick_cull2(const f3 v[3], float emax, const EmLite &L0, const EmLite &L1,
                                            const float *sinT0, const float *sinT1, const unsigned char *lut0,
                                            const unsigned char *lut1, int &st0, int &st1) {
    const float2 nox = f2(-L0.o[0], -L1.o[0]), noy = f2(-L0.o[1], -L1.o[1]), noz = f2(-L0.o[2], -L1.o[2]);
    const float2 ux = f2(L0.Au[0], L1.Au[0]), uy = f2(L0.Au[1], L1.Au[1]), uz = f2(L0.Au[2], L1.Au[2]);
    float s0[3], s1[3], r0 = 0.f, r1 = 0.f;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const float2 ax = __fadd2_rn(f2(v[k].x, v[k].x), nox);
        const float2 ay = __fadd2_rn(f2(v[k].y, v[k].y), noy);
        const float2 az = __fadd2_rn(f2(v[k].z, v[k].z), noz);
        const float2 w2 = __ffma2_rn(az, az, __ffma2_rn(ay, ay, __fmul2_rn(ax, ax)));
        const float2 xu = __ffma2_rn(uz, az, __ffma2_rn(uy, ay, __fmul2_rn(ux, ax)));
        const float2 iw = f2(rsqrtf(w2.x), rsqrtf(w2.y));
        const float2 rr = __fmul2_rn(w2, iw), ss = __fmul2_rn(xu, iw);
        s0[k] = ss.x;
        s1[k] = ss.y;
        r0 = fmaxf(r0, rr.x);
        r1 = fmaxf(r1, rr.y);
    }
    st0 = quick_tail(s0, r0, emax, L0, sinT0, lut0);
    st1 = quick_tail(s1, r1, emax, L1, sinT1, lut1);
}

// --------------------------------------------------- A6 setup + certified test --
struct Setup {
    f3 n0, n1, n2;     // sigma_k * s * n_k: hit <=> all d.n_k >= 0
    float B0, B1, B2;  // certified error bounds of d.n_k
    f3 N;              // s * (e1 x e2): d.N > 0 for hits
    float habs;        // |N . a0|
    float TN;          // fp32 t certified iff d.N >= TN
};

// A6 setup of one (triangle, emitter) pair, computed once into the five values every kernel stores
// or reads (so K4, the split path and the fused kernel use bit-identical thresholds):
//   out[k] = (sigma_k s n_k, B_k) for the three canonical edges (hit <=> all d.n_k >= 0; B_k certified
//            bound of d.n_k), out[3] = (s N, |h|), out[4].x = TN (fp32 t certified iff d.N >= TN).
// The plane (N, h) is computed in fp64 from the exact fp64 edges and rounded: t = h / d.N is then
// certified to 4.5e-6 for all but |cos(view)| < ~0.05.  Computed plane
// first and one edge at a time (fewer live values: the fused kernel runs at the register cap).
// Returns false when the pair can never hit (Vol == 0: origin in the plane / degenerate triangle)
// or is rejected by the face mode.  Explicit _rn intrinsics: no contraction freedom.
template <typename Store>
__device__ __forceinline__ bool setup_core(const f3 v[3], f3 o, int faces, Store &&store) {
    const d3 V0 = tod(v[0]);
    const d3 E1 = subd(tod(v[1]), V0), E2 = subd(tod(v[2]), V0);
    const d3 N64 = crossd(E1, E2);
    const d3 A0 = subd(V0, tod(o));
    const double h64 = dotd(N64, A0);
    if (!(h64 > 0.0 || h64 < 0.0)) return false;
    const float s = h64 > 0.0 ? 1.f : -1.f;
    if ((faces == 1 && s < 0.f) || (faces == 2 && s > 0.f)) return false;
    const f3 N = {(float)N64.x, (float)N64.y, (float)N64.z};
    const float habs = (float)fabs(h64);
    // generous bound of the fp64 error of h64 (2^-48 relative to its L1 magnitudes)
    const float sE1 = __fadd_rn(__fadd_rn(fabsf((float)E1.x), fabsf((float)E1.y)), fabsf((float)E1.z));
    const float sE2 = __fadd_rn(__fadd_rn(fabsf((float)E2.x), fabsf((float)E2.y)), fabsf((float)E2.z));
    const float sN = __fadd_rn(__fadd_rn(fabsf(N.x), fabsf(N.y)), fabsf(N.z));
    const float l1 = __fadd_rn(__fmul_rn(sE1, sE2), sN);
    const float la = __fadd_rn(__fadd_rn(fabsf((float)A0.x), fabsf((float)A0.y)), fabsf((float)A0.z));
    const float err64 = __fmul_rn(__fmul_rn(3.64e-15f, l1), la);
    const bool sign_ok = habs > 2.f * err64;   // else every candidate goes to fp64 (B = inf)
    const float rh = __fadd_rn(1.01f * kU, __fmul_rn(__fdividef(err64, habs), 1.02f));
    const float nn = dotf(N, N);
    const float Bn = __fmul_rn(3.11f * kU, nn > 0.f ? __fmul_rn(nn, rsqrtf(nn)) : 0.f);
    // budget: kTRel = rel(d.N) + rh + 6u, where 6u covers the rounding of N and h and the approximate
    // division in test_fast (rcp.approx then multiply: <= 2 ulp = 4u)
    const float TN = (!sign_ok || !(rh < 2e-6f)) ? CUDART_INF_F
                                                 : __fmul_rn(__fdividef(Bn, __fsub_rn(kTRel - 6.f * kU, rh)), 1.0002f);
    const f3 SN = scalef(N, s);
    store(3, make_float4(SN.x, SN.y, SN.z, habs));
    store(4, make_float4(TN, 0.f, 0.f, 0.f));
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        f3 Pp = v[k], Qq = v[(k + 1) % 3];
        const bool sw = lexless(Qq, Pp);   // canonical direction: adjacent triangles share bits
        if (sw) { f3 t = Pp; Pp = Qq; Qq = t; }
        const f3 aP = subf(Pp, o), e = subf(Qq, Pp);
        const f3 n = scalef(crossf(aP, e), s * (sw ? -1.f : 1.f));
        const float pe = __fmul_rn(dotf(aP, aP), dotf(e, e));
        const float B = __fmul_rn(16.1f * kU, pe > 0.f ? __fmul_rn(pe, rsqrtf(pe)) : 0.f);   // 16u|a||e|
        store(k, make_float4(n.x, n.y, n.z, sign_ok ? B : CUDART_INF_F));
    }
    return true;
}

// The setup as a Setup struct (K4, split path, serial fallback).
__device__ __forceinline__ bool make_setup(const f3 v[3], f3 o, int faces, Setup &S, unsigned &setup64) {
    (void)setup64;
    return setup_core(v, o, faces, [&](int k, float4 q) {
        if (k < 3) {
            const f3 n = {q.x, q.y, q.z};
            if (k == 0) { S.n0 = n; S.B0 = q.w; }
            if (k == 1) { S.n1 = n; S.B1 = q.w; }
            if (k == 2) { S.n2 = n; S.B2 = q.w; }
        } else if (k == 3) {
            S.N = {q.x, q.y, q.z};
            S.habs = q.w;
        } else {
            S.TN = q.x;
        }
    });
}

// The setup written straight into a lane's slot column (fused kernel): slot[k * 32] for k < 4,
// slot[4 * 32] = (TN, id, tri, emitter).
__device__ __forceinline__ bool setup_to_slot(const f3 v[3], f3 o, int faces, float4 *slot, uint32_t id, int tri,
                                              int em) {
    return setup_core(v, o, faces, [&](int k, float4 q) {
        if (k == 4) q = make_float4(q.x, __uint_as_float(id), __int_as_float(tri), __int_as_float(em));
        slot[k * 32] = q;
    });
}

__device__ __forceinline__ float rcp_approx(float x) {   // rcp.approx.ftz.f32 (MUFU.RCP, <= 1 ulp)
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// 0 = certified miss, 1 = certified hit (t set), 2 = uncertain -> fp64
__device__ __forceinline__ int test_fast(float4 d4, const Setup &S, float dmax_lo, float dmax_hi, float &t) {
    const f3 d = {d4.x, d4.y, d4.z};
    const float F0 = dotf(d, S.n0), F1 = dotf(d, S.n1), F2 = dotf(d, S.n2);
    if (F0 < -S.B0 || F1 < -S.B1 || F2 < -S.B2) return 0;
    if (!(F0 > S.B0 && F1 > S.B1 && F2 > S.B2)) return 2;
    const float dN = dotf(d, S.N);
    if (!(dN >= S.TN && dN <= 1e30f)) return 2;   // (upper guard: the reciprocal must not flush to 0)
    t = __fmul_rn(S.habs, rcp_approx(dN));        // <= 2 ulp, inside TN's budget
    if (t <= dmax_lo) return 1;
    if (t > dmax_hi) return 0;
    return 2;
}

// fp64 decision (canonical edges, closed triangle, 0 < t <= dmax).  Returns the fp32-rounded t
// of a hit, -1 otherwise.  All arguments by value and no out-parameter: the call must not force
// the caller's ray / vertices / t through local memory (it sits inside the hot item loops).
template <bool kInline>
__device__ __forceinline__ float test_exact_body(f3 v0, f3 v1, f3 v2, f3 o, float4 d4, double dmax, int faces) {
    const f3 v[3] = {v0, v1, v2};
    const d3 d = {(double)d4.x, (double)d4.y, (double)d4.z};
    const d3 O = tod(o);
    double F[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        f3 P = v[k], Q = v[(k + 1) % 3];
        const bool sw = lexless(Q, P);
        if (sw) { f3 t = P; P = Q; Q = t; }
        d3 aP = subd(tod(P), O), e = subd(tod(Q), tod(P));
        double f = dotd(d, crossd(aP, e));
        F[k] = sw ? -f : f;
    }
    d3 V0 = tod(v[0]);
    d3 N = crossd(subd(tod(v[1]), V0), subd(tod(v[2]), V0));
    double h = dotd(N, subd(V0, O));
    if (!(h > 0.0 || h < 0.0)) return -1.f;
    if ((faces == 1 && h < 0.0) || (faces == 2 && h > 0.0)) return -1.f;
    if (h < 0.0) { F[0] = -F[0]; F[1] = -F[1]; F[2] = -F[2]; }
    if (F[0] < 0.0 || F[1] < 0.0 || F[2] < 0.0) return -1.f;
    double dN = dotd(d, N);
    if (!(dN > 0.0 || dN < 0.0)) return -1.f;
    double t = h / dN;
    if (!(t > 0.0 && t <= dmax)) return -1.f;
    return (float)t;   // >= +0: a hit (the caller tests r >= 0)
}
__device__ __noinline__ float test_exact(f3 v0, f3 v1, f3 v2, f3 o, float4 d4, double dmax, int faces) {
    return test_exact_body<false>(v0, v1, v2, o, d4, dmax, faces);
}
// 1 = hit (t set), 0 = miss: adapter for the call sites.  kInline expands the fp64 test at the
// call site (no CALL: nothing live across an ABI call has to be spilled around it).
template <bool kInline = false>
__device__ __forceinline__ int test_exact_r(const f3 v[3], f3 o, float4 d4, double dmax, int faces, float &t) {
    const float r = kInline ? test_exact_body<true>(v[0], v[1], v[2], o, d4, dmax, faces)
                            : test_exact(v[0], v[1], v[2], o, d4, dmax, faces);
    if (r >= 0.f) { t = r; return 1; }
    return 0;
}

// Closest-hit update on the packed key (fp32 t bits << 32 | id).  t > 0 so the raw bits
// order like the value (PAPER.md:2343-2356 f_sort, widened with the id as tie-break).
// mc != NULL (NEXT-f3 fused NVLS merge): the key goes to the multicast address of the ranks' hit
// buffers, and the NVSwitch applies the min to every rank's copy (multimem.red: no separate
// all-reduce).  Otherwise a local RED.MIN.
#ifdef GRCA_CHECK
__device__ long long g_check_n_rays;   // rays of the current cast (set by the host before each cast)
#endif
__device__ __forceinline__ void record_hit(unsigned long long *hits, unsigned long long *mc, unsigned *allhits, int g,
                                           float t, uint32_t id) {
    const unsigned long long key = ((unsigned long long)__float_as_uint(t) << 32) | id;
#ifdef GRCA_CHECK
    g = (int)chk_idx(g, g_check_n_rays, CHK_RAY);
#endif
    if (allhits) atomicAdd(allhits + g, 1u);
    if (mc)
        asm volatile("multimem.red.relaxed.sys.global.min.u64 [%0], %1;" ::"l"(mc + g), "l"(key) : "memory");
    else
        atomicMin(hits + g, key);   // result unused -> RED.MIN: fire-and-forget, no L2 round trip
}

}  // namespace grca
