/*
 * oracle/grca_oracle.c -- brute-force CPU oracle for the GRCA hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant with the CUDA library in
 * paper_2605_10457_b200/ and it does not include any of its headers.
 *
 * What it computes is the plain definition of the result, not the paper's
 * (approximate) culling method:
 *
 *   "for each ray the simulation must find the closest triangle it
 *    intersects and its distance"
 *   Total RTIC = sum_n gamma_n * chi_n * tau        (Eq. 1)
 *
 * i.e. every ray is tested against every triangle (Eq. 1 realised).
 *
 *  O1  ray definition (Eq. ray_dir and the angular grid):
 *      dtheta = H / chi  (H = 2*pi for a 360 deg emitter, pi for 180 deg),
 *      theta_i = -floor(chi/2)*dtheta + i*dtheta
 *      phi_j   = channel_elev_rad[j]   (sorted table)
 *      (noise model: a perturbed per-ray azimuth table theta*_i replaces the
 *       grid when given; per-channel perturbed elevations are simply the elevation table)
 *      d = RN32( cos(theta)cos(phi) f + sin(theta)cos(phi) r + sin(phi) u )
 *      evaluated in fp64 left to right, rounded componentwise to fp32.
 *      Global ray index g = O_n + j*chi_n + i
 *  O2  hit test: textbook fp64 Moller-Trumbore (ref [moller1997])
 *      on the fp32 inputs converted exactly to fp64; closed triangle
 *      (u >= 0, v >= 0, u+v <= 1), 0 < t <= D_max, two-sided unless a
 *      face mode is set (keep iff sign(d.N) matches).
 *  O3  result per ray: minimum t, ties -> smaller triangle id; miss -> (+inf, -1)
 *      ("rays with no intersection retain D = +inf").
 *
 * Everything is fp64; there is no blocking, no culling and no reordering.
 * Parallelism: std pthreads over disjoint ray ranges (each ray independent).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

typedef struct {
    float origin[3];
    float forward[3];
    float right[3];
    float up[3];
    const float *channel_elev_rad; /* gamma entries, radians */
    int32_t n_channels;            /* gamma_n */
    int32_t rays_per_channel;      /* chi_n   */
    int32_t hfov_deg;              /* 360 or 180 */
    float max_range;               /* <= 0 or +inf: no limit */
    const float *ray_azimuth_rad;  /* NULL: grid theta_i; else the pre-stored perturbed azimuths
                                      theta*_i of the noise model */
} oracle_emitter;

/* ---------------------------------------------------------------- O1 -- */

int64_t oracle_n_rays(const oracle_emitter *em, int32_t n_em)
{
    int64_t total = 0;
    for (int32_t n = 0; n < n_em; ++n)
        total += (int64_t)em[n].n_channels * (int64_t)em[n].rays_per_channel;
    return total;
}

/* Locate emitter n and (j, i) of global ray g.  Returns 0 on success. */
static int ray_locate(const oracle_emitter *em, int32_t n_em, int64_t g,
                      int32_t *n_out, int32_t *j_out, int32_t *i_out)
{
    int64_t base = 0; /* O_n = sum_{m<n} gamma_m chi_m */
    for (int32_t n = 0; n < n_em; ++n) {
        int64_t cnt = (int64_t)em[n].n_channels * em[n].rays_per_channel;
        if (g < base + cnt) {
            int64_t local = g - base;
            *n_out = n;
            *j_out = (int32_t)(local / em[n].rays_per_channel);
            *i_out = (int32_t)(local % em[n].rays_per_channel);
            return 0;
        }
        base += cnt;
    }
    return -1;
}

/* Eq. ray_dir at grid angles. */
static void ray_direction(const oracle_emitter *e, int32_t j, int32_t i,
                          double d64[3], float d32[3])
{
    const double H = (e->hfov_deg == 180) ? M_PI : 2.0 * M_PI;
    const double dtheta = H / (double)e->rays_per_channel;
    const double theta0 = -(double)(e->rays_per_channel / 2) * dtheta;
    const double theta = e->ray_azimuth_rad ? (double)e->ray_azimuth_rad[i] : theta0 + (double)i * dtheta;
    const double phi = (double)e->channel_elev_rad[j];
    const double ct = cos(theta), st = sin(theta);
    const double cp = cos(phi), sp = sin(phi);
    for (int c = 0; c < 3; ++c) {
        double v = ct * cp * (double)e->forward[c] + st * cp * (double)e->right[c] +
                   sp * (double)e->up[c];
        d32[c] = (float)v; /* RN32 */
        d64[c] = v;
    }
}

void oracle_ray_table(const oracle_emitter *em, int32_t n_em, float *out_xyz)
{
    int64_t g = 0;
    for (int32_t n = 0; n < n_em; ++n)
        for (int32_t j = 0; j < em[n].n_channels; ++j)
            for (int32_t i = 0; i < em[n].rays_per_channel; ++i, ++g) {
                double d64[3];
                ray_direction(&em[n], j, i, d64, &out_xyz[3 * g]);
            }
}

/* ---------------------------------------------------------------- O2 -- */

static void sub3(const double a[3], const double b[3], double r[3])
{
    r[0] = a[0] - b[0];
    r[1] = a[1] - b[1];
    r[2] = a[2] - b[2];
}
static void cross3(const double a[3], const double b[3], double r[3])
{
    r[0] = a[1] * b[2] - a[2] * b[1];
    r[1] = a[2] * b[0] - a[0] * b[2];
    r[2] = a[0] * b[1] - a[1] * b[0];
}
static double dot3(const double a[3], const double b[3])
{
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}

/*
 * Textbook Moller-Trumbore, fp64.
 * Returns 0 when det == 0 (ray parallel to the plane: no intersection),
 * else 1 with the ray parameter t and barycentrics (u, v) of the line hit.
 * Also returns d.N with N = e1 x e2 for the face modes.
 */
int oracle_mt(const double o[3], const double d[3], const double v0[3],
              const double v1[3], const double v2[3], double *t, double *u,
              double *v, double *dN)
{
    double e1[3], e2[3], p[3], s[3], q[3], N[3];
    sub3(v1, v0, e1);
    sub3(v2, v0, e2);
    cross3(d, e2, p);
    const double det = dot3(e1, p);
    cross3(e1, e2, N);
    if (dN) *dN = dot3(d, N);
    if (det == 0.0) return 0;
    const double inv = 1.0 / det;
    sub3(o, v0, s);
    *u = dot3(s, p) * inv;
    cross3(s, e1, q);
    *v = dot3(d, q) * inv;
    *t = dot3(e2, q) * inv;
    return 1;
}

/* faces: 0 two-sided, 1 keep d.N > 0, 2 keep d.N < 0 */
static int hit_accept(double t, double u, double v, double dN, double dmax,
                      int32_t faces)
{
    if (!(u >= 0.0 && v >= 0.0 && u + v <= 1.0)) return 0;
    if (!(t > 0.0 && t <= dmax)) return 0;
    if (faces == 1 && !(dN > 0.0)) return 0;
    if (faces == 2 && !(dN < 0.0)) return 0;
    return 1;
}

static double emitter_dmax(const oracle_emitter *e)
{
    double r = (double)e->max_range;
    if (!(r > 0.0) || isinf(r)) return INFINITY;
    return r;
}

/*
 * Single (ray, triangle) query used by the comparator: the fp64 t and
 * barycentric coordinates (u, v) of ray g against the triangle tri9
 * (v0, v1, v2 as 9 floats); *hit = accepted under O2.
 * Returns 0 if det == 0, 1 otherwise, -1 on a bad ray index.
 */
int oracle_ray_tri(const oracle_emitter *em, int32_t n_em, int64_t g,
                   const float *tri9, int32_t faces, double *t, double *u,
                   double *v, int32_t *hit)
{
    int32_t n, j, i;
    if (ray_locate(em, n_em, g, &n, &j, &i)) return -1;
    double d64[3], o[3], d[3], a[3], b[3], c[3], dN = 0.0;
    float d32[3];
    ray_direction(&em[n], j, i, d64, d32);
    for (int k = 0; k < 3; ++k) {
        d[k] = (double)d32[k];
        o[k] = (double)em[n].origin[k];
        a[k] = (double)tri9[k];
        b[k] = (double)tri9[3 + k];
        c[k] = (double)tri9[6 + k];
    }
    *hit = 0;
    if (!oracle_mt(o, d, a, b, c, t, u, v, &dN)) return 0;
    *hit = hit_accept(*t, *u, *v, dN, emitter_dmax(&em[n]), faces);
    return 1;
}

/* ---------------------------------------------------------------- O3 -- */

typedef struct {
    const oracle_emitter *em;
    int32_t n_em;
    const float *tri9;
    const int32_t *tri_ids;
    int64_t n_tri;
    int32_t faces;
    const int64_t *rays;
    int64_t n_rays;
    float *out_t;
    int32_t *out_id;
    double *out_t64;
    uint32_t *out_allhits;
    int64_t begin, end;
} cast_job;

static void *cast_worker(void *arg)
{
    cast_job *J = (cast_job *)arg;
    for (int64_t r = J->begin; r < J->end; ++r) {
        const int64_t g = J->rays ? J->rays[r] : r;
        int32_t n, j, i;
        double best_t = INFINITY;
        int32_t best_id = -1;
        uint32_t nhits = 0;
        if (ray_locate(J->em, J->n_em, g, &n, &j, &i) == 0) {
            const oracle_emitter *e = &J->em[n];
            double d64[3], o[3], d[3];
            float d32[3];
            ray_direction(e, j, i, d64, d32);
            for (int k = 0; k < 3; ++k) {
                d[k] = (double)d32[k]; /* the ray is the fp32 direction */
                o[k] = (double)e->origin[k];
            }
            const double dmax = emitter_dmax(e);
            for (int64_t q = 0; q < J->n_tri; ++q) {
                const float *T = &J->tri9[9 * q];
                double a[3], b[3], c[3], t, u, v, dN;
                for (int k = 0; k < 3; ++k) {
                    a[k] = (double)T[k];
                    b[k] = (double)T[3 + k];
                    c[k] = (double)T[6 + k];
                }
                if (!oracle_mt(o, d, a, b, c, &t, &u, &v, &dN)) continue;
                if (!hit_accept(t, u, v, dN, dmax, J->faces)) continue;
                ++nhits;
                const int32_t id = J->tri_ids ? J->tri_ids[q] : (int32_t)q;
                if (t < best_t || (t == best_t && id < best_id)) {
                    best_t = t;
                    best_id = id;
                }
            }
        }
        J->out_t[r] = (float)best_t; /* RN32(t); +inf on a miss */
        J->out_id[r] = best_id;
        if (J->out_t64) J->out_t64[r] = best_t;
        if (J->out_allhits) J->out_allhits[r] = nhits;
    }
    return NULL;
}

/*
 * Brute-force closest hit for rays[0..n_rays) (global indices; NULL -> all
 * rays 0..n_rays-1) against all n_tri triangles (tri9: 9 floats each).
 * tri_ids: global id per triangle (NULL -> position).  out_t64 / out_allhits
 * are optional.  n_threads <= 0 -> 1.  Returns 0.
 */
int oracle_cast(const oracle_emitter *em, int32_t n_em, const float *tri9,
                const int32_t *tri_ids, int64_t n_tri, int32_t faces,
                const int64_t *rays, int64_t n_rays, int32_t n_threads,
                float *out_t, int32_t *out_id, double *out_t64,
                uint32_t *out_allhits)
{
    if (n_threads <= 0) n_threads = 1;
    if (n_threads > 1024) n_threads = 1024;
    if ((int64_t)n_threads > n_rays) n_threads = n_rays > 0 ? (int32_t)n_rays : 1;
    cast_job *jobs = (cast_job *)calloc((size_t)n_threads, sizeof(cast_job));
    pthread_t *th = (pthread_t *)calloc((size_t)n_threads, sizeof(pthread_t));
    if (!jobs || !th) {
        free(jobs);
        free(th);
        return -1;
    }
    for (int32_t k = 0; k < n_threads; ++k) {
        cast_job *J = &jobs[k];
        J->em = em;
        J->n_em = n_em;
        J->tri9 = tri9;
        J->tri_ids = tri_ids;
        J->n_tri = n_tri;
        J->faces = faces;
        J->rays = rays;
        J->n_rays = n_rays;
        J->out_t = out_t;
        J->out_id = out_id;
        J->out_t64 = out_t64;
        J->out_allhits = out_allhits;
        J->begin = n_rays * k / n_threads;
        J->end = n_rays * (k + 1) / n_threads;
    }
    for (int32_t k = 1; k < n_threads; ++k)
        pthread_create(&th[k], NULL, cast_worker, &jobs[k]);
    cast_worker(&jobs[0]);
    for (int32_t k = 1; k < n_threads; ++k) pthread_join(th[k], NULL);
    free(jobs);
    free(th);
    return 0;
}

/*
 * Comparator helper (SURVEY 8(c) "excused": a disagreement is excused when the triangle involved has
 * fp64 barycentric margin min(u, v, 1-u-v) within eps of its boundary for the ray): the number of
 * triangles whose line hit by ray g has t > 0 (and t <= D_max) and |margin| <= eps -- the triangles on
 * whose edges an all-hit count may legitimately differ by one.  Same O1/O2 definitions as above.
 */
int64_t oracle_near_edge_count(const oracle_emitter *em, int32_t n_em, int64_t g, const float *tri9,
                               int64_t n_tri, double eps)
{
    int32_t n, j, i;
    if (ray_locate(em, n_em, g, &n, &j, &i)) return -1;
    double d64[3], o[3], d[3];
    float d32[3];
    ray_direction(&em[n], j, i, d64, d32);
    for (int k = 0; k < 3; ++k) {
        d[k] = (double)d32[k];
        o[k] = (double)em[n].origin[k];
    }
    const double dmax = emitter_dmax(&em[n]);
    int64_t cnt = 0;
    for (int64_t q = 0; q < n_tri; ++q) {
        const float *T = &tri9[9 * q];
        double a[3], b[3], c[3], t, u, v, dN;
        for (int k = 0; k < 3; ++k) {
            a[k] = (double)T[k];
            b[k] = (double)T[3 + k];
            c[k] = (double)T[6 + k];
        }
        if (!oracle_mt(o, d, a, b, c, &t, &u, &v, &dN)) continue;
        if (!(t > 0.0 && t <= dmax)) continue;
        double m = u < v ? u : v;
        if (1.0 - u - v < m) m = 1.0 - u - v;
        if (fabs(m) <= eps) ++cnt;
    }
    return cnt;
}
