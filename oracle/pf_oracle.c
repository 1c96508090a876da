/*
 * pf_oracle.c -- CPU ORACLE (test infrastructure only; see pf_oracle.h).
 *
 * Build with -O2 -ffp-contract=off (oracle/Makefile): the reference's results
 * depend on the exact rounding sequence, so no FMA contraction is allowed.
 * Every function cites the reference (or SPEC) lines it restates.
 */
#include "pf_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define OR_PI 3.14159265358979323846
#define OR_TWO_PI (2.0 * OR_PI)
#define OR_INV_4PI (1.0 / (4.0 * OR_PI))

/* ===== rng: proj/include/pf/rng.hpp ===================================== */

/* Pcg32::next_u32, rng.hpp:27-33 (XSH-RR on the pre-advance state). */
uint32_t or_next_u32(or_pcg32 *r) {
    uint64_t old = r->state;
    r->state = old * 6364136223846793005ULL + r->inc;
    uint32_t xs = (uint32_t)(((old >> 18u) ^ old) >> 27u);
    uint32_t rot = (uint32_t)(old >> 59u);
    return (xs >> rot) | (xs << ((0u - rot) & 31u));
}

/* Pcg32::seed, rng.hpp:19-25. */
void or_pcg_seed(or_pcg32 *r, uint64_t initstate, uint64_t initseq) {
    r->state = 0u;
    r->inc = (initseq << 1u) | 1u;
    or_next_u32(r);
    r->state += initstate;
    or_next_u32(r);
}

/* next_u64: high word first, rng.hpp:35-38. */
uint64_t or_next_u64(or_pcg32 *r) {
    uint64_t hi = or_next_u32(r);
    uint64_t lo = or_next_u32(r);
    return (hi << 32) | lo;
}

/* next_double: 53-bit mantissa, rng.hpp:41. */
double or_next_double(or_pcg32 *r) { return (double)(or_next_u64(r) >> 11) * 0x1.0p-53; }

/* next_below, rng.hpp:44-46. */
uint32_t or_next_below(or_pcg32 *r, uint32_t n) {
    return (uint32_t)(((uint64_t)or_next_u32(r) * n) >> 32);
}

/* splitmix64, rng.hpp:53-58. */
uint64_t or_splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

/* make_rng, rng.hpp:73-76: the index selects the PCG stream. */
void or_make_rng(or_pcg32 *r, uint64_t seed, uint64_t stream, uint64_t index) {
    uint64_t initstate = or_splitmix64(seed ^ (stream * 0x9e3779b97f4a7c15ULL));
    or_pcg_seed(r, initstate, index);
}

/* sample_uniform_sphere, rng.hpp:78-83. */
void or_sample_uniform_sphere(or_pcg32 *r, double out[3]) {
    double z = 1.0 - 2.0 * or_next_double(r);
    double phi = OR_TWO_PI * or_next_double(r);
    double t = 1.0 - z * z;
    double rr = sqrt(t > 0.0 ? t : 0.0);
    out[0] = rr * cos(phi);
    out[1] = rr * sin(phi);
    out[2] = z;
}

/* ===== math / phase ====================================================== */

/* std::max / std::min argument order: NaN in the second operand is ignored
 * (math.hpp:104-105 relies on this for axis-parallel rays). */
static inline double or_stdmax(double a, double b) { return (a < b) ? b : a; }
static inline double or_stdmin(double a, double b) { return (b < a) ? b : a; }

/* Aabb::intersect over the unit cube, math.hpp:95-108. */
int or_aabb_intersect(const double o[3], const double d[3], double tmin, double tmax,
                      double *t0, double *t1) {
    double a0 = tmin, a1 = tmax;
    for (int a = 0; a < 3; ++a) {
        double inv = 1.0 / d[a];
        double tn = (0.0 - o[a]) * inv;
        double tf = (1.0 - o[a]) * inv;
        if (inv < 0.0) {
            double s = tn;
            tn = tf;
            tf = s;
        }
        a0 = or_stdmax(a0, tn);
        a1 = or_stdmin(a1, tf);
        if (a0 > a1) {
            *t0 = a0;
            *t1 = a1;
            return 0;
        }
    }
    *t0 = a0;
    *t1 = a1;
    return 1;
}

/* hg_eval with |g| <= 0.999 clamp, phase.hpp:13-23. */
double or_hg_eval(double g, double c) {
    g = g < -0.999 ? -0.999 : (g > 0.999 ? 0.999 : g);
    double denom = 1.0 + g * g - 2.0 * g * c;
    denom = denom < 1e-12 ? 1e-12 : denom;
    return OR_INV_4PI * (1.0 - g * g) / (denom * sqrt(denom));
}

/* ===== volume: proj/src/volume.cpp ======================================= */

/* VolumeGrid ctor validation + attained range, volume.cpp:24-39. */
int or_grid_init(or_grid *g, int nx, int ny, int nz, const float *data) {
    if (nx <= 0 || ny <= 0 || nz <= 0) return 1;
    size_t n = (size_t)nx * ny * nz;
    float lo = 1.f, hi = 0.f;
    for (size_t i = 0; i < n; ++i) {
        float v = data[i];
        if (!isfinite(v) || v < 0.f || v > 1.f) return 1;
        lo = v < lo ? v : lo;
        hi = v > hi ? v : hi;
    }
    g->nx = nx;
    g->ny = ny;
    g->nz = nz;
    g->data = data;
    g->value_min = lo;
    g->value_max = hi;
    return 0;
}

/* Cell-centred axis split with boundary clamp, volume.cpp:44-57. */
static inline void or_axis(double x, int n, int *i0, double *f) {
    double c = x * n - 0.5;
    double lo = floor(c);
    int i = (int)lo;
    double fr = c - lo;
    if (i < 0) {
        i = 0;
        fr = 0.0;
    } else if (i >= n - 1) {
        i = n - 1;
        fr = 0.0;
    }
    *i0 = i;
    *f = fr;
}

static inline double or_voxel(const or_grid *g, int ix, int iy, int iz) {
    return (double)g->data[(size_t)ix + (size_t)g->nx * ((size_t)iy + (size_t)g->ny * (size_t)iz)];
}

/* VolumeGrid::sample, volume.cpp:41-77 (lerp x, then y, then z). */
double or_grid_sample(const or_grid *g, const double p[3]) {
    int ix, iy, iz;
    double fx, fy, fz;
    or_axis(p[0], g->nx, &ix, &fx);
    or_axis(p[1], g->ny, &iy, &fy);
    or_axis(p[2], g->nz, &iz, &fz);
    int jx = ix + 1 < g->nx - 1 ? ix + 1 : g->nx - 1;
    int jy = iy + 1 < g->ny - 1 ? iy + 1 : g->ny - 1;
    int jz = iz + 1 < g->nz - 1 ? iz + 1 : g->nz - 1;
    double c000 = or_voxel(g, ix, iy, iz), c100 = or_voxel(g, jx, iy, iz);
    double c010 = or_voxel(g, ix, jy, iz), c110 = or_voxel(g, jx, jy, iz);
    double c001 = or_voxel(g, ix, iy, jz), c101 = or_voxel(g, jx, iy, jz);
    double c011 = or_voxel(g, ix, jy, jz), c111 = or_voxel(g, jx, jy, jz);
    double c00 = c000 * (1.0 - fx) + c100 * fx;
    double c10 = c010 * (1.0 - fx) + c110 * fx;
    double c01 = c001 * (1.0 - fx) + c101 * fx;
    double c11 = c011 * (1.0 - fx) + c111 * fx;
    double c0 = c00 * (1.0 - fy) + c10 * fy;
    double c1 = c01 * (1.0 - fy) + c11 * fy;
    return c0 * (1.0 - fz) + c1 * fz;
}

/* TransferFunction::classify: clamp, linear scan, clamped lerp (volume.cpp:151-161). */
void or_tf_classify(const or_tf *tf, double scalar, double rgba[4]) {
    double s = scalar < 0.0 ? 0.0 : (scalar > 1.0 ? 1.0 : scalar);
    int hi = 1;
    while (hi + 1 < tf->n && tf->pts[hi * 5] < s) ++hi;
    const double *a = tf->pts + (hi - 1) * 5;
    const double *b = tf->pts + hi * 5;
    double t = (s - a[0]) / (b[0] - a[0]);
    t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
    for (int c = 0; c < 4; ++c) rgba[c] = a[1 + c] + (b[1 + c] - a[1 + c]) * t;
}

/* TransferFunction::max_alpha, volume.cpp:163-168. */
double or_tf_max_alpha(const or_tf *tf, double lo, double hi) {
    double ra[4], rb[4];
    or_tf_classify(tf, lo, ra);
    or_tf_classify(tf, hi, rb);
    double m = or_stdmax(ra[3], rb[3]);
    for (int i = 0; i < tf->n; ++i) {
        double s = tf->pts[i * 5];
        if (s > lo && s < hi) m = or_stdmax(m, tf->pts[i * 5 + 4]);
    }
    return m;
}

/* Medium ctor: sigma_max = density_scale * max_alpha(range), volume.cpp:197-202. */
int or_medium_init(or_medium *m, const or_grid *g, const or_tf *tf, double density_scale) {
    if (!(density_scale > 0.0) || !isfinite(density_scale)) return 1;
    m->grid = *g;
    m->tf = *tf;
    m->density_scale = density_scale;
    m->sigma_max = density_scale * or_tf_max_alpha(tf, (double)g->value_min, (double)g->value_max);
    return 0;
}

static inline int or_finite3(const double v[3]) {
    return isfinite(v[0]) && isfinite(v[1]) && isfinite(v[2]);
}

/* delta_track (Woodcock tracking), volume.cpp:204-225. */
int or_delta_track(const or_medium *m, const double o[3], const double d[3], double tmin,
                   double tmax, or_pcg32 *rng, double pos[3], double *scalar, double rgba[4]) {
    if (!or_finite3(o) || !or_finite3(d) || !isfinite(tmin) || tmin < 0.0 || tmin > tmax)
        return -1;
    double t0, t1;
    if (!or_aabb_intersect(o, d, tmin, tmax, &t0, &t1)) return 0;
    const double sigma_max = m->sigma_max;
    if (sigma_max <= 0.0) return 0;
    double t = t0;
    const double inv_sigma_max = 1.0 / sigma_max;
    for (;;) {
        t -= log(1.0 - or_next_double(rng)) * inv_sigma_max;
        if (t > t1) return 0;
        double x[3] = {o[0] + d[0] * t, o[1] + d[1] * t, o[2] + d[2] * t};
        double s = or_grid_sample(&m->grid, x);
        double c[4];
        or_tf_classify(&m->tf, s, c);
        double sigma = m->density_scale * c[3];
        if (or_next_double(rng) * sigma_max < sigma) {
            pos[0] = x[0];
            pos[1] = x[1];
            pos[2] = x[2];
            if (scalar) *scalar = s;
            if (rgba) memcpy(rgba, c, sizeof(c));
            return 1;
        }
    }
}

/* transmittance: n_trials delta flights a -> b, volume.cpp:227-256. */
double or_transmittance(const or_medium *m, const double a[3], const double b[3], or_pcg32 *rng,
                        int n_trials) {
    if (n_trials <= 0) return -1.0;
    double dv[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
    double len = sqrt(dv[0] * dv[0] + dv[1] * dv[1] + dv[2] * dv[2]);
    if (len == 0.0) return 1.0;
    double dir[3] = {dv[0] / len, dv[1] / len, dv[2] / len};
    double t0, t1;
    if (!or_aabb_intersect(a, dir, 0.0, len, &t0, &t1)) return 1.0;
    if (m->sigma_max <= 0.0) return 1.0;
    int passed = 0;
    for (int trial = 0; trial < n_trials; ++trial) {
        double t = t0;
        int collided = 0;
        const double inv_sigma_max = 1.0 / m->sigma_max;
        for (;;) {
            t -= log(1.0 - or_next_double(rng)) * inv_sigma_max;
            if (t > t1) break;
            double x[3] = {a[0] + dir[0] * t, a[1] + dir[1] * t, a[2] + dir[2] * t};
            double c[4];
            or_tf_classify(&m->tf, or_grid_sample(&m->grid, x), c);
            double sigma = m->density_scale * c[3];
            if (or_next_double(rng) * m->sigma_max < sigma) {
                collided = 1;
                break;
            }
        }
        if (!collided) ++passed;
    }
    return (double)passed / n_trials;
}

int or_delta_track_batch(const or_medium *m, size_t n, const double *o3, const double *d3,
                         const double *tmin, const double *tmax, uint64_t seed, uint64_t stream,
                         const uint64_t *idx, int *hit, double *pos3, double *scalar1, double *rgba4) {
    for (size_t i = 0; i < n; ++i) {
        or_pcg32 r;
        or_make_rng(&r, seed, stream, idx[i]);
        double pos[3] = {0, 0, 0}, rgba[4] = {0, 0, 0, 0}, s;
        int h = or_delta_track(m, o3 + 3 * i, d3 + 3 * i, tmin[i], tmax[i], &r, pos, &s, rgba);
        if (h < 0) return -1;
        hit[i] = h;
        if (pos3) memcpy(pos3 + 3 * i, pos, sizeof(pos));
        if (scalar1) scalar1[i] = h ? s : 0.0;
        if (rgba4) memcpy(rgba4 + 4 * i, rgba, sizeof(rgba));
    }
    return 0;
}

void or_transmittance_batch(const or_medium *m, size_t n, const double *a3, const double *b3,
                            uint64_t seed, uint64_t stream, const uint64_t *idx, int n_trials,
                            double *out) {
    for (size_t i = 0; i < n; ++i) {
        or_pcg32 r;
        or_make_rng(&r, seed, stream, idx[i]);
        out[i] = or_transmittance(m, a3 + 3 * i, b3 + 3 * i, &r, n_trials);
    }
}

void or_rng_doubles(uint64_t seed, uint64_t stream, size_t n, const uint64_t *idx, int draws,
                    double *out) {
    for (size_t i = 0; i < n; ++i) {
        or_pcg32 r;
        or_make_rng(&r, seed, stream, idx[i]);
        for (int k = 0; k < draws; ++k) out[i * (size_t)draws + k] = or_next_double(&r);
    }
}

/* ===== neural field: SPEC.md:352-447 ====================================== */

/* N_l = floor(base * growth^l)  (pinned App. B.6). */
int or_hashgrid_level_res(const or_hashgrid_cfg *c, int l) {
    return (int)floor((double)c->base_res * pow(c->growth, (double)l));
}

/* 1 when the level's (N_l+1)^d vertices fit in T (dense addressing). */
static int or_hashgrid_level_dense(const or_hashgrid_cfg *c, int l) {
    uint64_t n1 = (uint64_t)or_hashgrid_level_res(c, l) + 1u;
    uint64_t T = 1ull << c->log2_table;
    uint64_t v = 1;
    for (int i = 0; i < c->dims; ++i) {
        v *= n1;
        if (v > T) return 0;
    }
    return 1;
}

/* (N_l+1)^d vertices, dense when that fits in T, else hashed into T. */
uint32_t or_hashgrid_level_size(const or_hashgrid_cfg *c, int l) {
    uint64_t n1 = (uint64_t)or_hashgrid_level_res(c, l) + 1u;
    uint64_t T = 1ull << c->log2_table;
    uint64_t v = 1;
    for (int i = 0; i < c->dims; ++i) {
        v *= n1;
        if (v > T) return (uint32_t)T;
    }
    return (uint32_t)v;
}

size_t or_hashgrid_param_count(const or_hashgrid_cfg *c) {
    size_t n = 0;
    for (int l = 0; l < c->levels; ++l) n += (size_t)or_hashgrid_level_size(c, l) * c->features;
    return n;
}

int or_field_input_dim(const or_field_cfg *c) {
    return c->pos.levels * c->pos.features + c->dir.levels * c->dir.features + 1;
}

size_t or_field_param_count(const or_field_cfg *c) {
    size_t din = (size_t)or_field_input_dim(c), w = (size_t)c->width;
    return or_hashgrid_param_count(&c->pos) + or_hashgrid_param_count(&c->dir) + din * w + w +
           (size_t)(c->hidden_layers - 1) * (w * w + w) + 3 * w + 3;
}

/* Multilinear hashgrid lookup of one input. */
/* Per-level constants, memoised per thread (they only depend on the config). */
typedef struct {
    or_hashgrid_cfg cfg;
    int valid;
    int N[64];
    uint32_t size[64];
    int dense[64];
} or_level_cache;
static _Thread_local or_level_cache g_level_cache[2];

static const or_level_cache *or_levels(const or_hashgrid_cfg *c) {
    or_level_cache *lc = &g_level_cache[c->dims == 3 ? 0 : 1];
    if (!lc->valid || lc->cfg.dims != c->dims || lc->cfg.levels != c->levels ||
        lc->cfg.features != c->features || lc->cfg.base_res != c->base_res ||
        lc->cfg.growth != c->growth || lc->cfg.log2_table != c->log2_table) {
        for (int l = 0; l < c->levels && l < 64; ++l) {
            lc->N[l] = or_hashgrid_level_res(c, l);
            lc->size[l] = or_hashgrid_level_size(c, l);
            lc->dense[l] = or_hashgrid_level_dense(c, l);
        }
        lc->cfg = *c;
        lc->valid = 1;
    }
    return lc;
}

static void or_hashgrid_encode(const or_hashgrid_cfg *c, const float *table, const double *in,
                               double *out) {
    static const uint32_t primes[3] = {1u, 2654435761u, 805459861u};
    const int d = c->dims, F = c->features;
    const uint32_t Tmask = (1u << c->log2_table) - 1u;
    const or_level_cache *lc = or_levels(c);
    size_t off = 0;
    for (int l = 0; l < c->levels; ++l) {
        const int N = lc->N[l];
        const uint32_t size = lc->size[l];
        const int dense = lc->dense[l];
        int ci[3];
        double f[3];
        for (int i = 0; i < d; ++i) {
            double p = in[i] < 0.0 ? 0.0 : (in[i] > 1.0 ? 1.0 : in[i]);
            double s = p * N;
            double fl = floor(s);
            int cc = (int)fl;
            if (cc > N - 1) cc = N - 1;
            ci[i] = cc;
            f[i] = s - (double)cc;
        }
        for (int k = 0; k < F; ++k) out[l * F + k] = 0.0;
        for (int corner = 0; corner < (1 << d); ++corner) {
            double w = 1.0;
            uint32_t v[3] = {0, 0, 0};
            for (int i = 0; i < d; ++i) {
                int bit = (corner >> i) & 1;
                w *= bit ? f[i] : (1.0 - f[i]);
                v[i] = (uint32_t)(ci[i] + bit);
            }
            uint32_t idx;
            if (dense) {
                uint32_t n1 = (uint32_t)N + 1u;
                idx = v[0];
                uint32_t mul = n1;
                for (int i = 1; i < d; ++i) {
                    idx += v[i] * mul;
                    mul *= n1;
                }
            } else {
                uint32_t h = 0;
                for (int i = 0; i < d; ++i) h ^= v[i] * primes[i];
                idx = h & Tmask;
            }
            const float *e = table + off + (size_t)idx * F;
            for (int k = 0; k < F; ++k) out[l * F + k] += w * (double)e[k];
        }
        off += (size_t)size * F;
    }
}

/* Deterministic field init, the same draw order as the
 * product's pf_field_init: make_rng(seed, FieldInit, 0); tables U(-e, e);
 * per layer W ~ He-uniform by fan-in, then biases U(-b, b).  Lets the
 * reference CPU arm build its parameters without the GPU library. */
void or_field_init(const or_field_cfg *c, uint64_t seed, double embed_scale, double bias_scale,
                   float *out) {
    or_pcg32 r;
    or_make_rng(&r, seed, 6 /* Stream::FieldInit, rng.hpp:68 */, 0);
    const size_t ntab = or_hashgrid_param_count(&c->pos) + or_hashgrid_param_count(&c->dir);
    size_t p = 0;
    for (; p < ntab; ++p) out[p] = (float)((2.0 * or_next_double(&r) - 1.0) * embed_scale);
    const int din = or_field_input_dim(c);
    for (int L = 0; L <= c->hidden_layers; ++L) {
        const int K = L == 0 ? din : c->width, N = L < c->hidden_layers ? c->width : 3;
        const double a = sqrt(6.0 / K);
        for (int i = 0; i < N * K; ++i) out[p++] = (float)((2.0 * or_next_double(&r) - 1.0) * a);
        for (int i = 0; i < N; ++i) out[p++] = (float)((2.0 * or_next_double(&r) - 1.0) * bias_scale);
    }
}

void or_field_encode(const or_field_cfg *c, const float *params, const double x[3],
                     const double wsph[2], double g, double *feat) {
    const size_t npos = or_hashgrid_param_count(&c->pos);
    or_hashgrid_encode(&c->pos, params, x, feat);
    or_hashgrid_encode(&c->dir, params + npos, wsph, feat + c->pos.levels * c->pos.features);
    feat[or_field_input_dim(c) - 1] = (g + 1.0) / 2.0;
}

/* Dense layer out[o] = (sum_k W[o][k] x[k]) + b[o], k ascending. */
static void or_dense(const float *W, const float *b, int nin, int nout, const double *x,
                     double *y, int relu) {
    for (int o = 0; o < nout; ++o) {
        double acc = 0.0;
        for (int k = 0; k < nin; ++k) acc += (double)W[(size_t)o * nin + k] * x[k];
        acc += (double)b[o];
        y[o] = (relu && acc < 0.0) ? 0.0 : acc;
    }
}

void or_field_forward(const or_field_cfg *c, const float *params, size_t n, const double *x3,
                      const double *w2, const double *g, double *out3) {
    const int din = or_field_input_dim(c), w = c->width;
    const float *mlp =
        params + or_hashgrid_param_count(&c->pos) + or_hashgrid_param_count(&c->dir);
    double *feat = (double *)malloc(sizeof(double) * (size_t)(din > w ? din : w));
    double *h0 = (double *)malloc(sizeof(double) * (size_t)w);
    double *h1 = (double *)malloc(sizeof(double) * (size_t)w);
    for (size_t i = 0; i < n; ++i) {
        or_field_encode(c, params, x3 + 3 * i, w2 + 2 * i, g[i], feat);
        const float *p = mlp;
        or_dense(p, p + (size_t)w * din, din, w, feat, h0, 1);
        p += (size_t)w * din + w;
        for (int L = 1; L < c->hidden_layers; ++L) {
            or_dense(p, p + (size_t)w * w, w, w, h0, h1, 1);
            p += (size_t)w * w + w;
            double *t = h0;
            h0 = h1;
            h1 = t;
        }
        or_dense(p, p + 3 * w, w, 3, h0, out3 + 3 * i, 0);
    }
    free(feat);
    free(h0);
    free(h1);
}

void or_field_infer(const or_field_cfg *c, const float *params, size_t n, const double *x3,
                    const double *w2, const double *g, double *out3) {
    or_field_forward(c, params, n, x3, w2, g, out3);
    for (size_t i = 0; i < 3 * n; ++i) out3[i] = or_decode_log(out3[i], c->psi);
}

/* (theta/pi, (phi+pi)/2pi), phi = atan2(w_y, w_x). */
void or_dir_to_sph(const double w[3], double out[2]) {
    double z = w[2] < -1.0 ? -1.0 : (w[2] > 1.0 ? 1.0 : w[2]);
    out[0] = acos(z) / OR_PI;
    out[1] = (atan2(w[1], w[0]) + OR_PI) / OR_TWO_PI;
}

/* ===== training: SPEC.md:403-411 (train_step), 380-383 (AdamState) ========
 * binary64 throughout (parameters included), so the finite-difference oracle
 * of SPEC.md:409 applies to it directly; the GPU trainer (binary32 master
 * parameters) is checked against these gradients. */

/* lr(step) = lr0 * decay^floor(max(0, step - start*T) / interval). */
double or_lr_at(const or_adam_cfg *a, uint64_t step, uint64_t total) {
    double s = (double)step - a->decay_start * (double)total;
    if (s < 0.0) s = 0.0;
    return a->lr * pow(a->decay, floor(s / (double)a->decay_interval));
}

/* Corner table offsets (entries, relative to the grid's first entry) and
 * multilinear weights of one input at every level: the same arithmetic as
 * or_hashgrid_encode. idx/w hold levels * 2^dims values. */
static void or_grid_corners(const or_hashgrid_cfg *c, const double *in, uint32_t *idx_out, double *w_out) {
    static const uint32_t primes[3] = {1u, 2654435761u, 805459861u};
    const int d = c->dims;
    const uint32_t Tmask = (1u << c->log2_table) - 1u;
    const or_level_cache *lc = or_levels(c);
    size_t off = 0;
    for (int l = 0; l < c->levels; ++l) {
        const int N = lc->N[l];
        int ci[3];
        double f[3];
        for (int i = 0; i < d; ++i) {
            double p = in[i] < 0.0 ? 0.0 : (in[i] > 1.0 ? 1.0 : in[i]);
            double s = p * N;
            int cc = (int)floor(s);
            if (cc > N - 1) cc = N - 1;
            ci[i] = cc;
            f[i] = s - (double)cc;
        }
        for (int corner = 0; corner < (1 << d); ++corner) {
            double w = 1.0;
            uint32_t v[3] = {0, 0, 0};
            for (int i = 0; i < d; ++i) {
                int bit = (corner >> i) & 1;
                w *= bit ? f[i] : (1.0 - f[i]);
                v[i] = (uint32_t)(ci[i] + bit);
            }
            uint32_t idx;
            if (lc->dense[l]) {
                uint32_t n1 = (uint32_t)N + 1u;
                idx = v[0];
                uint32_t mul = n1;
                for (int i = 1; i < d; ++i) {
                    idx += v[i] * mul;
                    mul *= n1;
                }
            } else {
                uint32_t h = 0;
                for (int i = 0; i < d; ++i) h ^= v[i] * primes[i];
                idx = h & Tmask;
            }
            idx_out[l * (1 << d) + corner] = (uint32_t)(off + idx);
            w_out[l * (1 << d) + corner] = w;
        }
        off += (size_t)lc->size[l];
    }
}

/* Loss (rMSE) of a batch and, if grad != NULL, its gradient
 * w.r.t. every parameter (dense vector, zero where untouched) and the
 * per-entry touched flags of the two tables (touched may be NULL). */
double or_train_grad(const or_field_cfg *c, const double *params, size_t n, const double *x3, const double *w2,
                     const double *g, const double *targets3, double eps_rel, double *grad,
                     uint8_t *touched, double *pred_out, const double *den_in) {
    const int din = or_field_input_dim(c), W = c->width, H = c->hidden_layers;
    const size_t npos = or_hashgrid_param_count(&c->pos), ndir = or_hashgrid_param_count(&c->dir);
    const size_t nparams = or_field_param_count(c);
    const double *mlp = params + npos + ndir;
    const int Fp = c->pos.features, Fd = c->dir.features;
    const int cp = 1 << c->pos.dims, cd = 1 << c->dir.dims;
    if (grad) memset(grad, 0, sizeof(double) * nparams);
    if (touched) memset(touched, 0, (npos / Fp) + (ndir / Fd));
    double *a = (double *)malloc(sizeof(double) * (size_t)(din + H * W + 3)); /* a_0 | a_1..a_H | out */
    double *dz = (double *)malloc(sizeof(double) * (size_t)(W > din ? W : din));
    double *da = (double *)malloc(sizeof(double) * (size_t)(W > din ? W : din));
    uint32_t *ip = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(c->pos.levels * cp));
    uint32_t *id = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(c->dir.levels * cd));
    double *wp = (double *)malloc(sizeof(double) * (size_t)(c->pos.levels * cp));
    double *wd = (double *)malloc(sizeof(double) * (size_t)(c->dir.levels * cd));
    double loss = 0.0;
    const double inv = 1.0 / (3.0 * (double)n);
    for (size_t q = 0; q < n; ++q) {
        /* encode */
        or_grid_corners(&c->pos, x3 + 3 * q, ip, wp);
        or_grid_corners(&c->dir, w2 + 2 * q, id, wd);
        for (int k = 0; k < din; ++k) a[k] = 0.0;
        for (int l = 0; l < c->pos.levels; ++l)
            for (int j = 0; j < cp; ++j)
                for (int f = 0; f < Fp; ++f)
                    a[l * Fp + f] += wp[l * cp + j] * params[(size_t)ip[l * cp + j] * Fp + f];
        const int o0 = c->pos.levels * Fp;
        for (int l = 0; l < c->dir.levels; ++l)
            for (int j = 0; j < cd; ++j)
                for (int f = 0; f < Fd; ++f)
                    a[o0 + l * Fd + f] += wd[l * cd + j] * params[npos + (size_t)id[l * cd + j] * Fd + f];
        a[din - 1] = (g[q] + 1.0) / 2.0;
        /* MLP forward, keeping a_l */
        const double *p = mlp;
        const double *in = a;
        int nin = din;
        double *outp = a + din;
        for (int L = 0; L <= H; ++L) {
            const int nout = L < H ? W : 3;
            for (int o = 0; o < nout; ++o) {
                double acc = 0.0;
                for (int k = 0; k < nin; ++k) acc += p[(size_t)o * nin + k] * in[k];
                acc += p[(size_t)nout * nin + o];
                outp[o] = (L < H && acc < 0.0) ? 0.0 : acc;
            }
            p += (size_t)nout * nin + nout;
            in = outp;
            outp += nout;
            nin = nout;
        }
        const double *pred = a + din + (size_t)H * W;
        for (int ch = 0; ch < 3; ++ch) {
            const double e = pred[ch] - targets3[3 * q + ch];
            /* prediction detached; den_in freezes it (finite-difference oracle) */
            const double den = den_in ? den_in[3 * q + ch] : pred[ch] * pred[ch] + eps_rel;
            if (pred_out) pred_out[3 * q + ch] = pred[ch];
            loss += e * e / den;
            dz[ch] = 2.0 * e / den * inv;
        }
        if (!grad) continue;
        /* MLP backward: layer L maps a_L (nin) -> z_L (nout) */
        size_t off[16];
        {
            size_t o = npos + ndir;
            int ni = din;
            for (int L = 0; L <= H; ++L) {
                const int no = L < H ? W : 3;
                off[L] = o;
                o += (size_t)no * ni + no;
                ni = no;
            }
        }
        for (int L = H; L >= 0; --L) {
            const int nout = L < H ? W : 3, nin2 = L == 0 ? din : W;
            const double *aL = L == 0 ? a : a + din + (size_t)(L - 1) * W;
            double *gW = grad + off[L], *gb = gW + (size_t)nout * nin2;
            const double *Wl = params + off[L];
            for (int o = 0; o < nout; ++o) {
                for (int k = 0; k < nin2; ++k) gW[(size_t)o * nin2 + k] += dz[o] * aL[k];
                gb[o] += dz[o];
            }
            for (int k = 0; k < nin2; ++k) {
                double s = 0.0;
                for (int o = 0; o < nout; ++o) s += Wl[(size_t)o * nin2 + k] * dz[o];
                da[k] = s;
            }
            if (L > 0)
                for (int k = 0; k < nin2; ++k) dz[k] = aL[k] > 0.0 ? da[k] : 0.0; /* relu'(z) = [z > 0] */
        }
        /* da = d loss / d feature -> tables */
        for (int l = 0; l < c->pos.levels; ++l)
            for (int j = 0; j < cp; ++j) {
                const size_t e = ip[l * cp + j];
                for (int f = 0; f < Fp; ++f) grad[e * Fp + f] += wp[l * cp + j] * da[l * Fp + f];
                if (touched) touched[e] = 1;
            }
        for (int l = 0; l < c->dir.levels; ++l)
            for (int j = 0; j < cd; ++j) {
                const size_t e = id[l * cd + j];
                for (int f = 0; f < Fd; ++f) grad[npos + e * Fd + f] += wd[l * cd + j] * da[o0 + l * Fd + f];
                if (touched) touched[npos / Fp + e] = 1;
            }
    }
    free(a);
    free(dz);
    free(da);
    free(ip);
    free(id);
    free(wp);
    free(wd);
    return loss * inv;
}

/* Adam with bias correction on the global step t = step + 1:
 * MLP parameters always, table parameters only for touched entries (sparse
 * gradients).  params / m / v updated in place. */
void or_adam_update(const or_field_cfg *c, const or_adam_cfg *a, double *params, const double *grad,
                    const uint8_t *touched, double *m, double *v, uint64_t step, uint64_t total) {
    const size_t npos = or_hashgrid_param_count(&c->pos), ndir = or_hashgrid_param_count(&c->dir);
    const size_t n = or_field_param_count(c);
    const double lr = or_lr_at(a, step, total);
    const double t = (double)(step + 1);
    const double bc1 = 1.0 - pow(a->beta1, t), bc2 = 1.0 - pow(a->beta2, t);
    for (size_t i = 0; i < n; ++i) {
        if (i < npos + ndir) {
            const size_t e = i < npos ? i / (size_t)c->pos.features
                                      : npos / (size_t)c->pos.features + (i - npos) / (size_t)c->dir.features;
            if (!touched[e]) continue;
        }
        m[i] = a->beta1 * m[i] + (1.0 - a->beta1) * grad[i];
        v[i] = a->beta2 * v[i] + (1.0 - a->beta2) * grad[i] * grad[i];
        const double mh = m[i] / bc1, vh = v[i] / bc2;
        params[i] -= lr * mh / (sqrt(vh) + a->eps);
    }
}

/* ===== estimator: SPEC.md:299-326 ======================================== */

/* Eq. 7 with the L > 1 clamp. */
double or_encode_log(double L, double psi) {
    if (L > 1.0) return 0.0;
    if (L > pow(10.0, -psi)) return -log10(L) / psi;
    return 1.0;
}

/* Eq. 8 with L' clamped to [0,1]. */
double or_decode_log(double Lp, double psi) {
    double c = Lp < 0.0 ? 0.0 : (Lp > 1.0 ? 1.0 : Lp);
    return pow(10.0, -c * psi);
}

/* ===== KNN: SPEC.md:239-267 ============================================== */

static inline float or_d2(const float p[3], const float q[3]) {
    float dx = p[0] - q[0], dy = p[1] - q[1], dz = p[2] - q[2];
    float a = dx * dx;
    float b = dy * dy;
    float c = dz * dz;
    return (a + b) + c;
}

/* Sorted top-K insertion on the (d2, id) lexicographic key. */
static inline int or_key_less(float da, uint32_t ia, float db, uint32_t ib) {
    return da < db || (da == db && ia < ib);
}

static void or_topk_insert(uint32_t *ids, float *d2, int *count, int K, float d, uint32_t id) {
    int n = *count;
    if (n == K) {
        if (!or_key_less(d, id, d2[K - 1], ids[K - 1])) return;
        n = K - 1;
    }
    int pos = n;
    while (pos > 0 && or_key_less(d, id, d2[pos - 1], ids[pos - 1])) {
        d2[pos] = d2[pos - 1];
        ids[pos] = ids[pos - 1];
        --pos;
    }
    d2[pos] = d;
    ids[pos] = id;
    *count = n + 1;
}

int or_knn_brute(const or_photon *ph, size_t n, const float q[3], int g_index, int K,
                 float r_max, uint32_t *ids, float *d2) {
    const float r2 = r_max * r_max;
    int count = 0;
    if (K <= 0) return 0;
    for (size_t i = 0; i < n; ++i) {
        if (ph[i].g_index != g_index) continue;
        float d = or_d2(ph[i].pos, q);
        if (!(d <= r2)) continue;
        or_topk_insert(ids, d2, &count, K, d, (uint32_t)i);
    }
    return count;
}

/* Balanced kd-tree: median split on the longest bbox axis, leaves <= 8. */
typedef struct {
    float lo[3], hi[3];
    int left, right; /* -1 for leaves */
    uint32_t begin, end;
} or_kdnode;

struct or_kdtree {
    const or_photon *ph;
    uint32_t *perm;
    or_kdnode *nodes;
    int n_nodes, cap;
};

static const or_photon *g_sort_ph;
static int g_sort_axis;
static int or_cmp_axis(const void *a, const void *b) {
    uint32_t ia = *(const uint32_t *)a, ib = *(const uint32_t *)b;
    float fa = g_sort_ph[ia].pos[g_sort_axis], fb = g_sort_ph[ib].pos[g_sort_axis];
    if (fa < fb) return -1;
    if (fa > fb) return 1;
    return ia < ib ? -1 : (ia > ib ? 1 : 0);
}

static int or_kd_new_node(or_kdtree *t) {
    if (t->n_nodes == t->cap) {
        t->cap = t->cap ? 2 * t->cap : 1024;
        t->nodes = (or_kdnode *)realloc(t->nodes, sizeof(or_kdnode) * (size_t)t->cap);
    }
    return t->n_nodes++;
}

static int or_kd_build_rec(or_kdtree *t, uint32_t b, uint32_t e) {
    int id = or_kd_new_node(t);
    or_kdnode nd;
    for (int a = 0; a < 3; ++a) {
        nd.lo[a] = INFINITY;
        nd.hi[a] = -INFINITY;
    }
    for (uint32_t i = b; i < e; ++i) {
        const float *p = t->ph[t->perm[i]].pos;
        for (int a = 0; a < 3; ++a) {
            nd.lo[a] = p[a] < nd.lo[a] ? p[a] : nd.lo[a];
            nd.hi[a] = p[a] > nd.hi[a] ? p[a] : nd.hi[a];
        }
    }
    nd.begin = b;
    nd.end = e;
    nd.left = nd.right = -1;
    if (e - b > 8) {
        int axis = 0;
        float ext = nd.hi[0] - nd.lo[0];
        for (int a = 1; a < 3; ++a)
            if (nd.hi[a] - nd.lo[a] > ext) {
                ext = nd.hi[a] - nd.lo[a];
                axis = a;
            }
        g_sort_ph = t->ph;
        g_sort_axis = axis;
        qsort(t->perm + b, e - b, sizeof(uint32_t), or_cmp_axis);
        uint32_t mid = b + (e - b) / 2;
        int l = or_kd_build_rec(t, b, mid);
        int r = or_kd_build_rec(t, mid, e);
        nd.left = l;
        nd.right = r;
    }
    t->nodes[id] = nd;
    return id;
}

or_kdtree *or_kd_build(const or_photon *ph, size_t n) {
    or_kdtree *t = (or_kdtree *)calloc(1, sizeof(or_kdtree));
    t->ph = ph;
    t->perm = (uint32_t *)malloc(sizeof(uint32_t) * (n ? n : 1));
    for (size_t i = 0; i < n; ++i) t->perm[i] = (uint32_t)i;
    if (n) or_kd_build_rec(t, 0, (uint32_t)n);
    return t;
}

void or_kd_free(or_kdtree *t) {
    if (!t) return;
    free(t->perm);
    free(t->nodes);
    free(t);
}

/* Lower bound (in double) of the squared distance from q to a node box. */
static double or_box_d2(const or_kdnode *nd, const float q[3]) {
    double s = 0.0;
    for (int a = 0; a < 3; ++a) {
        double d = 0.0;
        if (q[a] < nd->lo[a]) d = (double)nd->lo[a] - (double)q[a];
        else if (q[a] > nd->hi[a]) d = (double)q[a] - (double)nd->hi[a];
        s += d * d;
    }
    return s;
}

/* Iterative, explicit-stack traversal.  Pruning is conservative
 * by a relative 1e-5 so binary32 rounding of d2 can never drop a tie. */
int or_kd_knn(const or_kdtree *t, const float q[3], int g_index, int K, float r_max,
              uint32_t *ids, float *d2) {
    if (K <= 0 || t->n_nodes == 0) return 0;
    const float r2 = r_max * r_max;
    int count = 0;
    int stack[128];
    int sp = 0;
    stack[sp++] = 0;
    while (sp) {
        const or_kdnode *nd = &t->nodes[stack[--sp]];
        double lb = or_box_d2(nd, q) * (1.0 - 1e-5);
        if (lb > (double)r2) continue;
        if (count == K && lb > (double)d2[K - 1]) continue;
        if (nd->left < 0) {
            for (uint32_t i = nd->begin; i < nd->end; ++i) {
                uint32_t id = t->perm[i];
                if (t->ph[id].g_index != g_index) continue;
                float d = or_d2(t->ph[id].pos, q);
                if (!(d <= r2)) continue;
                or_topk_insert(ids, d2, &count, K, d, id);
            }
        } else {
            /* push the far child first so the near child is visited first */
            const or_kdnode *L = &t->nodes[nd->left], *R = &t->nodes[nd->right];
            double dl = or_box_d2(L, q), dr = or_box_d2(R, q);
            if (dl <= dr) {
                stack[sp++] = nd->right;
                stack[sp++] = nd->left;
            } else {
                stack[sp++] = nd->left;
                stack[sp++] = nd->right;
            }
        }
    }
    return count;
}

/* Eq. 6: sum_n p_g(w . w_n) Phi_n / ((4/3) pi r^3), r = farthest distance,
 * r < 1e-6 -> 0. */
void or_estimate_radiance(const or_photon *ph, const uint32_t *ids, const float *d2, int count,
                          const double w[3], double g, double out[3]) {
    out[0] = out[1] = out[2] = 0.0;
    if (count <= 0) return;
    double r = sqrt((double)d2[count - 1]);
    if (r < 1e-6) return;
    double s[3] = {0.0, 0.0, 0.0};
    for (int k = 0; k < count; ++k) {
        const or_photon *p = &ph[ids[k]];
        double c = w[0] * (double)p->dir[0] + w[1] * (double)p->dir[1] + w[2] * (double)p->dir[2];
        double f = or_hg_eval(g, c);
        for (int ch = 0; ch < 3; ++ch) s[ch] += f * (double)p->power[ch];
    }
    double vol = (4.0 / 3.0) * OR_PI * (r * r * r);
    for (int ch = 0; ch < 3; ++ch) out[ch] = s[ch] / vol;
}

void or_make_queries(uint64_t seed, uint64_t step, size_t batch, int n_phases, float *x3,
                     double *w3, uint8_t *gidx) {
    for (size_t i = 0; i < batch; ++i) {
        or_pcg32 r;
        or_make_rng(&r, seed, OR_STREAM_TRAIN, step * (uint64_t)batch + i);
        for (int a = 0; a < 3; ++a) x3[3 * i + a] = (float)or_next_double(&r);
        or_sample_uniform_sphere(&r, w3 + 3 * i);
        gidx[i] = (uint8_t)or_next_below(&r, (uint32_t)n_phases);
    }
}

/* First segment whose end fraction >= (step+1)/total. */
double or_schedule_radius(const double *ends, const double *radii, int n, uint64_t step,
                          uint64_t total) {
    double progress = (double)(step + 1) / (double)total;
    for (int i = 0; i < n; ++i)
        if (ends[i] >= progress) return radii[i];
    return radii[n - 1];
}

void or_knn_targets(const or_kdtree *t, const or_photon *ph, size_t nq, const float *x3,
                    const double *w3, const uint8_t *gidx, const double *phase_set, int K,
                    float r_max, double psi, uint32_t *ids, float *d2, int *counts,
                    double *targets3) {
    for (size_t i = 0; i < nq; ++i) {
        uint32_t *id = ids + i * (size_t)K;
        float *dd = d2 + i * (size_t)K;
        int c = or_kd_knn(t, x3 + 3 * i, gidx[i], K, r_max, id, dd);
        counts[i] = c;
        double L[3];
        or_estimate_radiance(ph, id, dd, c, w3 + 3 * i, phase_set[gidx[i]], L);
        for (int ch = 0; ch < 3; ++ch) targets3[3 * i + ch] = or_encode_log(L[ch], psi);
    }
}

/* ===== photon tracing: Alg. 1 ============================================= */

/* hg_sample_cos, phase.hpp:26-31. */
double or_hg_sample_cos(double g, double u) {
    g = g < -0.999 ? -0.999 : (g > 0.999 ? 0.999 : g);
    if (fabs(g) < 1e-6) return 1.0 - 2.0 * u;
    double sq = (1.0 - g * g) / (1.0 - g + 2.0 * g * u);
    double c = (1.0 + g * g - sq * sq) / (2.0 * g);
    return c < -1.0 ? -1.0 : (c > 1.0 ? 1.0 : c);
}

/* orthonormal_basis (Duff et al.) + from_local_frame, math.hpp:113-126. */
void or_from_local_frame(const double n[3], const double l[3], double out[3]) {
    const double sign = copysign(1.0, n[2]);
    const double a = -1.0 / (sign + n[2]);
    const double c = n[0] * n[1] * a;
    const double t[3] = {1.0 + sign * n[0] * n[0] * a, sign * c, -sign * n[0]};
    const double b[3] = {c, sign + n[1] * n[1] * a, -n[1]};
    for (int k = 0; k < 3; ++k) out[k] = t[k] * l[0] + b[k] * l[1] + n[k] * l[2];
}

/* hg_sample, phase.hpp:34-40. */
void or_hg_sample(double g, const double w_in[3], double u1, double u2, double out[3]) {
    double ct = or_hg_sample_cos(g, u1);
    double t = 1.0 - ct * ct;
    double st = sqrt(t > 0.0 ? t : 0.0);
    double phi = OR_TWO_PI * u2;
    double local[3] = {st * cos(phi), st * sin(phi), ct};
    or_from_local_frame(w_in, local, out);
}

/* emit_direction (photon.hpp:50): uniform over the cone the
 * unit box's bounding sphere (centre 0.5, radius sqrt(3)/2) subtends from the
 * light; full sphere for lights inside it.  Pinned: cos = 1 - u1 (1 - cos_max),
 * phi = 2 pi u2, rotated by from_local_frame about normalize(centre - P). */
void or_emit_direction(const double P[3], or_pcg32 *rng, double out[3]) {
    const double R = 0.5 * sqrt(3.0);
    double v[3] = {0.5 - P[0], 0.5 - P[1], 0.5 - P[2]};
    double d = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    if (d <= R) {
        or_sample_uniform_sphere(rng, out);
        return;
    }
    double axis[3] = {v[0] / d, v[1] / d, v[2] / d};
    double s = R / d;
    double t = 1.0 - s * s;
    double cos_max = sqrt(t > 0.0 ? t : 0.0);
    double u1 = or_next_double(rng), u2 = or_next_double(rng);
    double ct = 1.0 - u1 * (1.0 - cos_max);
    double t2 = 1.0 - ct * ct;
    double st = sqrt(t2 > 0.0 ? t2 : 0.0);
    double phi = OR_TWO_PI * u2;
    double local[3] = {st * cos(phi), st * sin(phi), ct};
    or_from_local_frame(axis, local, out);
}

/* trace_photons, pinned order:
 *   for bounce = 0 .. max_bounces-1:
 *     delta_track (miss -> stop); throughput *= alpha * rgb;
 *     w = hg_sample(g, w, rng);  bounce >= 1 -> deposit {x, w (post-scatter),
 *     I / n_pair * throughput, g_index};  bounce >= rr_start -> roulette with
 *     q = clamp(max throughput, rr_min, rr_max): u >= q stops, else throughput /= q. */
size_t or_trace_photons(const or_medium *m, const or_light *lights, int n_lights, const or_trace_cfg *cfg,
                        or_photon *out, size_t capacity, uint64_t *emitted, int *path_count) {
    const uint64_t pairs = (uint64_t)n_lights * (uint64_t)cfg->n_phases;
    size_t n_out = 0;
    if (pairs == 0) return 0;
    for (uint64_t p = 0; p < pairs; ++p)
        emitted[p] = cfg->n_total / pairs + (p < cfg->n_total % pairs ? 1u : 0u);
    for (uint64_t i = 0; i < cfg->n_total; ++i) {
        const uint64_t pr = i % pairs;
        const int li = (int)(pr / (uint64_t)cfg->n_phases), gi = (int)(pr % (uint64_t)cfg->n_phases);
        const double g = cfg->phase_set[gi];
        or_pcg32 rng;
        or_make_rng(&rng, cfg->seed, OR_STREAM_TRACE, i);
        double o[3] = {lights[li].pos[0], lights[li].pos[1], lights[li].pos[2]}, w[3];
        or_emit_direction(o, &rng, w);
        double thr[3] = {1.0, 1.0, 1.0};
        int deposited = 0;
        for (int bounce = 0; bounce < cfg->max_bounces; ++bounce) {
            double x[3], scal, c[4];
            if (or_delta_track(m, o, w, 0.0, INFINITY, &rng, x, &scal, c) != 1) break;
            for (int k = 0; k < 3; ++k) thr[k] *= c[3] * c[k];
            double nw[3];
            double u1 = or_next_double(&rng), u2 = or_next_double(&rng);
            or_hg_sample(g, w, u1, u2, nw);
            if (bounce >= 1) {
                if (n_out < capacity) {
                    or_photon *ph = &out[n_out];
                    for (int k = 0; k < 3; ++k) {
                        ph->pos[k] = (float)x[k];
                        ph->dir[k] = (float)nw[k];
                        ph->power[k] = (float)(lights[li].intensity[k] / (double)emitted[pr] * thr[k]);
                    }
                    ph->g_index = (uint8_t)gi;
                }
                ++n_out;
                ++deposited;
            }
            if (bounce >= cfg->rr_start_bounce) {
                double q = thr[0] > thr[1] ? thr[0] : thr[1];
                q = thr[2] > q ? thr[2] : q;
                q = q < cfg->rr_min_survival ? cfg->rr_min_survival : (q > cfg->rr_max_survival ? cfg->rr_max_survival : q);
                if (or_next_double(&rng) >= q) break;
                for (int k = 0; k < 3; ++k) thr[k] /= q;
            }
            for (int k = 0; k < 3; ++k) {
                o[k] = x[k];
                w[k] = nw[k];
            }
        }
        if (path_count) path_count[i] = deposited;
    }
    return n_out;
}

/* ===== render_neural ====================================================== */

static void or_normalize(double v[3]) {
    double len = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    v[0] = v[0] / len;
    v[1] = v[1] / len;
    v[2] = v[2] / len;
}

void or_camera_make(or_camera *c, const double pos[3], const double look_at[3],
                    const double up[3], double vfov_deg, int width, int height) {
    double f[3] = {look_at[0] - pos[0], look_at[1] - pos[1], look_at[2] - pos[2]};
    or_normalize(f);
    double r[3] = {f[1] * up[2] - f[2] * up[1], f[2] * up[0] - f[0] * up[2],
                   f[0] * up[1] - f[1] * up[0]};
    or_normalize(r);
    double u[3] = {r[1] * f[2] - r[2] * f[1], r[2] * f[0] - r[0] * f[2], r[0] * f[1] - r[1] * f[0]};
    double th = tan(vfov_deg * (OR_PI / 180.0) * 0.5);
    double aspect = (double)width / (double)height;
    for (int a = 0; a < 3; ++a) {
        c->origin[a] = pos[a];
        c->forward[a] = f[a];
        c->right[a] = r[a] * (aspect * th);
        c->up[a] = u[a] * th;
    }
    c->width = width;
    c->height = height;
}

/* Pinhole ray through film point (px+u, py+v) (pinned App. B.1). */
void or_camera_ray(const or_camera *c, int px, int py, double u, double v, double o[3],
                   double d[3]) {
    double sx = (2.0 * ((double)px + u)) / (double)c->width - 1.0;
    double sy = 1.0 - (2.0 * ((double)py + v)) / (double)c->height;
    for (int a = 0; a < 3; ++a) {
        o[a] = c->origin[a];
        d[a] = (c->forward[a] + c->right[a] * sx) + c->up[a] * sy;
    }
    or_normalize(d);
}

/* One light's NEE term (pinned App. B.3): hg(g, normalize(x-P).w_out) * T / |P-x|^2 * I. */
void or_nee_term(const double x[3], const double w_out[3], const or_light *l, double g,
                 double T, double acc[3]) {
    double dv[3] = {x[0] - l->pos[0], x[1] - l->pos[1], x[2] - l->pos[2]};
    double dist2 = dv[0] * dv[0] + dv[1] * dv[1] + dv[2] * dv[2];
    if (!(dist2 > 0.0) || T == 0.0) return;
    double len = sqrt(dist2);
    double din[3] = {dv[0] / len, dv[1] / len, dv[2] / len};
    double c = din[0] * w_out[0] + din[1] * w_out[1] + din[2] * w_out[2];
    double s = (or_hg_eval(g, c) * T) / dist2;
    for (int ch = 0; ch < 3; ++ch) acc[ch] += s * l->intensity[ch];
}

/* compose term (sigma_s SPEC.md:600): w_d L_d + w_i sigma_s L_i. */
void or_shade_sample(const double Ld[3], const double Li[3], const double rgba[4], double w_d,
                     double w_i, double out[3]) {
    double sigma_s = rgba[3] * ((rgba[0] + rgba[1] + rgba[2]) / 3.0);
    for (int ch = 0; ch < 3; ++ch) out[ch] = w_d * Ld[ch] + w_i * (sigma_s * Li[ch]);
}

/* render_path_traced's continuation (pinned in DESIGN.md):
 * the in-scattered radiance L_i at the first interaction x0, estimated by a
 * phase-sampled path on make_rng(seed, PathTrace, index).  Vertex k >= 1:
 *   w = hg_sample(g, w, rng); x_k = delta_track(x_{k-1}, w) (miss -> stop);
 *   L_d(x_k) = sum_l nee_term(x_k, -w, l, g, transmittance(x_k, P_l, rng, trials));
 *   L_i += thr * L_d(x_k); thr *= sigma_s(x_k) (stop at 0);
 *   k >= rr_start: q = clamp(thr, rr_min, rr_max), next_double() >= q stops, else thr /= q.
 * Point lights cannot be hit by phase sampling, so the balance-heuristic MIS
 * weight of NEE is 1 and escaped continuations carry no radiance. */
static void or_pt_indirect(const or_medium *m, const or_light *lights, int n_lights,
                           const or_render_cfg *rc, const or_pt_cfg *pt, uint64_t index,
                           const double x0[3], const double d0[3], double Li[3]) {
    Li[0] = Li[1] = Li[2] = 0.0;
    if (pt->max_bounces <= 1) return;
    or_pcg32 r;
    or_make_rng(&r, rc->seed, OR_STREAM_PATHTRACE, index);
    double o[3] = {x0[0], x0[1], x0[2]}, w[3] = {d0[0], d0[1], d0[2]};
    double thr = 1.0;
    for (int k = 1; k < pt->max_bounces; ++k) {
        double u1 = or_next_double(&r), u2 = or_next_double(&r), nw[3];
        or_hg_sample(rc->g, w, u1, u2, nw);
        w[0] = nw[0];
        w[1] = nw[1];
        w[2] = nw[2];
        double x[3], scal, rgba[4];
        if (or_delta_track(m, o, w, 0.0, INFINITY, &r, x, &scal, rgba) != 1) break;
        double w_out[3] = {-w[0], -w[1], -w[2]};
        double Ld[3] = {0.0, 0.0, 0.0};
        for (int l = 0; l < n_lights; ++l) {
            double T = or_transmittance(m, x, lights[l].pos, &r, rc->nee_trials);
            or_nee_term(x, w_out, &lights[l], rc->g, T, Ld);
        }
        for (int ch = 0; ch < 3; ++ch) Li[ch] += thr * Ld[ch];
        thr *= rgba[3] * ((rgba[0] + rgba[1] + rgba[2]) / 3.0);
        if (!(thr > 0.0)) break;
        if (k >= pt->rr_start_bounce) {
            double q = thr < pt->rr_min_survival ? pt->rr_min_survival
                                                  : (thr > pt->rr_max_survival ? pt->rr_max_survival : thr);
            if (or_next_double(&r) >= q) break;
            thr /= q;
        }
        o[0] = x[0];
        o[1] = x[1];
        o[2] = x[2];
    }
}

/* render_photon_map's L_i: Eq. 6 over knn_phase at the
 * first interaction, query position rounded to binary32 (App. B.8), omega =
 * w_out in binary64, g = the map's phase value. */
static void or_pm_radiance(const or_pm_src *pm, const double x[3], const double w_out[3], double g,
                           double Li[3]) {
    Li[0] = Li[1] = Li[2] = 0.0;
    if (pm->K <= 0) return;
    uint32_t ids[1024];
    float d2[1024];
    const float q[3] = {(float)x[0], (float)x[1], (float)x[2]};
    int c = pm->tree ? or_kd_knn(pm->tree, q, pm->g_index, pm->K, pm->r_max, ids, d2)
                     : or_knn_brute(pm->ph, pm->n, q, pm->g_index, pm->K, pm->r_max, ids, d2);
    or_estimate_radiance(pm->ph, ids, d2, c, w_out, g, Li);
}

/* The shared per-sample program of the three first-interaction renderers:
 * camera jitter + delta_track on CameraSample, NEE on the Nee stream, then
 * L_i from the field (neural), a continued path (path traced) or the photon
 * map, composed as w_d L_d + w_i sigma_s L_i. */
static void or_render_impl(const or_medium *m, const or_light *lights, int n_lights,
                           const or_camera *cam, const or_render_cfg *rc, const or_field_cfg *fc,
                           const float *params, const or_pt_cfg *pt, const or_pm_src *pm,
                           float *out_rgb, or_render_stats *st) {
    const int W = cam->width, spp = rc->spp;
    for (int py = rc->y0; py < rc->y1; ++py) {
        for (int px = rc->x0; px < rc->x1; ++px) {
            double acc[3] = {0.0, 0.0, 0.0};
            for (int s = 0; s < spp; ++s) {
                uint64_t index = ((uint64_t)py * (uint64_t)W + (uint64_t)px) * (uint64_t)spp + s;
                or_pcg32 rng;
                or_make_rng(&rng, rc->seed, OR_STREAM_CAMERA, index);
                double u = or_next_double(&rng);
                double v = or_next_double(&rng);
                double o[3], d[3], x[3], scal, rgba[4];
                or_camera_ray(cam, px, py, u, v, o, d);
                double sample[3];
                int hit = or_delta_track(m, o, d, 0.0, INFINITY, &rng, x, &scal, rgba);
                if (st) st->samples++;
                if (hit != 1) {
                    for (int ch = 0; ch < 3; ++ch) sample[ch] = rc->background[ch];
                } else {
                    if (st) st->hits++;
                    double w_out[3] = {-d[0], -d[1], -d[2]};
                    double Ld[3] = {0.0, 0.0, 0.0}, Li[3] = {0.0, 0.0, 0.0};
                    or_pcg32 nee;
                    or_make_rng(&nee, rc->seed, OR_STREAM_NEE, index);
                    for (int l = 0; l < n_lights; ++l) {
                        double T = or_transmittance(m, x, lights[l].pos, &nee, rc->nee_trials);
                        or_nee_term(x, w_out, &lights[l], rc->g, T, Ld);
                    }
                    if (pt) {
                        or_pt_indirect(m, lights, n_lights, rc, pt, index, x, d, Li);
                    } else if (pm) {
                        or_pm_radiance(pm, x, w_out, rc->g, Li);
                    } else if (rc->use_field) {
                        double sph[2];
                        or_dir_to_sph(w_out, sph);
                        or_field_infer(fc, params, 1, x, sph, &rc->g, Li);
                    }
                    or_shade_sample(Ld, Li, rgba, rc->w_d, rc->w_i, sample);
                }
                for (int ch = 0; ch < 3; ++ch) acc[ch] += sample[ch];
            }
            float *o3 = out_rgb + 3 * ((size_t)py * W + px);
            for (int ch = 0; ch < 3; ++ch) o3[ch] = (float)(acc[ch] / (double)spp);
        }
    }
}

void or_render_neural(const or_medium *m, const or_light *lights, int n_lights,
                      const or_field_cfg *fc, const float *params, const or_camera *cam,
                      const or_render_cfg *rc, float *out_rgb, or_render_stats *st) {
    or_render_impl(m, lights, n_lights, cam, rc, fc, params, NULL, NULL, out_rgb, st);
}

void or_render_path_traced(const or_medium *m, const or_light *lights, int n_lights,
                           const or_camera *cam, const or_render_cfg *rc, const or_pt_cfg *pt,
                           float *out_rgb, or_render_stats *st) {
    or_render_impl(m, lights, n_lights, cam, rc, NULL, NULL, pt, NULL, out_rgb, st);
}

void or_render_photon_map(const or_medium *m, const or_light *lights, int n_lights,
                          const or_pm_src *pm, const or_camera *cam, const or_render_cfg *rc,
                          float *out_rgb, or_render_stats *st) {
    or_render_impl(m, lights, n_lights, cam, rc, NULL, NULL, NULL, pm, out_rgb, st);
}
