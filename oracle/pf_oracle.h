/*
 * pf_oracle.h -- CPU ORACLE for the photon-field render hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing under oracle/ is part of the product:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load it, and only as the checker (or the timed
 * CPU arm).  The product path (paper_2304_07338_b200/) never links it.
 *
 * This is a plain-C restatement of the reference algorithm
 * (/root/reference/proj, arXiv 2304.07338 "Photon Field Networks"):
 *   - parts (a)/(b) restate proj/include/pf/{rng,math,phase}.hpp and
 *     proj/src/volume.cpp line by line (same operation order, same RNG
 *     consumption; compile with -ffp-contract=off).  They are PINNED against
 *     the reference itself: oracle/_ref/libpfref.so is compiled from the
 *     unmodified reference sources and tests/test_oracle_ref.py checks the
 *     two bit-for-bit.
 *   - part (c), the KNN gather, Eq. 6/7/8, compose and render_neural have no
 *     reference code; they restate SPEC.md:221-617 with the ambiguities pinned
 *     as in SURVEY.md Appendix B.  For those
 *     the SPEC known-answer examples are the golden vectors; field/KNN/render
 *     goldens beyond them are "parity unpinned" w.r.t. the reference (there is
 *     no reference code to run) and are self-consistency goldens.
 */
#ifndef PF_ORACLE_H
#define PF_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- rng: proj/include/pf/rng.hpp:14-83 --------------------------------- */
typedef struct {
    uint64_t state;
    uint64_t inc;
} or_pcg32;

enum {
    OR_STREAM_TRACE = 1, OR_STREAM_TRAIN = 2, OR_STREAM_CAMERA = 3, OR_STREAM_NEE = 4,
    OR_STREAM_PATHTRACE = 5, OR_STREAM_FIELDINIT = 6, OR_STREAM_SYNTH = 7, OR_STREAM_TEST = 8
};

void or_pcg_seed(or_pcg32 *r, uint64_t initstate, uint64_t initseq);
uint32_t or_next_u32(or_pcg32 *r);
uint64_t or_next_u64(or_pcg32 *r);
double or_next_double(or_pcg32 *r);
uint32_t or_next_below(or_pcg32 *r, uint32_t n);
uint64_t or_splitmix64(uint64_t x);
void or_make_rng(or_pcg32 *r, uint64_t seed, uint64_t stream, uint64_t index);
void or_sample_uniform_sphere(or_pcg32 *r, double out[3]);

/* ---- math / phase: proj/include/pf/math.hpp:95-108, phase.hpp:18-23 ------ */
int or_aabb_intersect(const double o[3], const double d[3], double tmin, double tmax,
                      double *t0, double *t1);
double or_hg_eval(double g, double cos_theta);

/* ---- volume: proj/src/volume.cpp ------------------------------------------ */
typedef struct {
    int nx, ny, nz;
    const float *data; /* x-fastest */
    float value_min, value_max;
} or_grid;

typedef struct {
    int n;
    const double *pts; /* n x 5: scalar, r, g, b, a */
} or_tf;

typedef struct {
    or_grid grid;
    or_tf tf;
    double density_scale;
    double sigma_max;
} or_medium;

/* VolumeGrid ctor validation + value range (volume.cpp:24-39).  0 ok, 1 invalid. */
int or_grid_init(or_grid *g, int nx, int ny, int nz, const float *data);
double or_grid_sample(const or_grid *g, const double p[3]);
void or_tf_classify(const or_tf *tf, double scalar, double rgba[4]);
double or_tf_max_alpha(const or_tf *tf, double lo, double hi);
/* Medium ctor (volume.cpp:197-202).  0 ok, 1 invalid density scale. */
int or_medium_init(or_medium *m, const or_grid *g, const or_tf *tf, double density_scale);

/* delta_track (volume.cpp:204-225): 1 = interaction (pos/scalar/rgba set),
 * 0 = absent, -1 = invalid ray (reference throws std::invalid_argument). */
int or_delta_track(const or_medium *m, const double o[3], const double d[3], double tmin,
                   double tmax, or_pcg32 *rng, double pos[3], double *scalar, double rgba[4]);
/* transmittance (volume.cpp:227-256): fraction of n_trials delta flights that
 * pass; -1.0 when n_trials <= 0 (reference throws). */
double or_transmittance(const or_medium *m, const double a[3], const double b[3], or_pcg32 *rng,
                        int n_trials);

/* Batched conveniences for the test harness: ray i uses make_rng(seed, stream, idx[i]). */
int or_delta_track_batch(const or_medium *m, size_t n, const double *o3, const double *d3,
                         const double *tmin, const double *tmax, uint64_t seed, uint64_t stream,
                         const uint64_t *idx, int *hit, double *pos3, double *scalar1, double *rgba4);
void or_transmittance_batch(const or_medium *m, size_t n, const double *a3, const double *b3,
                            uint64_t seed, uint64_t stream, const uint64_t *idx, int n_trials,
                            double *out);
void or_rng_doubles(uint64_t seed, uint64_t stream, size_t n, const uint64_t *idx, int draws,
                    double *out);

/* ---- neural field: SPEC.md:352-447 (no reference code) -------------------- */
typedef struct {
    int dims;          /* 3 (position) or 2 (direction) */
    int levels;        /* L */
    int features;      /* F */
    int base_res;      /* N_0 */
    double growth;     /* b */
    int log2_table;    /* log2 T */
} or_hashgrid_cfg;

typedef struct {
    or_hashgrid_cfg pos, dir;
    int hidden_layers; /* 5 */
    int width;         /* 64 */
    double psi;        /* Eq. 7/8 precision, 5 */
} or_field_cfg;

/* Resolution / table size of level l (pinned). */
int or_hashgrid_level_res(const or_hashgrid_cfg *c, int l);
uint32_t or_hashgrid_level_size(const or_hashgrid_cfg *c, int l);
size_t or_hashgrid_param_count(const or_hashgrid_cfg *c);
int or_field_input_dim(const or_field_cfg *c);
size_t or_field_param_count(const or_field_cfg *c);
/* Deterministic init, draw order of pf_field_init. */
void or_field_init(const or_field_cfg *c, uint64_t seed, double embed_scale, double bias_scale,
                   float *out);
/* encode_input -> D_in doubles. */
void or_field_encode(const or_field_cfg *c, const float *params, const double x[3],
                     const double wsph[2], double g, double *feat);
/* forward: log-space outputs L' (no clamp). */
void or_field_forward(const or_field_cfg *c, const float *params, size_t n, const double *x3,
                      const double *w2, const double *g, double *out3);
/* infer_radiance = decode_log(forward). */
void or_field_infer(const or_field_cfg *c, const float *params, size_t n, const double *x3,
                    const double *w2, const double *g, double *out3);
/* Direction -> normalized spherical coordinates. */
void or_dir_to_sph(const double w[3], double out[2]);

/* ---- training: binary64 parameters ---------------------- */
typedef struct {
    double lr;           /* 9e-4 */
    double beta1, beta2; /* 0.9, 0.99 */
    double eps;          /* 1e-8 */
    double decay;        /* 0.92 */
    double decay_start;  /* 0.7 of total steps */
    int decay_interval;  /* 25 */
} or_adam_cfg;
double or_lr_at(const or_adam_cfg *a, uint64_t step, uint64_t total);
/* rMSE loss = mean over batch x channels of (p - t)^2 / (p_detached^2 + eps_rel);
 * grad (may be NULL) = dense d loss / d params; touched[entry] flags table
 * entries (pos entries first, then dir) that received a contribution.
 * pred_out (may be NULL) receives the predictions; den_in (may be NULL)
 * replaces p_detached^2 + eps_rel (frozen denominators for finite differences). */
double or_train_grad(const or_field_cfg *c, const double *params, size_t n, const double *x3, const double *w2,
                     const double *g, const double *targets3, double eps_rel, double *grad,
                     uint8_t *touched, double *pred_out, const double *den_in);
void or_adam_update(const or_field_cfg *c, const or_adam_cfg *a, double *params, const double *grad,
                    const uint8_t *touched, double *m, double *v, uint64_t step, uint64_t total);

/* ---- estimator: SPEC.md:282-350 ------------------------------------------- */
double or_encode_log(double L, double psi);
double or_decode_log(double Lp, double psi);

/* ---- photon map / KNN: SPEC.md:221-280, photon.hpp:17-22 ------------------ */
typedef struct {
    float pos[3];
    float dir[3];
    float power[3];
    uint8_t g_index;
} or_photon; /* SoA on the GPU; this AoS mirrors pf::Photon (40 B in memory) */

/* Brute-force phase-selective KNN (the SPEC's own oracle):
 * min(K, m) photons with tag == g and d2 <= r_max2, ascending (d2, id).
 * d2 = ((dx*dx)+(dy*dy))+(dz*dz) in binary32, dx = photon - query.
 * Returns count; ids/d2 arrays must hold K entries. */
int or_knn_brute(const or_photon *ph, size_t n, const float q[3], int g_index, int K,
                 float r_max, uint32_t *ids, float *d2);

/* Balanced median-split kd-tree. */
typedef struct or_kdtree or_kdtree;
or_kdtree *or_kd_build(const or_photon *ph, size_t n);
void or_kd_free(or_kdtree *t);
int or_kd_knn(const or_kdtree *t, const float q[3], int g_index, int K, float r_max,
              uint32_t *ids, float *d2);

/* Eq. 6 on a sorted neighbour list; rgb out. */
void or_estimate_radiance(const or_photon *ph, const uint32_t *ids, const float *d2, int count,
                          const double w[3], double g, double out[3]);

/* make_batch query generation (pinned App. B): per sample i
 * rng = make_rng(seed, Train, step*batch + i); x ~ U^3, w ~ sphere, g ~ U(G). */
void or_make_queries(uint64_t seed, uint64_t step, size_t batch, int n_phases, float *x3,
                     double *w3, uint8_t *gidx);
/* schedule_radius. */
double or_schedule_radius(const double *ends, const double *radii, int n, uint64_t step,
                          uint64_t total);
/* Full target gather: KNN (kd-tree) -> Eq. 6 -> Eq. 7 for every query. */
void or_knn_targets(const or_kdtree *t, const or_photon *ph, size_t nq, const float *x3,
                    const double *w3, const uint8_t *gidx, const double *phase_set, int K,
                    float r_max, double psi, uint32_t *ids, float *d2, int *counts,
                    double *targets3);

/* ---- photon tracing: Alg. 1, SPEC.md:151-219 ----------- */
/* phase.hpp:26-46 + math.hpp:113-126 (checked bit-for-bit against the reference). */
double or_hg_sample_cos(double g, double u);
void or_hg_sample(double g, const double w_in[3], double u1, double u2, double out[3]);
void or_from_local_frame(const double axis[3], const double local[3], double out[3]);

typedef struct {
    double pos[3];
    double intensity[3];
} or_light;

typedef struct {
    uint64_t n_total;
    int n_phases;
    const double *phase_set;
    int max_bounces;
    int rr_start_bounce;
    double rr_min_survival, rr_max_survival;
    uint64_t seed;
} or_trace_cfg;

/* emit_direction (photon.hpp:50, pinned in DESIGN.md). */
void or_emit_direction(const double light_pos[3], or_pcg32 *rng, double out[3]);
/* trace_photons: photon i -> pair p = i % (nL*nG), light p / nG, phase p % nG,
 * rng = make_rng(seed, Trace, i); deposits in (i, bounce) order.  Returns the
 * number of records (<= capacity); emitted[nL*nG]; path_count[i] optional. */
size_t or_trace_photons(const or_medium *m, const or_light *lights, int n_lights, const or_trace_cfg *cfg,
                        or_photon *out, size_t capacity, uint64_t *emitted, int *path_count);

/* ---- render_neural (Alg. 2) ------------- */
typedef struct {
    double origin[3];
    double forward[3]; /* unit */
    double right[3];   /* unit right * aspect * tan(fov/2) */
    double up[3];      /* unit up * tan(fov/2) */
    int width, height;
} or_camera;

/* Host-side camera basis (pinned App. B.1).  Everything per-sample is in
 * or_camera_ray so the GPU reproduces it bit-for-bit. */
void or_camera_make(or_camera *c, const double pos[3], const double look_at[3],
                    const double up[3], double vfov_deg, int width, int height);
void or_camera_ray(const or_camera *c, int px, int py, double u, double v, double o[3],
                   double d[3]);

typedef struct {
    int spp;
    double g;
    uint64_t seed;
    double w_d, w_i;
    double background[3];
    int nee_trials;     /* reference-mode transmittance trials (1) */
    int use_field;      /* 0: L_i = 0 */
    /* pixel rectangle [x0,x1) x [y0,y1) rendered (others untouched) */
    int x0, y0, x1, y1;
} or_render_cfg;

typedef struct {
    uint64_t samples, hits;
} or_render_stats;

/* Single-sample pieces shared with the reference-driven CPU arm. */
void or_nee_term(const double x[3], const double w_out[3], const or_light *l, double g,
                 double T, double acc[3]);
void or_shade_sample(const double Ld[3], const double Li[3], const double rgba[4], double w_d,
                     double w_i, double out[3]);

void or_render_neural(const or_medium *m, const or_light *lights, int n_lights,
                      const or_field_cfg *fc, const float *params, const or_camera *cam,
                      const or_render_cfg *rc, float *out_rgb, or_render_stats *st);

/* ---- render_path_traced -------------------------------- */
typedef struct {
    int max_bounces;      /* path vertices incl. the first interaction (default 16) */
    int rr_start_bounce;  /* roulette from this vertex on (default 3) */
    double rr_min_survival, rr_max_survival; /* 0.05, 0.95 */
} or_pt_cfg;
/* Identical to render_neural up to and including the first interaction's NEE
 * (same CameraSample / Nee streams); L_i from a phase-sampled continuation on
 * make_rng(seed, PathTrace, index) (pinned in pf_oracle.c or_pt_indirect). */
void or_render_path_traced(const or_medium *m, const or_light *lights, int n_lights,
                           const or_camera *cam, const or_render_cfg *rc, const or_pt_cfg *pt,
                           float *out_rgb, or_render_stats *st);

/* ---- render_photon_map --------------------------------- */
typedef struct {
    const or_photon *ph;
    size_t n;
    const or_kdtree *tree; /* NULL: brute force */
    int g_index;           /* the render g's index in the map's phase set */
    int K;                 /* <= 1024 */
    float r_max;
} or_pm_src;
void or_render_photon_map(const or_medium *m, const or_light *lights, int n_lights,
                          const or_pm_src *pm, const or_camera *cam, const or_render_cfg *rc,
                          float *out_rgb, or_render_stats *st);

#ifdef __cplusplus
}
#endif
#endif
