/*
 * pf_gpu.h -- C ABI of the B200-native photon-field render hot path.
 *
 * The reference (arXiv 2304.07338, /root/reference/proj) is a C++20 library in
 * namespace pf with no device or process boundary.  This header is the thin
 * extern "C" layer a drop-in replacement exports so that the reference-side
 * C++ API (include/pf/gpu.hpp) -- or any FFI (ctypes, cgo, JNI) -- can reach
 * the sm_100a kernels.  Plain pointers and sizes only; no torch / CUDA types.
 *
 * Pointer arguments: every array argument may be a HOST pointer (staged
 * through the context with cudaMemcpyAsync on the context stream) or a DEVICE
 * pointer on the context's GPU (used in place).  The kind is detected with
 * cudaPointerGetAttributes per call.
 *
 * Errors: every int-returning entry point returns PF_OK (0),
 * PF_ERR_INVALID (1, the reference throws std::invalid_argument) or
 * PF_ERR_RUNTIME (2, std::runtime_error / CUDA / NCCL failure); the message
 * is in pf_last_error() (thread-local).  include/pf/gpu.hpp rethrows the
 * matching C++ exception type.
 *
 * Randomness: all device randomness is the reference's PCG32
 * (proj/include/pf/rng.hpp:14-76) with make_rng(seed, stream, index) streams,
 * so results never depend on launch geometry, tiling or GPU count.
 */
#ifndef PF_GPU_H
#define PF_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PF_OK 0
#define PF_ERR_INVALID 1
#define PF_ERR_RUNTIME 2

/* pf::Stream, proj/include/pf/rng.hpp:62-71 */
#define PF_STREAM_TRACE 1
#define PF_STREAM_TRAIN 2
#define PF_STREAM_CAMERA 3
#define PF_STREAM_NEE 4
#define PF_STREAM_PATHTRACE 5
#define PF_STREAM_FIELDINIT 6
#define PF_STREAM_SYNTH 7
#define PF_STREAM_TEST 8

/* Render modes.
 * PARITY: binary64 delta tracking with the reference's exact operation order
 *   and RNG consumption; NEE transmittance = nee_trials delta-tracked flights
 *   exactly as pf::transmittance (proj/src/volume.cpp:227-256).
 * FAST:   binary32 delta tracking against per-macro-cell majorants (DDA walk
 *   over PF_MACRO^3-voxel cells; empty space skipped) and ratio-tracked
 *   shadow rays with Russian roulette; unbiased, statistically equal to
 *   PARITY (same per-sample streams, consumed differently). */
#define PF_MODE_PARITY 0
#define PF_MODE_FAST 1

typedef struct pf_ctx pf_ctx;

/* Hash-grid encoding (HashGridConfig). */
typedef struct {
    int dims;       /* 3 = position, 2 = direction */
    int levels;     /* paper 16, desk 8 */
    int features;   /* paper 8, desk 4 (must be 2, 4 or 8) */
    int base_res;   /* 4 */
    double growth;  /* 2.0 */
    int log2_table; /* paper 19, desk 15 */
} pf_hashgrid_desc;

/* PhotonField = pos grid + dir grid + MLP. */
typedef struct {
    pf_hashgrid_desc pos, dir;
    int hidden_layers; /* 5 */
    int width;         /* 64 (the only width the tcgen05 kernel supports) */
    double psi;        /* Eq. 7/8 precision (5) */
} pf_field_desc;

/* Pinhole camera: film point (px+u, py+v) maps to
 * normalize((forward + right*sx) + up*sy), sx = 2(px+u)/W - 1,
 * sy = 1 - 2(py+v)/H; right/up carry aspect*tan(fov/2) / tan(fov/2). */
typedef struct {
    double origin[3];
    double forward[3];
    double right[3];
    double up[3];
    int width, height;
} pf_camera;

typedef struct {
    int spp;               /* samples per pixel, >= 1 */
    double g;              /* scene phase coefficient */
    uint64_t seed;         /* config seed: make_rng(seed, CameraSample|Nee, index) */
    double w_d, w_i;       /* compose weights */
    double background[3];  /* radiance of samples that never interact */
    int mode;              /* PF_MODE_PARITY | PF_MODE_FAST */
    int nee_trials;        /* parity-mode transmittance trials (>= 1) */
    int use_field;         /* 0: L_i = 0 (direct light only) */
    int tile_w, tile_h;    /* screen tiles (multi-GPU sharding unit), e.g. 16 x 16 */
    int shard_index;       /* this rank renders tiles t with t % shard_count == shard_index */
    int shard_count;       /* 1 on a single GPU */
} pf_render_desc;

typedef struct {
    uint64_t samples;        /* camera samples traced */
    uint64_t hits;           /* samples with a real interaction (= field queries) */
    uint64_t primary_steps;  /* tentative collisions, primary rays */
    uint64_t shadow_steps;   /* tentative collisions, shadow rays */
    float ms_trace, ms_field, ms_compose; /* device time per stage (0 unless timing on) */
    uint32_t kernel_launches;              /* device kernels this call launched */
    uint64_t voxel_fetches;  /* sigma(x) evaluations actually issued (PARITY: tentative
                                collisions not settled by the majorant-texture bound) */
} pf_render_stats;

/* Photon record, pf::Photon (proj/include/pf/photon.hpp:17-22): 40 bytes. */
typedef struct {
    float position[3];
    float direction[3];
    float power[3];
    uint8_t g_index;
    uint8_t pad_[3];
} pf_photon;

const char *pf_last_error(void);
const char *pf_version(void);

/* Context on one CUDA device (one process per GPU). */
int pf_ctx_create(int device, pf_ctx **out);
void pf_ctx_destroy(pf_ctx *ctx);
/* Use an external cudaStream_t (e.g. torch's current stream); NULL = own stream. */
int pf_ctx_set_stream(pf_ctx *ctx, void *cuda_stream);
int pf_ctx_synchronize(pf_ctx *ctx);
/* Enable per-stage CUDA-event timing inside pf_render_neural. */
int pf_ctx_set_timing(pf_ctx *ctx, int enabled);

/* ---- scene (replicated per GPU) ----------------------------------------- */
/* VolumeGrid(nx, ny, nz, data) (volume.hpp:25; validation volume.cpp:24-39):
 * x-fastest binary32 scalars in [0,1]. */
int pf_volume_upload(pf_ctx *ctx, int nx, int ny, int nz, const float *data);
/* Medium(grid, tf, density_scale) (volume.hpp:94): tf_pts = n x (s,r,g,b,a)
 * with TransferFunction's invariants (volume.cpp:136-149).  sigma_max < 0
 * computes density_scale * tf.max_alpha(grid range) like volume.cpp:197-202;
 * otherwise the caller's pf::Medium::sigma_max() is used bit-for-bit. */
int pf_medium_set(pf_ctx *ctx, const double *tf_pts, int n_pts, double density_scale,
                  double sigma_max);
int pf_medium_sigma_max(pf_ctx *ctx, double *out);
/* LightSource list (photon.hpp:24-27): n x (px,py,pz, Ir,Ig,Ib). */
int pf_lights_set(pf_ctx *ctx, const double *lights, int n);

/* ---- photon field (part c) ---------------------------------------------- */
int pf_field_param_count(const pf_field_desc *desc, size_t *out);
/* Deterministic init from make_rng(seed, FieldInit, 0), drawn in parameter
 * order: tables U(-embed_scale, embed_scale), weights U(+-sqrt(6/fan_in)),
 * biases U(-bias_scale, bias_scale).  Host-only helper. */
int pf_field_init(const pf_field_desc *desc, uint64_t seed, double embed_scale,
                  double bias_scale, float *params_out);
/* Flat parameter vector (layout: DESIGN.md "Field parameters"). */
int pf_field_load(pf_ctx *ctx, const pf_field_desc *desc, const float *params, size_t n);
/* Batched forward: x3 in [0,1]^3, w_sph2 = (theta/pi,
 * (phi+pi)/2pi), g raw in [-1,1].  decoded = 0 -> L' (forward), 1 -> radiance
 * (infer_radiance = decode_log(forward)). */
int pf_field_query(pf_ctx *ctx, size_t n, const float *x3, const float *w_sph2, const float *g,
                   float *out_rgb, int decoded);

/* ---- render_neural (Alg. 2) ---------------------------- */
int pf_camera_make(const double pos[3], const double look_at[3], const double up[3],
                   double vfov_deg, int width, int height, pf_camera *out);
/* Renders this shard's tiles into out_rgb (width*height*3 binary32, row-major);
 * pixels of other shards are left untouched.  stats may be NULL. */
int pf_render_neural(pf_ctx *ctx, const pf_camera *cam, const pf_render_desc *desc,
                     float *out_rgb, pf_render_stats *stats);
/* Pipelined frames into HOST memory: enqueue the frame and return at once; the
 * device->host copy of out_rgb (pinned memory for real overlap) runs on the
 * context's copy stream while the next frame's kernels run (two frames in
 * flight, double-buffered device staging).  out_rgb is complete after
 * pf_frame_wait(ctx, out_rgb) or pf_ctx_synchronize. */
int pf_render_neural_async(pf_ctx *ctx, const pf_camera *cam, const pf_render_desc *desc, float *host_out);
int pf_frame_wait(pf_ctx *ctx, const float *host_out);

/* ---- the comparison renderers of SPEC.md render module ------------------ */
/* render_path_traced(scene, camera, spp, max_bounces, rng):
 * the volumetric path tracer with NEE at every vertex, HG-sampled
 * continuation and Russian roulette (pinned: oracle or_render_path_traced).
 * Identical to pf_render_neural up to the first interaction's NEE (same
 * CameraSample / Nee streams); the continuation runs on make_rng(seed,
 * PathTrace, index).  desc->use_field is ignored. */
typedef struct {
    int max_bounces;         /* path vertices incl. the first interaction, >= 1 (16) */
    int rr_start_bounce;     /* roulette from this vertex on (3) */
    double rr_min_survival;  /* 0.05 */
    double rr_max_survival;  /* 0.95 */
} pf_path_desc;
int pf_render_path_traced(pf_ctx *ctx, const pf_camera *cam, const pf_render_desc *desc,
                          const pf_path_desc *path, float *out_rgb, pf_render_stats *stats);
/* render_photon_map(scene, map, camera, spp, K, r_max, g, rng):
 * render_neural with L_i = Eq. 6 over knn_phase of the resident photon map
 * (pf_knn_build / pf_knn_build_traced) at each first interaction (query =
 * position as binary32, omega = -ray direction).  desc->g must be one of the
 * map's phase values (else PF_ERR_INVALID, "g not in the map's phase set");
 * K in [1, 1024], r_max > 0.  desc->use_field is ignored. */
int pf_render_photon_map(pf_ctx *ctx, const pf_camera *cam, const pf_render_desc *desc, int K,
                         float r_max, float *out_rgb, pf_render_stats *stats);

/* Multi-GPU helpers: pack this shard's tiles contiguously (tile order) and
 * unpack all shards' packed buffers into a frame. */
int pf_tiles_count(const pf_camera *cam, const pf_render_desc *desc, int shard, int *n_tiles);
int pf_tiles_pack(pf_ctx *ctx, const pf_camera *cam, const pf_render_desc *desc,
                  const float *frame_rgb, float *packed);
int pf_tiles_unpack(pf_ctx *ctx, const pf_camera *cam, const pf_render_desc *desc,
                    const float *packed_all, size_t per_shard_floats, float *frame_rgb);

/* Tile gather over NVLink peer memory (CUDA IPC), the fused alternative to
 * pack -> all_gather -> unpack: rank 0 allocates the frame and exports a
 * 64-byte handle; every other rank maps it and passes the mapped pointer as
 * out_rgb to pf_render_*, so its compose kernel stores its tiles straight
 * into rank 0's frame.  A stream-ordered barrier (e.g. a 1-element NCCL
 * all-reduce) after the render makes the frame complete on rank 0. */
int pf_ipc_frame_create(pf_ctx *ctx, size_t bytes, void **dev_ptr, void *handle64);
int pf_ipc_frame_open(pf_ctx *ctx, const void *handle64, void **dev_ptr);
/* owner = 1 frees the allocation, 0 unmaps a peer mapping. */
int pf_ipc_frame_release(pf_ctx *ctx, void *dev_ptr, int owner);

/* ---- parity entry points: batched pf::delta_track / pf::transmittance --- */
/* Ray i: origin o3[3i..], unit direction d3[3i..], [tmin, tmax]; its RNG is
 * make_rng(seed, stream, idx[i]).  hit[i] = 1/0; pos3 / scalar1 / rgba4 (each
 * may be NULL) receive Interaction{position, scalar, albedo} (volume.hpp:82-86,
 * volume.cpp:223).  fp64 = 1: binary64 parity kernel; 0: binary32 fast kernel.
 * Invalid rays -> PF_ERR_INVALID (volume.cpp:205-207).
 * Replaces std::optional<Interaction> pf::delta_track(const Medium&, const Ray&,
 * Pcg32&) (proj/include/pf/volume.hpp:115), one call per ray batch. */
int pf_delta_track_batch(pf_ctx *ctx, size_t n, const double *o3, const double *d3,
                         const double *tmin, const double *tmax, uint64_t seed, uint64_t stream,
                         const uint64_t *idx, int fp64, int *hit, double *pos3, double *scalar1,
                         double *rgba4);
/* transmittance(medium, a, b, rng, n_trials) per segment (binary64). */
int pf_transmittance_batch(pf_ctx *ctx, size_t n, const double *a3, const double *b3,
                           uint64_t seed, uint64_t stream, const uint64_t *idx, int n_trials,
                           double *out);
/* Ratio-tracking transmittance (fast mode estimator, binary32): unbiased
 * estimate of the same quantity; n_trials estimates averaged. */
int pf_transmittance_ratio_batch(pf_ctx *ctx, size_t n, const double *a3, const double *b3,
                                 uint64_t seed, uint64_t stream, const uint64_t *idx,
                                 int n_trials, double *out);
/* Device PCG32: draws next_double() n_draws times from make_rng(seed,
 * stream, idx[i]) into out[i*n_draws + k] (rng.hpp:41). */
int pf_rng_doubles(pf_ctx *ctx, size_t n, uint64_t seed, uint64_t stream, const uint64_t *idx,
                   int n_draws, double *out);

/* ---- photon tracing: Alg. 1 (photon.hpp:29-57) ---------- */
/* pf::TraceConfig (photon.hpp:29-37). */
typedef struct {
    uint64_t n_total;         /* photons emitted, split over (light, phase) pairs */
    int n_phases;             /* |G| (1..8) */
    const double *phase_set;  /* G, distinct values in [-1, 1] */
    int max_bounces;          /* default 16 */
    int rr_start_bounce;      /* default 3 */
    double rr_min_survival;   /* default 0.05 */
    double rr_max_survival;   /* default 0.95 */
    uint64_t seed;
} pf_trace_desc;
/* trace_photons(medium, lights, cfg) (photon.hpp:56; declared there, pinned in
 * oracle/pf_oracle.c or_trace_photons): binary64 on the device over the
 * context's medium + lights.  Photon i uses make_rng(seed, Trace, i), pair
 * i % (nL*nG); records are in (photon index, bounce) order, identical to the
 * oracle up to last-ulp libm differences.  The map stays resident in ctx;
 * n_photons = deposits; emitted (optional, nL*nG) = TraceResult::emitted_per_pair.
 * Zero lights / empty or invalid G -> PF_ERR_INVALID (std::invalid_argument). */
int pf_trace_photons(pf_ctx *ctx, const pf_trace_desc *desc, size_t *n_photons, uint64_t *emitted);
/* Copy the resident trace (n must equal n_photons) to host or device memory. */
int pf_trace_fetch(pf_ctx *ctx, pf_photon *out, size_t n);
/* Deposits per emitted photon (n_total entries), host or device memory. */
int pf_trace_path_counts(pf_ctx *ctx, uint32_t *out, uint64_t n_total);
/* Kernel times of the last trace (needs pf_ctx_set_timing) + tentative collisions. */
int pf_trace_stats(pf_ctx *ctx, double *ms_trace, double *ms_compact, uint64_t *tentative_collisions);
/* pf_knn_build straight from the resident trace (no host round trip). */
int pf_knn_build_traced(pf_ctx *ctx, int n_phases, const double *phase_set);

/* ---- photon map + KNN training-target gather (config 3) ----------------- */
/* build(photons): per-phase cell grid, ids = load order. */
int pf_knn_build(pf_ctx *ctx, const pf_photon *photons, size_t n, int n_phases,
                 const double *phase_set);
/* knn_phase: exact min(K, m) nearest photons of tag gidx[i]
 * with d2 <= r_max^2, ascending (d2, id); ids/d2 are nq x K (unused slots:
 * id 0xFFFFFFFF, d2 +inf); counts[i] = min(K, m).  Bit-exact with the oracle. */
int pf_knn_query(pf_ctx *ctx, size_t nq, const float *x3, const uint8_t *gidx, int K,
                 float r_max, uint32_t *ids, float *d2, int32_t *counts);
/* make_batch target gather: KNN -> Eq. 6 (binary64) -> Eq. 7, out3 = log
 * targets in [0,1] (binary64).  ids/d2/counts may be NULL. */
int pf_knn_targets(pf_ctx *ctx, size_t nq, const float *x3, const double *w3,
                   const uint8_t *gidx, int K, float r_max, double psi, double *out3,
                   uint32_t *ids, float *d2, int32_t *counts);
/* Whole make_batch on device: queries from
 * make_rng(seed, Train, step*batch + i) (x ~ U^3 as f32, w ~ uniform sphere,
 * g ~ next_below(n_phases)), then the target gather. */
int pf_make_batch(pf_ctx *ctx, uint64_t seed, uint64_t step, size_t batch, int K, float r_max,
                  double psi, float *x3, double *w3, uint8_t *gidx, double *targets3);

/* ---- photon-field training ------------------- */
/* AdamState + the rMSE epsilon of train_step. */
typedef struct {
    double lr;            /* 9e-4 */
    double beta1, beta2;  /* 0.9, 0.99 */
    double eps;           /* 1e-8 */
    double decay;         /* 0.92 every decay_interval steps ... */
    double decay_start;   /* ... after this fraction of total_steps (0.7) */
    int decay_interval;   /* 25 */
    double eps_rel;       /* relative-MSE epsilon, 0.01 */
} pf_adam_desc;
/* Optimizer state over a flat parameter vector (layout as pf_field_load,
 * which it also performs); adam NULL = the SPEC defaults.  Master parameters
 * and moments are binary32 on the device. */
int pf_train_init(pf_ctx *ctx, const pf_field_desc *desc, const float *params, size_t n,
                  const pf_adam_desc *adam);
/* train_step(field, batch, targets, adam): x3 in [0,1]^3,
 * w_sph2 = (theta/pi, (phi+pi)/2pi), g raw, targets3 in L' space.  loss =
 * mean over batch x channels of (p - t)^2 / (p_detached^2 + eps_rel), returned
 * pre-update; full backward through MLP + hash-grid interpolation, sparse
 * (touched-entry) Adam on the tables, dense on the MLP, lr(step, total).
 * Every reduction has a fixed order: a step is bit-reproducible. */
int pf_train_step(pf_ctx *ctx, size_t n, const float *x3, const float *w_sph2, const float *g,
                  const float *targets3, uint64_t step, uint64_t total_steps, double *loss);
/* Parity entry: loss + dense gradient (n_params floats, may be NULL) + per
 * table-entry touched flags (pos entries then dir, may be NULL); no update. */
int pf_train_grad(pf_ctx *ctx, size_t n, const float *x3, const float *w_sph2, const float *g,
                  const float *targets3, double *loss, float *grad, uint8_t *touched);
int pf_train_counts(pf_ctx *ctx, size_t *n_params, size_t *n_table_entries);
/* Data-parallel training (one process per GPU): train_step split
 * around a gradient all-reduce.  pf_train_backward runs forward, loss and
 * backward of this rank's shard (n of the n_global queries of the step) into
 * the context's gradient buffers, scaled so their SUM over ranks is the
 * global-batch gradient (loss_part likewise sums to the global loss).
 * pf_train_grad_buffers exposes them for an in-place all-reduce: table
 * gradients as int64 fixed point (n_tab, SUM -- integer, so exact and
 * independent of the reduction order), MLP gradients binary32 (n_mlp, SUM),
 * touched flags uint8 (n_entries, MAX).  pf_train_apply then runs Adam. */
int pf_train_backward(pf_ctx *ctx, size_t n, const float *x3, const float *w_sph2, const float *g,
                      const float *targets3, size_t n_global, double *loss_part);
int pf_train_grad_buffers(pf_ctx *ctx, void **gtab, size_t *n_tab, void **gmlp, size_t *n_mlp,
                          void **touched, size_t *n_entries);
int pf_train_apply(pf_ctx *ctx, uint64_t step, uint64_t total_steps);
/* Master parameters (host or device memory, n = n_params). */
int pf_train_params(pf_ctx *ctx, float *out, size_t n);
/* Master parameters -> the inference field used by pf_field_query / renders. */
int pf_train_commit(pf_ctx *ctx);
/* train(field, map, cfg): total_steps x {make_batch on the
 * resident photon map (queries from make_rng(seed, Train, step*batch + i),
 * KNN radius from the staggered schedule, Eq. 6 + Eq. 7 targets) ->
 * train_step}; loss_history (total_steps doubles, may be NULL), cumulative
 * KNN-sampling vs optimizer device time.  Commits the field at the end. */
typedef struct {
    uint64_t total_steps;      /* 3000 */
    size_t batch;              /* 2^16 paper, 2^12 desk */
    int K;                     /* 1024 paper, 256 desk */
    int n_segments;            /* KnnSchedule */
    const double *seg_end;     /* progress fractions, strictly increasing, last = 1 */
    const double *seg_radius;  /* strictly increasing radii */
    double psi;                /* Eq. 7 precision */
    uint64_t seed;
    uint64_t start_step;       /* resume: first step to run (a checkpoint's next step); 0 = fresh run */
    uint64_t stop_step;        /* run steps [start_step, stop_step) (checkpoint in chunks); 0 = total_steps */
} pf_train_desc;
/* ms_knn_steps / ms_step_steps (total_steps doubles each, may be NULL): the
 * per-step split for the training log.  Only steps
 * [start_step, stop_step) run -- radius schedule, query streams, lr and Adam
 * bias correction use the absolute step and total_steps, so a run split into
 * chunks (with a checkpoint between them) is bit-identical to one call -- and
 * only those entries of loss_history / ms_*_steps are written. */
int pf_train(pf_ctx *ctx, const pf_train_desc *desc, double *loss_history, double *ms_knn,
             double *ms_step, double *ms_knn_steps, double *ms_step_steps);
/* Optimizer state (checkpoint / resume): master parameters and
 * both Adam moments, n_params binary32 each, host or device memory; NULL
 * skips one on get.  set also commits the parameters to the inference field.
 * The Adam step counter is the caller's (pf_train_step's `step`). */
int pf_train_state_get(pf_ctx *ctx, float *params, float *m, float *v, size_t n);
int pf_train_state_set(pf_ctx *ctx, const float *params, const float *m, const float *v, size_t n);

#ifdef __cplusplus
}
#endif
#endif /* PF_GPU_H */
