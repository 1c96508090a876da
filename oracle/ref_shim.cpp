// ref_shim.cpp -- extern "C" access to the UNMODIFIED reference implementation.
//
// TEST INFRASTRUCTURE ONLY (see oracle/pf_oracle.h).  oracle/Makefile compiles
// this file together with /root/reference/proj/src/volume.cpp and parallel.cpp
// (read in place, never copied) into oracle/_ref/libpfref.so.  It exists to
//   (1) pin the C restatement in pf_oracle.c against the reference itself, and
//   (2) time the reference's own CPU render path (bench.py --impl reference):
//       pf::delta_track / pf::transmittance driven by pf::parallel_chunks
//       (proj/src/volume.cpp:204-256, proj/src/parallel.cpp:22-49); the
//       SPEC-only field query / NEE glue / compose come from pf_oracle.c.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "pf/math.hpp"
#include "pf/parallel.hpp"
#include "pf/phase.hpp"
#include "pf/rng.hpp"
#include "pf/volume.hpp"

#include "pf_oracle.h"

namespace {

struct RefScene {
    pf::VolumeGrid grid;
    pf::TransferFunction tf;
    pf::Medium *medium = nullptr;
};

thread_local char g_err[512];

int fail(const std::exception &e) {
    std::snprintf(g_err, sizeof(g_err), "%s", e.what());
    return 1;
}

}  // namespace

extern "C" {

const char *ref_last_error(void) { return g_err; }

// Pcg32 draws through make_rng (rng.hpp:73-76).
void ref_rng_u32(uint64_t seed, uint64_t stream, uint64_t index, int n, uint32_t *out) {
    pf::Pcg32 r = pf::make_rng(seed, static_cast<pf::Stream>(stream), index);
    for (int i = 0; i < n; ++i) out[i] = r.next_u32();
}
void ref_rng_double(uint64_t seed, uint64_t stream, uint64_t index, int n, double *out) {
    pf::Pcg32 r = pf::make_rng(seed, static_cast<pf::Stream>(stream), index);
    for (int i = 0; i < n; ++i) out[i] = r.next_double();
}
uint64_t ref_splitmix64(uint64_t x) { return pf::splitmix64(x); }
double ref_hg_eval(double g, double c) { return pf::hg_eval(g, c); }
double ref_hg_sample_cos(double g, double u) { return pf::hg_sample_cos(g, u); }
double ref_hg_cdf(double g, double c) { return pf::hg_cdf(g, c); }
void ref_hg_sample(double g, const double win[3], double u1, double u2, double out[3]) {
    pf::Vec3 w = pf::hg_sample(g, pf::Vec3{win[0], win[1], win[2]}, u1, u2);
    out[0] = w.x;
    out[1] = w.y;
    out[2] = w.z;
}
int ref_aabb_intersect(const double o[3], const double d[3], double tmin, double tmax,
                       double *t0, double *t1) {
    pf::Aabb box;
    pf::Ray r{{o[0], o[1], o[2]}, {d[0], d[1], d[2]}, tmin, tmax};
    return box.intersect(r, *t0, *t1) ? 1 : 0;
}

int ref_scene_create(int nx, int ny, int nz, const float *data, const double *tf_pts, int n_pts,
                     double density_scale, void **out) {
    try {
        auto *s = new RefScene();
        s->grid = pf::VolumeGrid(nx, ny, nz, std::vector<float>(data, data + (size_t)nx * ny * nz));
        std::vector<pf::TransferFunction::ControlPoint> pts(n_pts);
        for (int i = 0; i < n_pts; ++i) {
            pts[i].scalar = tf_pts[5 * i];
            pts[i].color = {tf_pts[5 * i + 1], tf_pts[5 * i + 2], tf_pts[5 * i + 3], tf_pts[5 * i + 4]};
        }
        s->tf = pf::TransferFunction(std::move(pts));
        s->medium = new pf::Medium(s->grid, s->tf, density_scale);
        *out = s;
        return 0;
    } catch (const std::exception &e) {
        return fail(e);
    }
}

void ref_scene_destroy(void *h) {
    auto *s = static_cast<RefScene *>(h);
    if (!s) return;
    delete s->medium;
    delete s;
}

double ref_scene_sigma_max(void *h) { return static_cast<RefScene *>(h)->medium->sigma_max(); }
double ref_grid_sample(void *h, const double p[3]) {
    return static_cast<RefScene *>(h)->grid.sample({p[0], p[1], p[2]});
}
void ref_tf_classify(void *h, double s, double rgba[4]) {
    pf::Rgba c = static_cast<RefScene *>(h)->tf.classify(s);
    rgba[0] = c.r;
    rgba[1] = c.g;
    rgba[2] = c.b;
    rgba[3] = c.a;
}

// Batched pf::delta_track; ray i uses make_rng(seed, stream, idx[i]).
// Returns 0, or 1 with ref_last_error() set if any ray is invalid.
// trace_photons (photon.hpp:52-57) is declared by the reference but never
// defined; this composes the pinned algorithm (see
// pf_oracle.c or_trace_photons) from the reference's OWN primitives --
// make_rng, Aabb::center/bounding_radius, sample_uniform_sphere,
// from_local_frame, delta_track, hg_sample(g, w, rng) -- so the restatement's
// composition is pinned against reference code, not against itself.
// out: 10 floats + tag per deposit in (photon, bounce) order; returns count
// (may exceed capacity, then only the first `capacity` are written).
size_t ref_trace_photons(void *h, const double *lights, int n_lights, uint64_t n_total, int n_phases,
                         const double *phase_set, int max_bounces, int rr_start, double rr_min, double rr_max,
                         uint64_t seed, float *out9, uint8_t *out_g, size_t capacity) {
    auto *s = static_cast<RefScene *>(h);
    const pf::Aabb &box = s->medium->world_box();
    const uint64_t pairs = (uint64_t)n_lights * (uint64_t)n_phases;
    size_t n_out = 0;
    for (uint64_t i = 0; i < n_total; ++i) {
        const uint64_t pr = i % pairs;
        const int li = (int)(pr / n_phases), gi = (int)(pr % n_phases);
        const double n_pair = (double)(n_total / pairs + (pr < n_total % pairs ? 1u : 0u));
        pf::Pcg32 rng = pf::make_rng(seed, pf::Stream::Trace, i);
        const pf::Vec3 P{lights[6 * li], lights[6 * li + 1], lights[6 * li + 2]};
        const pf::Vec3 I{lights[6 * li + 3], lights[6 * li + 4], lights[6 * li + 5]};
        pf::Vec3 w;
        {
            const pf::Vec3 v = box.center() - P;
            const double d = pf::length(v), R = box.bounding_radius();
            if (d <= R) {
                w = pf::sample_uniform_sphere(rng);
            } else {
                const pf::Vec3 axis = v / d;
                const double sr = R / d;
                const double cos_max = std::sqrt(std::max(0.0, 1.0 - sr * sr));
                const double u1 = rng.next_double(), u2 = rng.next_double();
                const double ct = 1.0 - u1 * (1.0 - cos_max);
                const double st = std::sqrt(std::max(0.0, 1.0 - ct * ct));
                const double phi = pf::kTwoPi * u2;
                w = pf::from_local_frame(axis, pf::Vec3{st * std::cos(phi), st * std::sin(phi), ct});
            }
        }
        pf::Vec3 o = P, thr{1.0, 1.0, 1.0};
        for (int bounce = 0; bounce < max_bounces; ++bounce) {
            auto it = pf::delta_track(*s->medium, pf::Ray{o, w, 0.0, INFINITY}, rng);
            if (!it) break;
            thr = thr * pf::Vec3{it->albedo.a * it->albedo.r, it->albedo.a * it->albedo.g,
                                 it->albedo.a * it->albedo.b};
            const pf::Vec3 nw = pf::hg_sample(phase_set[gi], w, rng);
            if (bounce >= 1) {
                if (n_out < capacity) {
                    float *r = out9 + 9 * n_out;
                    for (int k = 0; k < 3; ++k) {
                        r[k] = (float)it->position[k];
                        r[3 + k] = (float)nw[k];
                        r[6 + k] = (float)(I[k] / n_pair * thr[k]);
                    }
                    out_g[n_out] = (uint8_t)gi;
                }
                ++n_out;
            }
            if (bounce >= rr_start) {
                const double q = std::clamp(std::max({thr.x, thr.y, thr.z}), rr_min, rr_max);
                if (rng.next_double() >= q) break;
                thr /= q;
            }
            o = it->position;
            w = nw;
        }
    }
    return n_out;
}

int ref_delta_track_batch(void *h, size_t n, const double *o3, const double *d3,
                          const double *tmin, const double *tmax, uint64_t seed, uint64_t stream,
                          const uint64_t *idx, int *hit, double *pos3, double *scalar1, double *rgba4) {
    auto *s = static_cast<RefScene *>(h);
    try {
        for (size_t i = 0; i < n; ++i) {
            pf::Pcg32 rng = pf::make_rng(seed, static_cast<pf::Stream>(stream), idx[i]);
            pf::Ray r{{o3[3 * i], o3[3 * i + 1], o3[3 * i + 2]},
                      {d3[3 * i], d3[3 * i + 1], d3[3 * i + 2]},
                      tmin[i],
                      tmax[i]};
            auto it = pf::delta_track(*s->medium, r, rng);
            hit[i] = it ? 1 : 0;
            if (scalar1) scalar1[i] = 0.0;
            if (it) {
                pos3[3 * i] = it->position.x;
                pos3[3 * i + 1] = it->position.y;
                pos3[3 * i + 2] = it->position.z;
                if (scalar1) scalar1[i] = it->scalar;
                if (rgba4) {
                    rgba4[4 * i] = it->albedo.r;
                    rgba4[4 * i + 1] = it->albedo.g;
                    rgba4[4 * i + 2] = it->albedo.b;
                    rgba4[4 * i + 3] = it->albedo.a;
                }
            }
        }
        return 0;
    } catch (const std::exception &e) {
        return fail(e);
    }
}

int ref_transmittance_batch(void *h, size_t n, const double *a3, const double *b3, uint64_t seed,
                            uint64_t stream, const uint64_t *idx, int n_trials, double *out) {
    auto *s = static_cast<RefScene *>(h);
    try {
        for (size_t i = 0; i < n; ++i) {
            pf::Pcg32 rng = pf::make_rng(seed, static_cast<pf::Stream>(stream), idx[i]);
            out[i] = pf::transmittance(*s->medium, {a3[3 * i], a3[3 * i + 1], a3[3 * i + 2]},
                                       {b3[3 * i], b3[3 * i + 1], b3[3 * i + 2]}, rng, n_trials);
        }
        return 0;
    } catch (const std::exception &e) {
        return fail(e);
    }
}

// The reference CPU render path: the same per-sample program as
// or_render_neural, with the reference's own delta_track / transmittance /
// Pcg32 and the reference's parallel_chunks driver (chunk = one pixel row
// block).  Renders rows [y0, y1) of the frame into out_rgb (full frame layout).
int ref_render_neural(void *h, const or_light *lights, int n_lights, const or_field_cfg *fc,
                      const float *params, const or_camera *cam, const or_render_cfg *rc,
                      int workers, float *out_rgb, uint64_t *hits_out) {
    auto *s = static_cast<RefScene *>(h);
    const int W = cam->width, spp = rc->spp;
    pf::set_worker_count(workers);
    const size_t rows = (size_t)(rc->y1 - rc->y0);
    const size_t npix = rows * (size_t)(rc->x1 - rc->x0);
    // chunks of 4096 samples: 4096 / spp whole pixels
    const size_t chunk = std::max<size_t>(1, 4096 / (size_t)std::max(1, spp));
    std::vector<uint64_t> chunk_hits((npix + chunk - 1) / chunk, 0);
    try {
        pf::parallel_chunks(npix, chunk, [&](size_t ci, size_t b, size_t e) {
            uint64_t hits = 0;
            for (size_t p = b; p < e; ++p) {
                const int px = rc->x0 + (int)(p % (size_t)(rc->x1 - rc->x0));
                const int py = rc->y0 + (int)(p / (size_t)(rc->x1 - rc->x0));
                double acc[3] = {0.0, 0.0, 0.0};
                for (int k = 0; k < spp; ++k) {
                    uint64_t index = ((uint64_t)py * (uint64_t)W + (uint64_t)px) * (uint64_t)spp + k;
                    pf::Pcg32 rng = pf::make_rng(rc->seed, pf::Stream::CameraSample, index);
                    double u = rng.next_double();
                    double v = rng.next_double();
                    double o[3], d[3];
                    or_camera_ray(cam, px, py, u, v, o, d);
                    pf::Ray ray{{o[0], o[1], o[2]}, {d[0], d[1], d[2]}, 0.0, pf::kInfinity};
                    auto it = pf::delta_track(*s->medium, ray, rng);
                    double sample[3];
                    if (!it) {
                        for (int c = 0; c < 3; ++c) sample[c] = rc->background[c];
                    } else {
                        ++hits;
                        double x[3] = {it->position.x, it->position.y, it->position.z};
                        double w_out[3] = {-d[0], -d[1], -d[2]};
                        double Ld[3] = {0, 0, 0}, Li[3] = {0, 0, 0};
                        pf::Pcg32 nee = pf::make_rng(rc->seed, pf::Stream::Nee, index);
                        for (int l = 0; l < n_lights; ++l) {
                            double T = pf::transmittance(
                                *s->medium, it->position,
                                {lights[l].pos[0], lights[l].pos[1], lights[l].pos[2]}, nee,
                                rc->nee_trials);
                            or_nee_term(x, w_out, &lights[l], rc->g, T, Ld);
                        }
                        if (rc->use_field) {
                            double sph[2];
                            or_dir_to_sph(w_out, sph);
                            or_field_infer(fc, params, 1, x, sph, &rc->g, Li);
                        }
                        double rgba[4] = {it->albedo.r, it->albedo.g, it->albedo.b, it->albedo.a};
                        or_shade_sample(Ld, Li, rgba, rc->w_d, rc->w_i, sample);
                    }
                    for (int c = 0; c < 3; ++c) acc[c] += sample[c];
                }
                float *o3 = out_rgb + 3 * ((size_t)py * W + px);
                for (int c = 0; c < 3; ++c) o3[c] = (float)(acc[c] / (double)spp);
            }
            chunk_hits[ci] = hits;
        });
    } catch (const std::exception &e) {
        return fail(e);
    }
    uint64_t total = 0;
    for (uint64_t v : chunk_hits) total += v;
    if (hits_out) *hits_out = total;
    return 0;
}

// render_path_traced composed from the reference's OWN
// primitives -- make_rng, delta_track, transmittance, hg_sample(g, w, rng) --
// with the order pinned in pf_oracle.c or_render_path_traced / or_pt_indirect,
// driven by the reference's parallel_chunks.  Rows [y0, y1) into out_rgb.
int ref_render_path_traced(void *h, const or_light *lights, int n_lights, const or_camera *cam,
                           const or_render_cfg *rc, const or_pt_cfg *pt, int workers, float *out_rgb,
                           uint64_t *hits_out) {
    auto *s = static_cast<RefScene *>(h);
    const int W = cam->width, spp = rc->spp;
    pf::set_worker_count(workers);
    const size_t npix = (size_t)(rc->y1 - rc->y0) * (size_t)(rc->x1 - rc->x0);
    std::vector<uint64_t> chunk_hits((npix + 63) / 64, 0);
    auto lit = [&](const pf::Vec3 &x, const double w_out[3], pf::Pcg32 &rng, double Ld[3]) {
        const double xa[3] = {x.x, x.y, x.z};
        for (int l = 0; l < n_lights; ++l) {
            const double T = pf::transmittance(*s->medium, x, {lights[l].pos[0], lights[l].pos[1], lights[l].pos[2]},
                                               rng, rc->nee_trials);
            or_nee_term(xa, w_out, &lights[l], rc->g, T, Ld);
        }
    };
    try {
        pf::parallel_chunks(npix, 64, [&](size_t ci, size_t b, size_t e) {
            uint64_t hits = 0;
            for (size_t p = b; p < e; ++p) {
                const int px = rc->x0 + (int)(p % (size_t)(rc->x1 - rc->x0));
                const int py = rc->y0 + (int)(p / (size_t)(rc->x1 - rc->x0));
                double acc[3] = {0.0, 0.0, 0.0};
                for (int k = 0; k < spp; ++k) {
                    const uint64_t index = ((uint64_t)py * (uint64_t)W + (uint64_t)px) * (uint64_t)spp + k;
                    pf::Pcg32 rng = pf::make_rng(rc->seed, pf::Stream::CameraSample, index);
                    const double u = rng.next_double();
                    const double v = rng.next_double();
                    double o[3], d[3];
                    or_camera_ray(cam, px, py, u, v, o, d);
                    auto it = pf::delta_track(*s->medium, pf::Ray{{o[0], o[1], o[2]}, {d[0], d[1], d[2]}, 0.0,
                                                                  pf::kInfinity},
                                              rng);
                    double sample[3];
                    if (!it) {
                        for (int c = 0; c < 3; ++c) sample[c] = rc->background[c];
                    } else {
                        ++hits;
                        const double w_out[3] = {-d[0], -d[1], -d[2]};
                        double Ld[3] = {0, 0, 0}, Li[3] = {0, 0, 0};
                        pf::Pcg32 nee = pf::make_rng(rc->seed, pf::Stream::Nee, index);
                        lit(it->position, w_out, nee, Ld);
                        if (pt->max_bounces > 1) {
                            pf::Pcg32 r = pf::make_rng(rc->seed, pf::Stream::PathTrace, index);
                            pf::Vec3 x = it->position, w{d[0], d[1], d[2]};
                            double thr = 1.0;
                            for (int b2 = 1; b2 < pt->max_bounces; ++b2) {
                                w = pf::hg_sample(rc->g, w, r);
                                auto nx = pf::delta_track(*s->medium, pf::Ray{x, w, 0.0, pf::kInfinity}, r);
                                if (!nx) break;
                                const double wo[3] = {-w.x, -w.y, -w.z};
                                double Lk[3] = {0, 0, 0};
                                lit(nx->position, wo, r, Lk);
                                for (int c = 0; c < 3; ++c) Li[c] += thr * Lk[c];
                                thr *= nx->albedo.a * ((nx->albedo.r + nx->albedo.g + nx->albedo.b) / 3.0);
                                if (!(thr > 0.0)) break;
                                if (b2 >= pt->rr_start_bounce) {
                                    const double q = std::clamp(thr, pt->rr_min_survival, pt->rr_max_survival);
                                    if (r.next_double() >= q) break;
                                    thr /= q;
                                }
                                x = nx->position;
                            }
                        }
                        const double rgba[4] = {it->albedo.r, it->albedo.g, it->albedo.b, it->albedo.a};
                        or_shade_sample(Ld, Li, rgba, rc->w_d, rc->w_i, sample);
                    }
                    for (int c = 0; c < 3; ++c) acc[c] += sample[c];
                }
                float *o3 = out_rgb + 3 * ((size_t)py * W + px);
                for (int c = 0; c < 3; ++c) o3[c] = (float)(acc[c] / (double)spp);
            }
            chunk_hits[ci] = hits;
        });
    } catch (const std::exception &e) {
        return fail(e);
    }
    uint64_t total = 0;
    for (uint64_t v : chunk_hits) total += v;
    if (hits_out) *hits_out = total;
    return 0;
}

}  // extern "C"
