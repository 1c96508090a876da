// pf/gpu.hpp -- reference-side C++ API over the C ABI (include/pf_gpu.h).
//
// Drop-in for the render hot path of the reference C++20 library
// (namespace pf, /root/reference/proj).  Include it next to the reference
// headers; it takes the reference's own types (pf::Medium, pf::Ray,
// pf::Photon, pf::LightSource, pf::Stream) and rethrows the reference's
// exception types (std::invalid_argument / std::runtime_error), so call sites
// such as
//     auto it = pf::delta_track(medium, ray, rng);          // volume.hpp:115
// become the batched
//     auto its = dev.delta_track(rays, seed, pf::Stream::CameraSample, idx);
// with make_rng(seed, stream, idx[i]) per ray -- bit-identical streams.
#pragma once

#include <cstddef>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "pf/photon.hpp"  // reference: Photon, LightSource      (photon.hpp:17-27)
#include "pf/rng.hpp"     // reference: Stream                   (rng.hpp:62-71)
#include "pf/volume.hpp"  // reference: VolumeGrid, TransferFunction, Medium, Interaction
#include "pf_gpu.h"

namespace pf::gpu {

static_assert(sizeof(pf::Photon) == sizeof(pf_photon), "pf::Photon must be 40 bytes");

inline void check(int rc) {
    if (rc == PF_OK) return;
    if (rc == PF_ERR_INVALID) throw std::invalid_argument(pf_last_error());
    throw std::runtime_error(pf_last_error());
}

// One CUDA device.  Scene, field and photon map are device-resident copies of
// caller-owned objects (the reference's Medium only borrows them,
// volume.hpp:107-108); call set_medium again after a TF / volume change.
class Device {
  public:
    explicit Device(int device = 0) { check(pf_ctx_create(device, &ctx_)); }
    ~Device() { pf_ctx_destroy(ctx_); }
    Device(const Device &) = delete;
    Device &operator=(const Device &) = delete;

    pf_ctx *handle() const { return ctx_; }

    // Medium(grid, tf, density_scale) (volume.hpp:94): uploads the grid and the
    // TF and reuses medium.sigma_max() bit-for-bit as the majorant.
    void set_medium(const pf::Medium &m) {
        const pf::VolumeGrid &g = m.grid();
        if (g.nx() != nx_ || g.ny() != ny_ || g.nz() != nz_ || g.data().data() != vol_) {
            check(pf_volume_upload(ctx_, g.nx(), g.ny(), g.nz(), g.data().data()));
            nx_ = g.nx();
            ny_ = g.ny();
            nz_ = g.nz();
            vol_ = g.data().data();
        }
        std::vector<double> pts;
        for (const auto &p : m.tf().control_points())
            pts.insert(pts.end(), {p.scalar, p.color.r, p.color.g, p.color.b, p.color.a});
        check(pf_medium_set(ctx_, pts.data(), (int)(pts.size() / 5), m.density_scale(), m.sigma_max()));
    }

    void set_lights(const std::vector<pf::LightSource> &lights) {
        std::vector<double> v;
        for (const auto &l : lights)
            v.insert(v.end(), {l.position.x, l.position.y, l.position.z, l.intensity.x, l.intensity.y,
                               l.intensity.z});
        check(pf_lights_set(ctx_, v.data(), (int)lights.size()));
        n_lights_ = lights.size();
    }

    // Batched pf::delta_track (volume.cpp:204-225).
    std::vector<std::optional<pf::Interaction>> delta_track(const std::vector<pf::Ray> &rays, uint64_t seed,
                                                            pf::Stream stream, const std::vector<uint64_t> &idx,
                                                            bool fp64 = true) {
        const size_t n = rays.size();
        if (idx.size() != n) throw std::invalid_argument("delta_track: idx size mismatch");
        std::vector<double> o(3 * n), d(3 * n), t0(n), t1(n), pos(3 * n), scalar(n), rgba(4 * n);
        for (size_t i = 0; i < n; ++i) {
            o[3 * i] = rays[i].origin.x, o[3 * i + 1] = rays[i].origin.y, o[3 * i + 2] = rays[i].origin.z;
            d[3 * i] = rays[i].direction.x, d[3 * i + 1] = rays[i].direction.y,
            d[3 * i + 2] = rays[i].direction.z;
            t0[i] = rays[i].t_min;
            t1[i] = rays[i].t_max;
        }
        std::vector<int> hit(n);
        check(pf_delta_track_batch(ctx_, n, o.data(), d.data(), t0.data(), t1.data(), seed, (uint64_t)stream,
                                   idx.data(), fp64 ? 1 : 0, hit.data(), pos.data(), scalar.data(), rgba.data()));
        std::vector<std::optional<pf::Interaction>> out(n);
        for (size_t i = 0; i < n; ++i) {
            if (!hit[i]) continue;
            pf::Interaction it;
            it.position = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
            it.scalar = scalar[i];
            it.albedo = {rgba[4 * i], rgba[4 * i + 1], rgba[4 * i + 2], rgba[4 * i + 3]};
            out[i] = it;
        }
        return out;
    }

    // Batched pf::transmittance (volume.cpp:227-256); ratio = fast-mode estimator.
    std::vector<double> transmittance(const std::vector<pf::Vec3> &a, const std::vector<pf::Vec3> &b, uint64_t seed,
                                      pf::Stream stream, const std::vector<uint64_t> &idx, int n_trials,
                                      bool ratio = false) {
        const size_t n = a.size();
        if (b.size() != n || idx.size() != n) throw std::invalid_argument("transmittance: size mismatch");
        std::vector<double> av(3 * n), bv(3 * n), out(n);
        for (size_t i = 0; i < n; ++i) {
            av[3 * i] = a[i].x, av[3 * i + 1] = a[i].y, av[3 * i + 2] = a[i].z;
            bv[3 * i] = b[i].x, bv[3 * i + 1] = b[i].y, bv[3 * i + 2] = b[i].z;
        }
        check((ratio ? pf_transmittance_ratio_batch : pf_transmittance_batch)(
            ctx_, n, av.data(), bv.data(), seed, (uint64_t)stream, idx.data(), n_trials, out.data()));
        return out;
    }

    // PhotonField: flat parameter vector.
    void load_field(const pf_field_desc &desc, const std::vector<float> &params) {
        check(pf_field_load(ctx_, &desc, params.data(), params.size()));
    }
    // infer_radiance / forward over a batch.
    std::vector<float> query_field(const std::vector<float> &x3, const std::vector<float> &w_sph2,
                                   const std::vector<float> &g, bool decoded = true) {
        std::vector<float> out(3 * g.size());
        check(pf_field_query(ctx_, g.size(), x3.data(), w_sph2.data(), g.data(), out.data(), decoded ? 1 : 0));
        return out;
    }

    // render_neural: row-major RGB binary32 frame.
    std::vector<float> render_neural(const pf_camera &cam, const pf_render_desc &desc,
                                     pf_render_stats *stats = nullptr) {
        std::vector<float> frame((size_t)cam.width * cam.height * 3);
        check(pf_render_neural(ctx_, &cam, &desc, frame.data(), stats));
        return frame;
    }

    // train(field, map, cfg) and its pieces
    void train_init(const pf_field_desc &desc, const std::vector<float> &params,
                    const pf_adam_desc *adam = nullptr) {
        check(pf_train_init(ctx_, &desc, params.data(), params.size(), adam));
    }
    double train_step(size_t n, const float *x3, const float *w_sph2, const float *g, const float *targets3,
                      uint64_t step, uint64_t total_steps) {
        double loss = 0.0;
        check(pf_train_step(ctx_, n, x3, w_sph2, g, targets3, step, total_steps, &loss));
        return loss;
    }
    // data-parallel train_step: this rank's shard backward, then the caller
    // all-reduces grad_buffers() in place (int64 SUM, float SUM, uint8 MAX,
    // e.g. ncclAllReduce on the context's stream), then train_apply().
    double train_backward(size_t n, const float *x3, const float *w_sph2, const float *g, const float *targets3,
                          size_t n_global) {
        double loss_part = 0.0;
        check(pf_train_backward(ctx_, n, x3, w_sph2, g, targets3, n_global, &loss_part));
        return loss_part;
    }
    struct GradBuffers {
        void *gtab, *gmlp, *touched;
        size_t n_tab, n_mlp, n_entries;
    };
    GradBuffers grad_buffers() {
        GradBuffers b{};
        check(pf_train_grad_buffers(ctx_, &b.gtab, &b.n_tab, &b.gmlp, &b.n_mlp, &b.touched, &b.n_entries));
        return b;
    }
    void train_apply(uint64_t step, uint64_t total_steps) { check(pf_train_apply(ctx_, step, total_steps)); }
    std::vector<double> train(const pf_train_desc &cfg, double *ms_knn = nullptr, double *ms_step = nullptr) {
        std::vector<double> hist(cfg.total_steps);
        check(pf_train(ctx_, &cfg, hist.data(), ms_knn, ms_step, nullptr, nullptr));
        return hist;
    }

    // render_path_traced: NEE + HG continuation + roulette.
    std::vector<float> render_path_traced(const pf_camera &cam, const pf_render_desc &desc,
                                          const pf_path_desc &path, pf_render_stats *stats = nullptr) {
        std::vector<float> frame((size_t)cam.width * cam.height * 3, 0.0f);
        check(pf_render_path_traced(ctx_, &cam, &desc, &path, frame.data(), stats));
        return frame;
    }

    // render_photon_map: L_i = Eq. 6 over the resident map;
    // desc.g outside the map's phase set throws std::invalid_argument.
    std::vector<float> render_photon_map(const pf_camera &cam, const pf_render_desc &desc, int K, float r_max,
                                         pf_render_stats *stats = nullptr) {
        std::vector<float> frame((size_t)cam.width * cam.height * 3, 0.0f);
        check(pf_render_photon_map(ctx_, &cam, &desc, K, r_max, frame.data(), stats));
        return frame;
    }

    // trace_photons(medium, lights, cfg) (photon.hpp:56 -- declared by the
    // reference, defined here on the device): call set_medium / set_lights
    // first.  Returns the reference's TraceResult with the photons in
    // (photon index, bounce) order and emitted_per_pair filled.
    pf::TraceResult trace_photons(const pf::TraceConfig &cfg) {
        pf_trace_desc d{cfg.n_total, (int)cfg.phase_set.size(), cfg.phase_set.data(), cfg.max_bounces,
                        cfg.rr_start_bounce, cfg.rr_min_survival, cfg.rr_max_survival, cfg.seed};
        pf::TraceResult r;
        r.phase_set = cfg.phase_set;
        r.n_lights = n_lights_;
        r.emitted_per_pair.resize(n_lights_ * cfg.phase_set.size());
        size_t n = 0;
        check(pf_trace_photons(ctx_, &d, &n, r.emitted_per_pair.data()));
        r.photons.resize(n);
        check(pf_trace_fetch(ctx_, reinterpret_cast<pf_photon *>(r.photons.data()), n));
        return r;
    }

    // build(photons) -- ids are load-order indices into `photons`.
    void build(const std::vector<pf::Photon> &photons, const std::vector<double> &phase_set) {
        check(pf_knn_build(ctx_, reinterpret_cast<const pf_photon *>(photons.data()), photons.size(),
                           (int)phase_set.size(), phase_set.data()));
    }
    // knn_phase: per query the ascending (id, distance^2) list.
    std::vector<std::vector<std::pair<uint32_t, float>>> knn_phase(const std::vector<float> &x3,
                                                                    const std::vector<uint8_t> &g_index, int K,
                                                                    float r_max) {
        const size_t nq = g_index.size();
        std::vector<uint32_t> ids(nq * (size_t)K);
        std::vector<float> d2(nq * (size_t)K);
        std::vector<int32_t> cnt(nq);
        check(pf_knn_query(ctx_, nq, x3.data(), g_index.data(), K, r_max, ids.data(), d2.data(), cnt.data()));
        std::vector<std::vector<std::pair<uint32_t, float>>> out(nq);
        for (size_t i = 0; i < nq; ++i)
            for (int k = 0; k < cnt[i]; ++k) out[i].emplace_back(ids[i * K + k], d2[i * K + k]);
        return out;
    }

  private:
    pf_ctx *ctx_ = nullptr;
    int nx_ = 0, ny_ = 0, nz_ = 0;
    const float *vol_ = nullptr;
    size_t n_lights_ = 0;
};

}  // namespace pf::gpu
