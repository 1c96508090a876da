// The C ABI alone (include/pf_gpu.h), no Python, no reference headers: what a
// cgo / JNI / plain-C host does.  Builds a synthetic scene, renders the three
// first-interaction renderers, traces a photon map, runs a few training steps
// and queries the trained field; prints one line of stats.  Compiled and run
// by tests/test_gpu_capi.py on the GPU box.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "pf_gpu.h"

#define CHECK(x)                                                                  \
    do {                                                                          \
        int rc_ = (x);                                                            \
        if (rc_ != PF_OK) {                                                       \
            std::fprintf(stderr, "%s -> %d: %s\n", #x, rc_, pf_last_error()); \
            return 1;                                                             \
        }                                                                         \
    } while (0)

int main() {
    pf_ctx *ctx = nullptr;
    CHECK(pf_ctx_create(0, &ctx));
    const int n = 48;
    std::vector<float> vol((size_t)n * n * n);
    for (int z = 0; z < n; ++z)
        for (int y = 0; y < n; ++y)
            for (int x = 0; x < n; ++x) {
                const double px = (x + 0.5) / n - 0.5, py = (y + 0.5) / n - 0.5, pz = (z + 0.5) / n - 0.5;
                const double r = std::sqrt(px * px + py * py + pz * pz);
                vol[((size_t)z * n + y) * n + x] = (float)std::fmax(0.0, 1.0 - r / 0.45);
            }
    CHECK(pf_volume_upload(ctx, n, n, n, vol.data()));
    const double tf[] = {0.0, 1, 1, 1, 0.0, 0.02, 0.9, 0.6, 0.3, 0.02, 0.5, 0.8, 0.8, 0.8, 0.3, 1.0, 1, 1, 1, 0.6};
    CHECK(pf_medium_set(ctx, tf, 4, 100.0, -1.0));
    const double light[] = {2.0, 2.5, -1.0, 1.0, 1.0, 1.0};
    CHECK(pf_lights_set(ctx, light, 1));

    pf_field_desc fd = {{3, 8, 4, 4, 2.0, 15}, {2, 8, 4, 4, 2.0, 15}, 5, 64, 5.0};
    size_t np = 0;
    CHECK(pf_field_param_count(&fd, &np));
    std::vector<float> params(np);
    CHECK(pf_field_init(&fd, 1, 1e-4, 0.0, params.data()));
    CHECK(pf_field_load(ctx, &fd, params.data(), np));

    const double pos[] = {0.5, 0.5, -0.9}, at[] = {0.5, 0.5, 0.5}, up[] = {0, 1, 0};
    pf_camera cam;
    CHECK(pf_camera_make(pos, at, up, 40.0, 96, 64, &cam));
    pf_render_desc d = {4, 0.0, 7, 1.0, 1.0, {0, 0, 0}, PF_MODE_FAST, 1, 1, 16, 16, 0, 1};
    std::vector<float> a((size_t)96 * 64 * 3), b(a.size()), c(a.size());
    pf_render_stats st;
    CHECK(pf_render_neural(ctx, &cam, &d, a.data(), &st));
    pf_path_desc pd = {16, 3, 0.05, 0.95};
    CHECK(pf_render_path_traced(ctx, &cam, &d, &pd, b.data(), nullptr));

    const double G[] = {-0.75, 0.0, 0.75};
    pf_trace_desc td = {200000, 3, G, 16, 3, 0.05, 0.95, 3};
    size_t n_ph = 0;
    CHECK(pf_trace_photons(ctx, &td, &n_ph, nullptr));
    CHECK(pf_knn_build_traced(ctx, 3, G));
    CHECK(pf_render_photon_map(ctx, &cam, &d, 32, INFINITY, c.data(), nullptr));

    CHECK(pf_train_init(ctx, &fd, params.data(), np, nullptr));
    const double ends[] = {0.5, 1.0}, radii[] = {0.1, 0.2};
    pf_train_desc tr = {50, 2048, 32, 2, ends, radii, 5.0, 9};
    std::vector<double> loss(50);
    double ms_knn = 0, ms_step = 0;
    CHECK(pf_train(ctx, &tr, loss.data(), &ms_knn, &ms_step, nullptr, nullptr));

    // data-parallel step pieces (one rank here): backward of a shard, the
    // device gradient buffers an NCCL all-reduce would use, Adam
    {
        const size_t nb = 512;
        std::vector<float> x(nb * 3), w(nb * 2), gg(nb), t(nb * 3);
        for (size_t i = 0; i < nb; ++i) {
            for (int a = 0; a < 3; ++a) x[3 * i + a] = (float)((i * 37 + a * 11) % 97) / 97.0f;
            w[2 * i] = (float)(i % 13) / 13.0f;
            w[2 * i + 1] = (float)(i % 7) / 7.0f;
            gg[i] = (float)G[i % 3];
            for (int a = 0; a < 3; ++a) t[3 * i + a] = 0.5f;
        }
        double part = -1.0;
        CHECK(pf_train_backward(ctx, nb, x.data(), w.data(), gg.data(), t.data(), 2 * nb, &part));
        void *gt = nullptr, *gm = nullptr, *tc = nullptr;
        size_t nt = 0, nm = 0, ne = 0;
        CHECK(pf_train_grad_buffers(ctx, &gt, &nt, &gm, &nm, &tc, &ne));
        if (!gt || !gm || !tc || nt + nm != np || ne == 0 || !(part >= 0.0)) return 3;
        CHECK(pf_train_apply(ctx, 0, 10));
    }

    // errors come back as status codes + message, never as a CPU fallback
    pf_render_desc bad = d;
    bad.spp = 0;
    if (pf_render_neural(ctx, &cam, &bad, a.data(), nullptr) != PF_ERR_INVALID) return 2;

    double sa = 0, sb = 0, sc = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        sa += a[i];
        sb += b[i];
        sc += c[i];
    }
    const bool finite = std::isfinite(sa) && std::isfinite(sb) && std::isfinite(sc);
    std::printf("capi ok hits=%llu photons=%zu mean_neural=%.6g mean_pt=%.6g mean_pm=%.6g loss0=%.6g loss49=%.6g finite=%d\n",
                (unsigned long long)st.hits, n_ph, sa / a.size(), sb / b.size(), sc / c.size(), loss[0], loss[49],
                finite ? 1 : 0);
    pf_ctx_destroy(ctx);
    return finite && loss[49] < loss[0] ? 0 : 5;
}
