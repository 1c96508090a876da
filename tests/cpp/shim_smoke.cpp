// Compiles the reference-side shim (include/pf/gpu.hpp) against the
// reference's own headers and links libpfgpu.so.  Without a GPU the Device
// constructor must throw std::runtime_error (no silent CPU fallback); with one
// it tracks a few rays through pf::Medium built by the reference code.
#include <cstdio>
#include <stdexcept>

#include "pf/gpu.hpp"

int main() {
    try {
        pf::gpu::Device dev(0);
        pf::VolumeGrid grid(2, 2, 2, std::vector<float>(8, 1.0f));
        pf::TransferFunction tf;  // constant white, alpha 1
        pf::Medium medium(grid, tf, 5.0);
        dev.set_medium(medium);
        std::vector<pf::Ray> rays(4, pf::Ray{{0.5, 0.5, -1.0}, {0.0, 0.0, 1.0}, 0.0, pf::kInfinity});
        auto its = dev.delta_track(rays, 7, pf::Stream::CameraSample, {0, 1, 2, 3});
        int hits = 0;
        for (auto &it : its) {
            hits += it.has_value();
            if (it && it->scalar != 1.0) return 5;  // Interaction::scalar of the constant-1 grid
        }
        dev.set_lights({pf::LightSource{{2.0, 2.5, -1.0}, {1.0, 1.0, 1.0}}});
        pf::TraceConfig tc;
        tc.n_total = 1000;
        pf::TraceResult tr = dev.trace_photons(tc);
        if (tr.emitted_per_pair.size() != 3 || tr.photons.empty()) return 4;
        std::printf("gpu ok hits=%d photons=%zu\n", hits, tr.photons.size());
        try {
            dev.transmittance({{0, 0, 0}}, {{1, 1, 1}}, 0, pf::Stream::Nee, {0}, 0);
            return 3;
        } catch (const std::invalid_argument &) {
        }
        return 0;
    } catch (const std::runtime_error &e) {
        std::printf("no gpu: %s\n", e.what());
        return 0;
    }
}
