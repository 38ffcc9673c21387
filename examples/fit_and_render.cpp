// The C++ layer beyond the per-point API (include/nasg/nasg_gpu.hpp): a few
// iterations of the built-in render loop (SPEC tracer module), the explicit
// vMF / NASG mixture entries (sphdist.hpp) and one NASG-vs-vMF fit (SPEC run_fit).
//   g++ -std=c++20 -Iinclude -I/usr/local/cuda/include examples/fit_and_render.cpp \
//       -Lpaper_2303_08064_b200/lib -lnasg_b200 -L/usr/local/cuda/lib64 -lcudart \
//       -Wl,-rpath,$PWD/paper_2303_08064_b200/lib
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <vector>

#include "nasg/nasg_gpu.hpp"

namespace g = nasg::gpu;

int main() {
    try {
        float bmin[3], bmax[3];
        g::check(nasg_render_scene_bounds(NASG_SCENE_BOX, bmin, bmax));
        g::Guide guide(g::TrainerConfig{}, 0, bmin, bmax);
        guide.set_precision(g::Precision::BF16);
        guide.set_train_precision(g::Precision::BF16);
        nasg_render_config rc;
        nasg_render_config_default(&rc);
        rc.width = rc.height = 128;
        rc.schedule_m = 1;
        rc.schedule_b = 4;
        g::Render render(guide, rc);
        nasg_render_stats st{};
        for (int i = 0; i < 8; ++i) st = render.iteration();
        const std::vector<float> img = render.image(128 * 128);
        double mean = 0.0;
        for (float v : img) mean += v;
        std::printf("render: %lld vertices, %lld guided, b = %.3f, mean %.4f\n", (long long)st.vertices,
                    (long long)st.guided_vertices, st.b, mean / img.size());

        // one vMF lobe, sampled and evaluated on the device
        const int n = 1024;
        std::vector<g::VmfRecord> comp(n, g::VmfRecord{{0.f, 0.f, 1.f}, 10.f});
        std::vector<float> w(n, 1.f), xi(4 * n);
        for (int i = 0; i < n; ++i)
            for (int k = 0; k < 4; ++k) xi[4 * i + k] = (float)((i * 7 + k * 13) % 97) / 97.f;
        float *d = nullptr;
        cudaMalloc(&d, sizeof(float) * 13 * n);
        float *dc = d, *dw = d + 4 * n, *dxi = d + 5 * n, *dout = d + 9 * n;
        cudaMemcpy(dc, comp.data(), sizeof(g::VmfRecord) * n, cudaMemcpyHostToDevice);
        cudaMemcpy(dw, w.data(), sizeof(float) * n, cudaMemcpyHostToDevice);
        cudaMemcpy(dxi, xi.data(), sizeof(float) * 4 * n, cudaMemcpyHostToDevice);
        g::mixture_sample(g::Family::VMF, n, 1, dc, dw, dxi, dout);
        std::vector<float> o(4 * n);
        cudaMemcpy(o.data(), dout, sizeof(float) * 4 * n, cudaMemcpyDeviceToHost);
        cudaFree(d);
        const double k10 = 10.0 / (2.0 * M_PI * (1.0 - std::exp(-20.0)));  // vmf pdf at mu
        std::printf("vmf: sample 0 = (%f %f %f) pdf %f (pdf at mu %f)\n", o[0], o[1], o[2], o[3], k10);

        // 8-lobe NASG vs 14-lobe vMF on a single anisotropic NASG target
        g::NasgRecord target{{1.f, 0.f, 0.f}, 40.f, {0.f, 1.f, 0.f}, 100.f, {0.f, 0.f, 1.f}, 0.f};
        const float tw = 1.f;
        nasg_fit_config fc{NASG_DIST_NASG, 8, 1024, 800, 1, 0.02f, 3};
        const g::FitResult a = g::fit(fc, 2, g::Family::NASG, 1, &target, &tw);
        fc.model = NASG_DIST_VMF;
        fc.n_components = 14;
        const g::FitResult b = g::fit(fc, 2, g::Family::NASG, 1, &target, &tw);
        std::printf("fit: KL nasg8 %.4f %.4f, vmf14 %.4f %.4f\n", a.kl[0], a.kl[1], b.kl[0], b.kl[1]);
    } catch (const g::Error &e) {
        std::fprintf(stderr, "nasg error: %s\n", e.what());
        return 1;
    }
    return 0;
}
