// Minimal renderer-side use of the C++ layer (include/nasg/nasg_gpu.hpp): one
// progressive iteration of SPEC.md's render loop reduced to its guiding calls —
// query + sample at every shading point, MIS pdf, then train on the collected
// samples and publish (guiding.hpp:149).
//   g++ -std=c++20 -Iinclude -I/usr/local/cuda/include examples/render_step.cpp \
//       -Lpaper_2303_08064_b200/lib -lnasg_b200 -L/usr/local/cuda/lib64 -lcudart \
//       -Wl,-rpath,$PWD/paper_2303_08064_b200/lib
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "nasg/nasg_gpu.hpp"

int main() {
    const float bmin[3] = {-1, -1, -1}, bmax[3] = {1, 1, 1};
    const int64_t n = 1 << 16;
    try {
        nasg::gpu::Guide guide(nasg::gpu::TrainerConfig{}, 0, bmin, bmax);
        guide.set_precision(nasg::gpu::Precision::BF16);
        std::vector<float> x(4 * n), wo(4 * n), nrm(4 * n), xi(4 * n);
        nasg_synth_queries(1, 0, n, bmin, bmax, x.data(), wo.data(), nrm.data(), xi.data());
        float *d = nullptr;
        cudaMalloc(&d, sizeof(float) * n * 21);
        float *dx = d, *dwo = d + 4 * n, *dn = d + 8 * n, *dxi = d + 12 * n, *out = d + 16 * n, *c = d + 20 * n;
        cudaMemcpy(dx, x.data(), 16 * n, cudaMemcpyHostToDevice);
        cudaMemcpy(dwo, wo.data(), 16 * n, cudaMemcpyHostToDevice);
        cudaMemcpy(dn, nrm.data(), 16 * n, cudaMemcpyHostToDevice);
        cudaMemcpy(dxi, xi.data(), 16 * n, cudaMemcpyHostToDevice);
        guide.sample(n, dx, dwo, dn, dxi, out, c);
        std::vector<float> o(4 * n);
        cudaMemcpy(o.data(), out, 16 * n, cudaMemcpyDeviceToHost);
        std::vector<nasg::gpu::TrainingSample> s(n);
        nasg_synth_samples(2, 0, n, bmin, bmax, s.data());
        nasg::gpu::TrainingSample *ds = nullptr;
        cudaMalloc(&ds, sizeof(*ds) * n);
        cudaMemcpy(ds, s.data(), sizeof(*ds) * n, cudaMemcpyHostToDevice);
        nasg::gpu::TrainStats st = guide.train_iteration({ds, (size_t)n}, nasg_blend_coefficient(4, 4, 64));
        std::printf("dir0 = (%f %f %f) pdf %f; train: %d steps, mean loss %g, dropped %llu\n", o[0], o[1], o[2],
                    o[3], st.steps, st.mean_loss, (unsigned long long)st.dropped_samples);
        // resume point: weights (the reference's NASGNET1 file) + the Adam state
        guide.save_checkpoint("render_step.nasg", /*optimizer=*/true);
        nasg::gpu::Guide resumed(nasg::gpu::TrainerConfig{}, 0, bmin, bmax);
        resumed.load_checkpoint("render_step.nasg");
        std::printf("resumed: %s\n", resumed.parameters() == guide.parameters() ? "same weights" : "DIFFERENT");
        cudaFree(ds);
        cudaFree(d);
    } catch (const nasg::gpu::Error &e) {
        std::fprintf(stderr, "nasg error: %s\n", e.what());
        return 1;
    }
    return 0;
}
