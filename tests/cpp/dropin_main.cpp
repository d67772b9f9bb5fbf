// Drop-in check: the reference API, spelled through include/gbil_b200.hpp.
// Usage: dropin_main <out.bin>  -- renders a seeded ortho scene, writes
// inputs, per-tile lists, forward outputs and gradients for tests/test_cpp_dropin.py.
#include <cstdio>
#include <cstring>
#include <vector>

#include "gbil_b200.hpp"

namespace gbil = gbil_b200;  // the one-line switch a reference user makes

template <typename T>
static void put(FILE* f, const std::vector<T>& v) {
    const uint64_t n = v.size();
    std::fwrite(&n, 8, 1, f);
    if (n) std::fwrite(v.data(), sizeof(T), n, f);
}

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    const int K = 2000, n = 4, W = 160, H = 120;
    gb_scene_spec spec{};
    spec.mode = GB_MODE_ORTHO;
    spec.n = n;
    spec.count = K;
    spec.seed = 77;
    spec.log_scale_lo = -0.7;
    spec.log_scale_hi = 2.0;
    spec.width = W;
    spec.height = H;
    std::vector<float> pos(2 * K), dk(K), th(K), ls(2 * K), op(K), gr(K * n * n * 3);
    if (gb_scene_generate(&spec, pos.data(), dk.data(), th.data(), nullptr, ls.data(), op.data(), gr.data()) != GB_OK)
        return 3;
    gbil::SplatSet set(K, gbil::ColorGridConfig{n, 0.5});
    set.position.assign(pos.begin(), pos.end());
    set.depth_key.assign(dk.begin(), dk.end());
    set.theta.assign(th.begin(), th.end());
    set.log_scale.assign(ls.begin(), ls.end());
    set.opacity_logit.assign(op.begin(), op.end());
    set.grid.assign(gr.begin(), gr.end());
    gbil::ImagePlaneCamera cam{W, H, {0.1, 0.2, 0.3}};
    const gbil::TileBinning bin = gbil::build_binning(set, cam, gbil::RasterConfig{});
    const gbil::RenderOutput out = gbil::render_forward(set, cam, bin);
    std::vector<double> ig(out.color.size());
    for (std::size_t i = 0; i < ig.size(); ++i) ig[i] = (i * 2654435761u) % 3 == 0 ? -1.0 : 1.0;
    const gbil::GradientBuffer g = gbil::render_backward(set, cam, bin, out, ig);
    // reference error behaviour: a mismatched camera must throw std::invalid_argument
    bool threw = false;
    try {
        gbil::render_forward(set, gbil::ImagePlaneCamera{W + 1, H, {0, 0, 0}}, bin);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    FILE* f = std::fopen(argv[1], "wb");
    if (!f) return 4;
    put(f, pos); put(f, dk); put(f, th); put(f, ls); put(f, op); put(f, gr);
    std::vector<int32_t> flat;
    std::vector<int64_t> offs{0};
    for (const auto& l : bin.tiles()) {
        flat.insert(flat.end(), l.begin(), l.end());
        offs.push_back((int64_t)flat.size());
    }
    put(f, offs); put(f, flat);
    put(f, out.color); put(f, out.final_transmittance); put(f, out.last_rank); put(f, ig);
    put(f, g.position); put(f, g.theta); put(f, g.log_scale); put(f, g.opacity_logit); put(f, g.grid);
    std::vector<int32_t> t{threw ? 1 : 0};
    put(f, t);
    std::fclose(f);
    return 0;
}
