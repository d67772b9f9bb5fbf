// Drop-in check of the training-loop half of the reference API through include/gbil_b200.hpp:
// fit (train.hpp:174-219), psnr/ssim (metrics.hpp), save/load_splats (serialize.hpp).
// Usage: fit_main <in.bin> <out.bin> <tmpdir>
//   in : W, H, K, n, iters, mse_ssim, seed (int64 each) then W*H*3 doubles (target)
//   out: history (m x 4 doubles), final position/depth_key/theta/log_scale/opacity/grid, psnr(target, 0.5),
//        ssim(target, 0.5), and 1 if a save/load round trip of the final set was exact
#include <cstdio>
#include <vector>

#include "gbil_b200.hpp"

namespace gbil = gbil_b200;

template <typename T>
static void put(FILE* f, const std::vector<T>& v) {
    const uint64_t n = v.size();
    std::fwrite(&n, 8, 1, f);
    if (n) std::fwrite(v.data(), sizeof(T), n, f);
}

int main(int argc, char** argv) {
    if (argc < 4) return 2;
    FILE* in = std::fopen(argv[1], "rb");
    if (!in) return 3;
    int64_t hdr[7];
    if (std::fread(hdr, 8, 7, in) != 7) return 4;
    const int W = (int)hdr[0], H = (int)hdr[1];
    gbil::Image target(W, H);
    if (std::fread(target.data.data(), 8, target.data.size(), in) != target.data.size()) return 5;
    std::fclose(in);
    gbil::TrainConfig cfg;
    cfg.splat_count = (std::size_t)hdr[2];
    cfg.grid = gbil::ColorGridConfig{(int)hdr[3], 0.5};
    cfg.allow_any_n = true;
    cfg.iterations = hdr[4];
    cfg.loss = hdr[5] ? gbil::LossKind::mse_plus_ssim : gbil::LossKind::mse;
    cfg.seed = (uint64_t)hdr[6];
    cfg.log_every = 1;
    const gbil::FitResult r = gbil::fit(target, cfg);
    std::vector<double> hist;
    for (const auto& m : r.history) hist.insert(hist.end(), {(double)m.iter, m.loss, m.psnr, m.ssim});
    const gbil::Image grey(W, H, 0.5);
    std::vector<double> metrics{gbil::psnr(target, grey), W >= 11 && H >= 11 ? gbil::ssim(target, grey) : 0.0};
    const std::string path = std::string(argv[3]) + "/final.gbil";
    gbil::save_splats(path, r.splats);
    const gbil::SplatSet back = gbil::load_splats(path);
    const bool same = back.position == r.splats.position && back.theta == r.splats.theta &&
                      back.grid == r.splats.grid && back.depth_key == r.splats.depth_key;
    FILE* f = std::fopen(argv[2], "wb");
    if (!f) return 6;
    put(f, hist);
    put(f, r.splats.position); put(f, r.splats.depth_key); put(f, r.splats.theta);
    put(f, r.splats.log_scale); put(f, r.splats.opacity_logit); put(f, r.splats.grid);
    put(f, metrics);
    std::vector<int32_t> ok{same ? 1 : 0};
    put(f, ok);
    std::fclose(f);
    return 0;
}
