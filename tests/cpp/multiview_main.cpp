// C++ host of the view-sharded training step (include/gbil_b200.hpp, gbil_b200::multiview) on the GPUs
// listed on the command line, with NCCL communicators from ncclCommInitAll through the C-ABI.
//   multiview_main <inputs.bin> <outputs.bin> <steps> <sharded 0|1> [device ...]
// inputs.bin (little-endian): i64 K, i32 n, i32 W, i32 H, i32 views; f32 position[3K], quat[4K],
// log_scale[2K], opacity[K], grid[K*3n^2]; per view f64 fx, fy, cx, cy, rot[9], trans[3]; per view f32
// target[H*W*3].  outputs.bin: f64 losses[steps]; i64 T; f32 params[T] (rank 0); f32 grads[T] (rank 0,
// the last step's summed gradients in all-reduce mode); then the flat layout offsets (5 x i64).
#include <cstdio>
#include <fstream>
#include <iostream>

#include "gbil_b200.hpp"

namespace mv = gbil_b200::multiview;

template <typename T>
static void rd(std::ifstream& f, T* p, std::size_t n) {
    f.read(reinterpret_cast<char*>(p), sizeof(T) * n);
    if (!f) throw std::runtime_error("short input");
}

int main(int argc, char** argv) {
    if (argc < 5) {
        std::fprintf(stderr, "usage: %s in out steps sharded [devices]\n", argv[0]);
        return 2;
    }
    std::ifstream in(argv[1], std::ios::binary);
    std::int64_t K;
    std::int32_t n, W, H, V;
    rd(in, &K, 1);
    rd(in, &n, 1);
    rd(in, &W, 1);
    rd(in, &H, 1);
    rd(in, &V, 1);
    mv::PinholeScene sc;
    sc.count = K;
    sc.n = n;
    sc.position.resize(3 * K);
    sc.quat.resize(4 * K);
    sc.log_scale.resize(2 * K);
    sc.opacity_logit.resize(K);
    sc.grid.resize(K * 3 * n * n);
    rd(in, sc.position.data(), sc.position.size());
    rd(in, sc.quat.data(), sc.quat.size());
    rd(in, sc.log_scale.data(), sc.log_scale.size());
    rd(in, sc.opacity_logit.data(), sc.opacity_logit.size());
    rd(in, sc.grid.data(), sc.grid.size());
    std::vector<mv::PinholeCamera> cams(V);
    for (auto& c : cams) {
        c.width = W;
        c.height = H;
        double v[16];
        rd(in, v, 16);
        c.fx = v[0];
        c.fy = v[1];
        c.cx = v[2];
        c.cy = v[3];
        for (int i = 0; i < 9; ++i) c.rot[i] = v[4 + i];
        for (int i = 0; i < 3; ++i) c.trans[i] = v[13 + i];
    }
    std::vector<std::vector<float>> targets(V, std::vector<float>(static_cast<std::size_t>(W) * H * 3));
    for (auto& t : targets) rd(in, t.data(), t.size());
    const int steps = std::atoi(argv[3]);
    mv::StepConfig cfg;
    cfg.sharded_adam = std::atoi(argv[4]) != 0;
    cfg.lrs.position *= 6.0;  // the bench's position LR x scene extent
    std::vector<int> devices;
    for (int i = 5; i < argc; ++i) devices.push_back(std::atoi(argv[i]));
    if (devices.empty()) devices.push_back(0);
    std::vector<std::vector<float>> params;
    // single rank: also read the summed gradients of the last step back through a Rank directly
    std::vector<double> losses;
    std::vector<float> grads;
    mv::detail::FlatLayout lay(K, n, static_cast<int>(devices.size()));
    if (devices.size() == 1 && !cfg.sharded_adam) {
        mv::Rank r(devices[0], sc, cams, mv::shard_views(V, 0, 1), cfg, 1, 0);
        gb_context* ctx = r.context();
        gb_comm* comm = nullptr;
        gbil_b200::detail::check(gb_comm_init_all(&ctx, 1, &comm), "ncclCommInitAll");
        r.attach(comm);
        std::vector<std::unique_ptr<mv::detail::Buffer>> tb;
        std::vector<const float*> tp;
        for (int v = 0; v < V; ++v) {
            tb.push_back(std::make_unique<mv::detail::Buffer>(ctx, sizeof(float) * targets[v].size()));
            gbil_b200::detail::check(gb_copy_h2d(ctx, tb.back()->ptr, targets[v].data(), sizeof(float) * targets[v].size(), 1),
                                     "targets");
            tp.push_back(tb.back()->f());
        }
        for (int s = 0; s < steps; ++s) losses.push_back(r.step(tp));
        params.push_back(r.download_params());
        grads = r.download_grads();
        tb.clear();
        gb_comm_destroy(comm);
    } else {
        losses = mv::train(devices, sc, cams, [&](int v) { return targets[v]; }, steps, cfg, &params);
    }
    std::ofstream out(argv[2], std::ios::binary);
    out.write(reinterpret_cast<const char*>(losses.data()), sizeof(double) * losses.size());
    const std::int64_t T = static_cast<std::int64_t>(params[0].size());
    out.write(reinterpret_cast<const char*>(&T), sizeof(T));
    out.write(reinterpret_cast<const char*>(params[0].data()), sizeof(float) * T);
    if (grads.empty()) grads.assign(T, 0.0f);
    out.write(reinterpret_cast<const char*>(grads.data()), sizeof(float) * T);
    const std::int64_t offs[5] = {lay.position, lay.quat, lay.log_scale, lay.opacity, lay.grid};
    out.write(reinterpret_cast<const char*>(offs), sizeof(offs));
    std::printf("multiview ok: %d rank(s), %d steps, loss %.6f -> %.6f\n", static_cast<int>(devices.size()), steps,
                losses.front(), losses.back());
    return 0;
}
