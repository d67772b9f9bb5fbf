// gb_mvhost.cpp -- a C entry point to the C++ host of the view-sharded training step
// (include/gbil_b200.hpp, gbil_b200::multiview::Rank), so that bench.py and tests can drive the C++ host
// through ctypes.  Built as libgb_mvhost.so on top of libgb_raster.so; one rank per handle (world size 1;
// multi-GPU hosts use multiview::train or Rank + gb_comm_init_rank directly).
#include <cstring>
#include <memory>
#include <string>

#include "gbil_b200.hpp"

namespace mv = gbil_b200::multiview;

namespace {
thread_local std::string g_err;
}

extern "C" {

__attribute__((visibility("default"))) const char* gb_mv_error(void) { return g_err.c_str(); }

// cam16: per camera fx, fy, cx, cy, rot[9], trans[3] (doubles); views: the camera indices this rank owns.
__attribute__((visibility("default"))) int gb_mv_create(int device, int64_t K, int n, const float* position,
                                                        const float* quat, const float* log_scale,
                                                        const float* opacity, const float* grid, int W, int H,
                                                        int ncam, const double* cam16, int nviews,
                                                        const int* views, int lanes, int graph,
                                                        double position_lr_scale, void** out) {
    try {
        mv::PinholeScene sc;
        sc.count = K;
        sc.n = n;
        sc.position.assign(position, position + 3 * K);
        sc.quat.assign(quat, quat + 4 * K);
        sc.log_scale.assign(log_scale, log_scale + 2 * K);
        sc.opacity_logit.assign(opacity, opacity + K);
        sc.grid.assign(grid, grid + K * 3 * n * n);
        std::vector<mv::PinholeCamera> cams(ncam);
        for (int i = 0; i < ncam; ++i) {
            const double* c = cam16 + 16 * i;
            cams[i].width = W;
            cams[i].height = H;
            cams[i].fx = c[0];
            cams[i].fy = c[1];
            cams[i].cx = c[2];
            cams[i].cy = c[3];
            for (int j = 0; j < 9; ++j) cams[i].rot[j] = c[4 + j];
            for (int j = 0; j < 3; ++j) cams[i].trans[j] = c[13 + j];
        }
        mv::StepConfig cfg;
        cfg.lrs.position *= position_lr_scale;
        *out = new mv::Rank(device, sc, cams, std::vector<int>(views, views + nviews), cfg, 1, 0, lanes, graph != 0);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// One step with device-resident targets (HWC fp32, one per owned view); *loss = the views' summed L1.
__attribute__((visibility("default"))) int gb_mv_step(void* h, int nviews, const float* const* targets,
                                                      double* loss) {
    try {
        auto* r = static_cast<mv::Rank*>(h);
        const double l = r->step(std::vector<const float*>(targets, targets + nviews));
        if (loss) *loss = l;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// The end-to-end step: targets in (pinned) host memory, copied every step inside the call.
__attribute__((visibility("default"))) int gb_mv_step_host(void* h, int nviews, const float* const* host_targets,
                                                           double* loss) {
    try {
        auto* r = static_cast<mv::Rank*>(h);
        const double l = r->step_host(std::vector<const float*>(host_targets, host_targets + nviews));
        if (loss) *loss = l;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

__attribute__((visibility("default"))) int gb_mv_params(void* h, float* out, int64_t cap) {
    try {
        const std::vector<float> p = static_cast<mv::Rank*>(h)->download_params();
        std::memcpy(out, p.data(), sizeof(float) * std::min<int64_t>(cap, static_cast<int64_t>(p.size())));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

__attribute__((visibility("default"))) int gb_mv_destroy(void* h) {
    delete static_cast<mv::Rank*>(h);
    return 0;
}

}  // extern "C"
