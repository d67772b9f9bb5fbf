// gb_composite.cu -- K3 / K4 with several pixels per thread (the default
// compositors for tile sizes that are multiples of 8).
//
// One CTA per tile, ts*ts/PPT threads; each warp owns an 8 x (4*PPT) pixel
// block and each lane PPT vertically adjacent pixels of one column.  Headers,
// ids and texels are read through L1 (__ldg); there is no shared-memory
// staging and no CTA barrier, so warps finish independently.
//
// Why several pixels per thread: both kernels are issue-bound (ncu: 75-85 %
// issue-active, DRAM < 12 %), and a large part of the per-(warp, entry) cost
// does not depend on how many pixels the warp covers -- the list walk and
// alpha-box ballot, the header loads and, in K4, the warp reductions and the
// global reds.  With PPT = 2 a lane first sums its two pixels' gradient terms
// in registers, so one reduction serves 64 pixels instead of 32.
//
// K3 restates render_forward (raster.hpp:201-261) + bilinear
// (texture.hpp:49-66); K4 restates render_backward (raster.hpp:277-387) +
// adj_bilinear_accum (texture.hpp:77-111), with the per-(tile, rank) partial
// records replaced by warp reductions + red.global.add (see gb_raster.cu).
#include "gb_compose.cuh"

namespace gb {

constexpr int kPPT = 2;  // pixels per thread

// lane -> pixel p of the warp's 8 x (4 PPT) block
__device__ __forceinline__ void mp_pixel(int warp, int lane, int p, int ts, int tx, int ty, int& x, int& y) {
    const int wx = ts >> 3;  // 8-wide warp blocks per tile row
    x = tx * ts + (warp % wx) * 8 + (lane & 7);
    y = ty * ts + (warp / wx) * (4 * kPPT) + (lane >> 3) * kPPT + p;
}

// ---------------------------------------------------------------------------
// K3 forward
// ---------------------------------------------------------------------------
template <int MODE, int NT>
__global__ void __launch_bounds__(128) k_forward_mp(const uint2* __restrict__ ranges, const int32_t* __restrict__ values,
                                                    const ScreenHeader* __restrict__ hdr, const float* __restrict__ tex,
                                                    const CamConst cc, const RasterConst rc, int n_rt,
                                                    float* __restrict__ out_color, float* __restrict__ out_trans,
                                                    int32_t* __restrict__ out_last) {
    const int N = tex_n<NT>(n_rt);
    const int F = 3 * N * N;
    const int ts = rc.tile_size;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tile = blockIdx.x;
    const uint2 range = ranges[tile];
    const int total = (int)(range.y - range.x);
    const int tx = tile % rc.tiles_x, ty = tile / rc.tiles_x;
    int x[kPPT], y[kPPT];
    float T[kPPT], a0[kPPT], a1[kPPT], a2[kPPT];
    int last[kPPT];
    bool done[kPPT];
#pragma unroll
    for (int p = 0; p < kPPT; ++p) {
        mp_pixel(warp, lane, p, ts, tx, ty, x[p], y[p]);
        T[p] = 1.0f;
        a0[p] = a1[p] = a2[p] = 0.0f;
        last[p] = -1;
        done[p] = x[p] >= cc.width || y[p] >= cc.height;
    }
    // the warp's pixel block (pixel indices) for the alpha-box test
    const float bx0 = (float)__reduce_min_sync(kFull, x[0]), bx1 = (float)__reduce_max_sync(kFull, x[0]);
    const float by0 = (float)__reduce_min_sync(kFull, y[0]), by1 = (float)__reduce_max_sync(kFull, y[kPPT - 1]);
    bool all_done = __all_sync(kFull, done[0] && done[kPPT - 1]);
    for (int c0 = 0; c0 < total && !all_done; c0 += 32) {
        int idl = -1;
        bool pass = false;
        if (c0 + lane < total) {
            idl = __ldg(&values[range.x + c0 + lane]);
            pass = !box_miss(__ldg(&hdr[idl].h3), bx0, bx1, by0, by1);
        }
        unsigned mask = __ballot_sync(kFull, pass);
        while (mask) {
            const int bit = __ffs(mask) - 1;
            mask &= mask - 1;
            const int id = __shfl_sync(kFull, idl, bit);
            ScreenHeader h;
            h.h0 = __ldg(&hdr[id].h0);
            h.h1 = __ldg(&hdr[id].h1);
            h.h2 = __ldg(&hdr[id].h2);
            const float* t = tex + (size_t)id * F;
#pragma unroll
            for (int p = 0; p < kPPT; ++p) {
                if (done[p]) continue;
                float u, v;
                bool hit;
                if (MODE == GB_MODE_ORTHO) {
                    hit = eval_uv_ortho(h, x[p], y[p], u, v);
                } else {
                    PinholeTerms pt;
                    hit = eval_uv_pinhole(h, x[p], y[p], u, v, pt);
                }
                if (!hit) continue;
                const float alpha = fminf(__fmul_rn(h.h1.z, gauss_weight(u, v)), kMaxAlphaF);  // raster.hpp:241
                if (alpha < rc.alpha_skip) continue;                                             // raster.hpp:242
                float c0_, c1_, c2_;
                if (N == 1) {
                    c0_ = __ldg(t);
                    c1_ = __ldg(t + 1);
                    c2_ = __ldg(t + 2);
                } else {
                    Bilin b;
                    bilin_setup(u, v, N, rc, b);
                    const float* p00 = t + b.o00;
                    const float* p10 = p00 + 3 * N;
                    c0_ = __ldg(p00) * b.w00 + __ldg(p10) * b.w10 + __ldg(p00 + 3) * b.w01 + __ldg(p10 + 3) * b.w11;
                    c1_ = __ldg(p00 + 1) * b.w00 + __ldg(p10 + 1) * b.w10 + __ldg(p00 + 4) * b.w01 +
                          __ldg(p10 + 4) * b.w11;
                    c2_ = __ldg(p00 + 2) * b.w00 + __ldg(p10 + 2) * b.w10 + __ldg(p00 + 5) * b.w01 +
                          __ldg(p10 + 5) * b.w11;
                }
                const float w = alpha * T[p];  // raster.hpp:244-249
                a0[p] = fmaf(c0_, w, a0[p]);
                a1[p] = fmaf(c1_, w, a1[p]);
                a2[p] = fmaf(c2_, w, a2[p]);
                T[p] = __fmul_rn(T[p], __fsub_rn(1.0f, alpha));
                last[p] = c0 + bit;
                if (rc.early_stop > 0.0f && T[p] < rc.early_stop) done[p] = true;  // raster.hpp:250
            }
            all_done = __all_sync(kFull, done[0] && done[kPPT - 1]);
            if (all_done) break;
        }
    }
#pragma unroll
    for (int p = 0; p < kPPT; ++p) {
        if (x[p] < cc.width && y[p] < cc.height) {  // raster.hpp:253-254
            const size_t q = (size_t)y[p] * cc.width + x[p];
            out_color[q * 3 + 0] = fmaf(T[p], cc.bg[0], a0[p]);
            out_color[q * 3 + 1] = fmaf(T[p], cc.bg[1], a1[p]);
            out_color[q * 3 + 2] = fmaf(T[p], cc.bg[2], a2[p]);
            out_trans[q] = T[p];
            out_last[q] = last[p];
        }
    }
}

// ---------------------------------------------------------------------------
// K4 backward
// ---------------------------------------------------------------------------
// Per-pixel state of the back-to-front walk (raster.hpp:313-322).
struct BwdPx {
    int x, y, last;
    float T, g0, g1, g2, bh0, bh1, bh2;
};

// One (pixel, entry) evaluation of render_backward (raster.hpp:324-362) +
// adj_bilinear_accum (texture.hpp:77-111).  Adds the screen-space terms into
// red[], writes the 12 texel terms to tg[] (corner-major: 00, 10, 01, 11 x
// RGB) with their base offset, and advances the rewind state.  Returns false
// (and touches nothing) when the entry is skipped for this pixel.
template <int MODE, int NT>
__device__ __forceinline__ bool bwd_px(const ScreenHeader& h, const float* __restrict__ t, int N, int rank, BwdPx& s,
                                       const RasterConst& rc, float (&red)[10], float (&tg)[12], int& tbase) {
    if (rank > s.last) return false;
    float u, v;
    PinholeTerms pt;
    bool hit;
    if (MODE == GB_MODE_ORTHO) {
        hit = eval_uv_ortho(h, s.x, s.y, u, v);
    } else {
        hit = eval_uv_pinhole(h, s.x, s.y, u, v, pt);
    }
    if (!hit) return false;
    const float G = gauss_weight(u, v);
    const float araw = __fmul_rn(h.h1.z, G);
    const float alpha = fminf(araw, kMaxAlphaF);
    if (alpha < rc.alpha_skip) return false;  // raster.hpp:332
    const float om = __fsub_rn(1.0f, alpha);
    s.T = __fdividef(s.T, om);  // raster.hpp:333
    const float aT = alpha * s.T;
    const float ch0 = aT * s.g0, ch1 = aT * s.g1, ch2 = aT * s.g2;  // c_hat, raster.hpp:338-340
    float c0, c1, c2, u_hat = 0.0f, v_hat = 0.0f;
    if (N == 1) {
        c0 = __ldg(t);
        c1 = __ldg(t + 1);
        c2 = __ldg(t + 2);
        tg[0] = ch0;
        tg[1] = ch1;
        tg[2] = ch2;
#pragma unroll
        for (int i = 3; i < 12; ++i) tg[i] = 0.0f;
        tbase = 0;
    } else {
        Bilin b;
        bilin_setup(u, v, N, rc, b);
        const float* p00 = t + b.o00;
        const float* p10 = p00 + 3 * N;
        const float gu = 1.0f - b.fu, gv = 1.0f - b.fv;
        const float chat[3] = {ch0, ch1, ch2};
        float cc[3], fu_hat = 0.0f, fv_hat = 0.0f;
#pragma unroll
        for (int c = 0; c < 3; ++c) {  // texture.hpp:94-103
            const float c00 = __ldg(p00 + c), c10 = __ldg(p10 + c), c01 = __ldg(p00 + 3 + c), c11 = __ldg(p10 + 3 + c);
            cc[c] = c00 * b.w00 + c10 * b.w10 + c01 * b.w01 + c11 * b.w11;
            tg[c] = chat[c] * b.w00;
            tg[3 + c] = chat[c] * b.w10;
            tg[6 + c] = chat[c] * b.w01;
            tg[9 + c] = chat[c] * b.w11;
            fu_hat = fmaf(chat[c], (c10 - c00) * gv + (c11 - c01) * b.fv, fu_hat);
            fv_hat = fmaf(chat[c], (c01 - c00) * gu + (c11 - c10) * b.fu, fv_hat);
        }
        c0 = cc[0];
        c1 = cc[1];
        c2 = cc[2];
        tbase = b.o00;
        const float sigma = rc.sigma;  // texture.hpp:106-109 (strict mask)
        if (u > -sigma && u < sigma) u_hat = rc.tex_scale * fu_hat;
        if (v > -sigma && v < sigma) v_hat = rc.tex_scale * fv_hat;
    }
    // raster.hpp:344-346
    const float alpha_hat = s.T * (s.g0 * (c0 - s.bh0) + s.g1 * (c1 - s.bh1) + s.g2 * (c2 - s.bh2));
    float op = 0.0f;
    if (araw < kMaxAlphaF) {  // raster.hpp:350-354
        op = alpha_hat * G;
        const float aa = alpha_hat * alpha;
        u_hat -= aa * u;
        v_hat -= aa * v;
    }
    if (MODE == GB_MODE_ORTHO) {
        red[0] += u_hat;
        red[1] += v_hat;
        red[2] += u_hat * v;
        red[3] += v_hat * u;
        red[4] += u_hat * u;
        red[5] += v_hat * v;
        red[6] += op;
    } else {
        // (u, v) = (c_x, c_y) / c_z with c = E' + dx X + dy Y (K1 header)
        const float gc0 = u_hat * pt.iz, gc1 = v_hat * pt.iz, gc2 = -(u_hat * u + v_hat * v) * pt.iz;
        red[0] += gc0;
        red[1] += gc1;
        red[2] += gc2;
        red[3] += pt.dx * gc0;
        red[4] += pt.dx * gc1;
        red[5] += pt.dx * gc2;
        red[6] += pt.dy * gc0;
        red[7] += pt.dy * gc1;
        red[8] += pt.dy * gc2;
        red[9] += op;
    }
    s.bh0 = alpha * c0 + om * s.bh0;  // raster.hpp:362
    s.bh1 = alpha * c1 + om * s.bh1;
    s.bh2 = alpha * c2 + om * s.bh2;
    return true;
}

__device__ __forceinline__ void red_texels(float* gg, int base, int N, const float (&tg)[12]) {
    if (N == 1) {
        red3(gg, tg[0], tg[1], tg[2]);
        return;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (tg[3 * k] != 0.0f || tg[3 * k + 1] != 0.0f || tg[3 * k + 2] != 0.0f)
            red3(gg + base + corner_offset(3 * k, N), tg[3 * k], tg[3 * k + 1], tg[3 * k + 2]);
}

template <int MODE, int NT>
__global__ void __launch_bounds__(128) k_backward_mp(const uint2* __restrict__ ranges,
                                                     const int32_t* __restrict__ values,
                                                     const ScreenHeader* __restrict__ hdr,
                                                     const float* __restrict__ tex, const CamConst cc,
                                                     const RasterConst rc, int n_rt, const float* __restrict__ in_trans,
                                                     const int32_t* __restrict__ in_last,
                                                     const float* __restrict__ image_grad, float* __restrict__ accum,
                                                     float* __restrict__ grid_grad) {
    constexpr int NS = MODE == GB_MODE_ORTHO ? 7 : 10;  // screen-space sums per entry
    __shared__ __align__(16) float red_scratch[4 * kRedRows * kRedStride];
    const int N = tex_n<NT>(n_rt);
    const int F = 3 * N * N;
    const int ts = rc.tile_size;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tile = blockIdx.x;
    const uint2 range = ranges[tile];
    const int tx = tile % rc.tiles_x, ty = tile / rc.tiles_x;
    BwdPx px[kPPT];
    int wl = -1;
#pragma unroll
    for (int p = 0; p < kPPT; ++p) {  // raster.hpp:313-322
        BwdPx& s = px[p];
        mp_pixel(warp, lane, p, ts, tx, ty, s.x, s.y);
        s.last = -1;
        s.T = 1.0f;
        s.g0 = s.g1 = s.g2 = 0.0f;
        if (s.x < cc.width && s.y < cc.height) {
            const size_t q = (size_t)s.y * cc.width + s.x;
            s.last = in_last[q];
            s.g0 = image_grad[q * 3 + 0];
            s.g1 = image_grad[q * 3 + 1];
            s.g2 = image_grad[q * 3 + 2];
            s.T = in_trans[q];
            if (s.g0 == 0.0f && s.g1 == 0.0f && s.g2 == 0.0f) s.last = -1;
        }
        s.bh0 = cc.bg[0];
        s.bh1 = cc.bg[1];
        s.bh2 = cc.bg[2];
        wl = max(wl, s.last);
    }
    const float bx0 = (float)__reduce_min_sync(kFull, px[0].x), bx1 = (float)__reduce_max_sync(kFull, px[0].x);
    const float by0 = (float)__reduce_min_sync(kFull, px[0].y);
    const float by1 = (float)__reduce_max_sync(kFull, px[kPPT - 1].y);
    const int wlast = __reduce_max_sync(kFull, wl);  // this warp never needs ranks above it
    float* wscratch = red_scratch + warp * kRedRows * kRedStride;
    for (int c0 = wlast & ~31; c0 >= 0; c0 -= 32) {
        int idl = -1;
        bool pass = false;
        if (c0 + lane <= wlast) {
            idl = __ldg(&values[range.x + c0 + lane]);
            pass = !box_miss(__ldg(&hdr[idl].h3), bx0, bx1, by0, by1);
        }
        unsigned mask = __ballot_sync(kFull, pass);
        while (mask) {
            const int bit = 31 - __clz(mask);
            mask &= ~(1u << bit);
            const int id = __shfl_sync(kFull, idl, bit);
            const int rank = c0 + bit;
            ScreenHeader h;
            h.h0 = __ldg(&hdr[id].h0);
            h.h1 = __ldg(&hdr[id].h1);
            h.h2 = __ldg(&hdr[id].h2);
            const float* t = tex + (size_t)id * F;
            float red[10];
#pragma unroll
            for (int i = 0; i < 10; ++i) red[i] = 0.0f;
            float tgA[12], tgB[12];
            int baseA = -1, baseB = -1;
            bool onA = bwd_px<MODE, NT>(h, t, N, rank, px[0], rc, red, tgA, baseA);
            bool onB = bwd_px<MODE, NT>(h, t, N, rank, px[1], rc, red, tgB, baseB);
            if (!__any_sync(kFull, onA || onB)) continue;
            {  // screen-space sums: lane l owns value l >> 1
                float sv[NS];
#pragma unroll
                for (int i = 0; i < NS; ++i) sv[i] = red[i];
                const float r2 = smem_reduce<NS>(sv, wscratch, lane);
                if ((lane & 1) == 0 && (lane >> 1) < NS) red_add(accum + (size_t)id * kAccumStride + (lane >> 1), r2);
            }
            // texel terms: merge the lane's two pixels when they share a bilinear cell
            if (onB && (!onA || baseB == baseA)) {
#pragma unroll
                for (int i = 0; i < 12; ++i) tgA[i] = onA ? tgA[i] + tgB[i] : tgB[i];
                baseA = baseB;
                onA = true;
                onB = false;
            }
            float* gg = grid_grad + (size_t)id * F;
            const unsigned actA = __ballot_sync(kFull, onA);
            const int b0 = __shfl_sync(kFull, baseA, actA ? __ffs(actA) - 1 : 0);
            if (__all_sync(kFull, !onB && (!onA || baseA == b0))) {
                // every active pixel of the warp shares one cell: one warp reduction
                if (!onA) {
#pragma unroll
                    for (int i = 0; i < 12; ++i) tgA[i] = 0.0f;
                }
                const float r2 = smem_reduce<12>(tgA, wscratch, lane);
                if ((lane & 1) == 0 && lane < 24 && (N > 1 || lane < 6))
                    red_add(gg + b0 + corner_offset(lane >> 1, N), r2);
            } else {
                // otherwise each lane adds its (at most 2 x 4) non-zero texels straight to HBM
                if (onA) red_texels(gg, baseA, N, tgA);
                if (onB) red_texels(gg, baseB, N, tgB);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// launchers (tile sizes that are multiples of 8: 8 -> 1 warp, 16 -> 4 warps)
// ---------------------------------------------------------------------------
bool mp_supported(int ts) { return ts == 8 || ts == 16; }

#define GB_MP_DISPATCH(KERNEL, MODE, ...)                                      \
    switch (n) {                                                               \
        case 1: KERNEL<MODE, 1><<<tiles, threads, 0, st>>>(__VA_ARGS__); break; \
        case 2: KERNEL<MODE, 2><<<tiles, threads, 0, st>>>(__VA_ARGS__); break; \
        case 4: KERNEL<MODE, 4><<<tiles, threads, 0, st>>>(__VA_ARGS__); break; \
        case 8: KERNEL<MODE, 8><<<tiles, threads, 0, st>>>(__VA_ARGS__); break; \
        case 16: KERNEL<MODE, 16><<<tiles, threads, 0, st>>>(__VA_ARGS__); break; \
        default: KERNEL<MODE, 0><<<tiles, threads, 0, st>>>(__VA_ARGS__); break; \
    }

cudaError_t launch_forward_mp(int mode, int n, int tiles, int ts, const uint2* ranges, const int32_t* values,
                              const ScreenHeader* hdr, const float* tex, const CamConst& cc, const RasterConst& rc,
                              float* color, float* trans, int32_t* last, cudaStream_t st) {
    const int threads = ts * ts / kPPT;
    if (mode == GB_MODE_ORTHO) {
        GB_MP_DISPATCH(k_forward_mp, GB_MODE_ORTHO, ranges, values, hdr, tex, cc, rc, n, color, trans, last)
    } else {
        GB_MP_DISPATCH(k_forward_mp, GB_MODE_PINHOLE, ranges, values, hdr, tex, cc, rc, n, color, trans, last)
    }
    return cudaGetLastError();
}

cudaError_t launch_backward_mp(int mode, int n, int tiles, int ts, const uint2* ranges, const int32_t* values,
                               const ScreenHeader* hdr, const float* tex, const CamConst& cc, const RasterConst& rc,
                               const float* trans, const int32_t* last, const float* image_grad, float* accum,
                               float* grid_grad, cudaStream_t st) {
    const int threads = ts * ts / kPPT;
    if (mode == GB_MODE_ORTHO) {
        GB_MP_DISPATCH(k_backward_mp, GB_MODE_ORTHO, ranges, values, hdr, tex, cc, rc, n, trans, last, image_grad,
                       accum, grid_grad)
    } else {
        GB_MP_DISPATCH(k_backward_mp, GB_MODE_PINHOLE, ranges, values, hdr, tex, cc, rc, n, trans, last, image_grad,
                       accum, grid_grad)
    }
    return cudaGetLastError();
}

}  // namespace gb
