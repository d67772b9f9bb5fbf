// gb_composite.cu -- K3 / K4 with sub-warp groups (the default compositors
// for 16x16 and 8x8 tiles).
//
// One CTA per tile, one thread per pixel.  Each warp (an 8x4 pixel block) is
// split into 32/G groups of G lanes; a group owns a small pixel block (2x2
// for G = 4, 4x2 for G = 8, 4x4 for G = 16) and walks the tile's sorted list
// on its own cursor.  When a group's window is used up the whole warp refills
// it: 32 lanes test the group's next 32 entries against its block with the
// exact alpha-skip-ellipse test (K1 alpha_ellipse, one entry per lane, one
// ballot) and park the ids in shared memory.  Then every group composites its
// next passing entry, all groups of a warp in the same step.
//
// Why: K3/K4 are issue-bound and, with a whole warp on one entry, only ~11 of
// 32 lanes do useful work on an average (warp, entry) step at configs[2]
// (profiles/k4_counters_r01_s3.txt): most surfels cover a few pixels, and the
// alpha-box test can only cull at the granularity of the warp's 8x4 block.
// Groups cull at the granularity of their own block and several entries are
// composited per step, so the steps per warp drop to the largest group's list
// instead of the union of all of them (tools/sim_steps.py: 0.63x of the union
// for G = 8 with exact culling).
//
// K4 reduces each step's per-lane gradient terms with one shared-memory
// transpose per warp that yields one sum per (value, group): V x 32/G sums,
// owned by distinct lanes, each issuing one red.global.add.  Texel terms go
// through the same reduction for groups whose active pixels share a bilinear
// cell, and straight to HBM with per-lane vector reds otherwise.
//
// K3 restates render_forward (raster.hpp:201-261) + bilinear
// (texture.hpp:49-66); K4 restates render_backward (raster.hpp:277-387) +
// adj_bilinear_accum (texture.hpp:77-111).
#include <cstdlib>
#include <cstring>

#include "gb_compose.cuh"

namespace gb {

template <int G>
__device__ __forceinline__ unsigned group_mask(int lane) {
    return G == 32 ? kFull : (((1u << G) - 1u) << (lane & ~(G - 1)));
}

// Group block: BW x BH pixels (G = 4: 2x2, G = 8: 4x2, G = 16: 4x4), tiled
// row-major over the warp's 8x4 block.
template <int G>
struct GroupShape {
    static constexpr int BW = G == 4 ? 2 : 4;
    static constexpr int BH = G / BW;
    static constexpr int PER_ROW = 8 / BW;
};

// origin of group g's block inside its warp's 8x4 block
template <int G>
__device__ __forceinline__ void group_origin(int g, int& gx, int& gy) {
    gx = (g % GroupShape<G>::PER_ROW) * GroupShape<G>::BW;
    gy = (g / GroupShape<G>::PER_ROW) * GroupShape<G>::BH;
}

// origin of warp w's 8x4 block in the image
__device__ __forceinline__ void warp_origin(int tid, int ts, int tx, int ty, int& wx0, int& wy0) {
    const int warp = tid >> 5, wx = ts >> 3;
    wx0 = tx * ts + (warp % wx) * 8;
    wy0 = ty * ts + (warp / wx) * 4;
}

// lane -> pixel of the tile
template <int G>
__device__ __forceinline__ void group_pixel(int tid, int ts, int tx, int ty, int& x, int& y) {
    const int lane = tid & 31;
    int wx0, wy0, gx, gy;
    warp_origin(tid, ts, tx, ty, wx0, wy0);
    group_origin<G>(lane / G, gx, gy);
    const int i = lane % G;
    x = wx0 + gx + i % GroupShape<G>::BW;
    y = wy0 + gy + i / GroupShape<G>::BW;
}

// ---------------------------------------------------------------------------
// The walk: a ring of two shared 32-entry windows per warp.  The warp tests a
// window's 32 entries (one per lane) against every group's block with the
// exact alpha-skip-ellipse test and parks the ids and the per-group pass masks
// in shared memory; each group then consumes its own mask, one entry per step,
// and moves to the next window as soon as it is done -- at most one window
// ahead of the slowest group (tools/sim_steps.py "ring2": within 1 % of fully
// independent group cursors, at one test round per 32 entries for all groups).
// Forward windows run front to back over [0, total); backward windows back to
// front over [0, L) with L = 1 + the warp's largest last rank.
// ---------------------------------------------------------------------------
template <int G>
struct WarpRing {
    int ids[2][32];
    unsigned masks[2][32 / G];
    int glast[32 / G];  // backward: the largest last rank of each group's pixels
};

// Group walk state (every field uniform across the group's lanes).
struct GroupWalk {
    int w;          // absolute index of the window being consumed (-1 before the first)
    unsigned pend;  // entries of window w still to composite (bit i <-> i-th rank of the window)
    bool fin;       // group finished (forward: every pixel terminated early)
};

// Window k: ranks first, first + dir, ... (count of them); dir = +1 forward, -1 backward.
template <int G, bool BWD>
__device__ __forceinline__ void ring_fill(WarpRing<G>& ring, int k, int first, int count, const int32_t* values,
                                          uint32_t base, const CullRec* __restrict__ cull, int wx0, int wy0,
                                          int lane) {
    constexpr int NG = 32 / G;
    const int r = BWD ? first - lane : first + lane;
    const bool valid = lane < count;
    int id = -1;
    float4 ca = make_float4(0.f, 0.f, 0.f, 0.f), cb = ca;
    if (valid) {
        id = __ldg(&values[base + r]);
        ca = __ldg(&cull[id].a);
        cb = __ldg(&cull[id].b);
    }
    ring.ids[k & 1][lane] = id;
#pragma unroll
    for (int g = 0; g < NG; ++g) {
        int gx, gy;
        group_origin<G>(g, gx, gy);
        const float x0 = (float)(wx0 + gx) - 0.05f, y0 = (float)(wy0 + gy) - 0.05f;
        const bool pass = valid && (!BWD || r <= ring.glast[g]) &&
                          ellipse_meets_rect(ca, cb, x0, x0 + (float)(GroupShape<G>::BW - 1) + 0.1f, y0,
                                             y0 + (float)(GroupShape<G>::BH - 1) + 0.1f);
        const unsigned m = __ballot_sync(kFull, pass);
        if (lane == 0) ring.masks[k & 1][g] = m;
    }
}

// Advance every group whose mask is used up, filling windows as needed.
// wc = windows filled so far (warp-uniform), nwin = windows in the walk.
template <int G, bool BWD>
__device__ __forceinline__ void ring_advance(WarpRing<G>& ring, GroupWalk& gw, int& wc, int nwin, int span,
                                             const int32_t* values, uint32_t base, const CullRec* __restrict__ cull,
                                             int wx0, int wy0, int lane) {
    const int g = lane / G;
    for (;;) {
        for (;;) {  // consume filled windows
            const bool adv = !gw.fin && gw.pend == 0 && gw.w + 1 < wc;
            if (!__any_sync(kFull, adv)) break;
            if (adv) {
                ++gw.w;
                gw.pend = ring.masks[gw.w & 1][g];
            }
        }
        const bool want = !gw.fin && gw.pend == 0 && gw.w + 1 == wc && wc < nwin;
        if (!__any_sync(kFull, want)) break;
        // slot wc & 1 still holds window wc - 2 while a group consumes it
        if (__reduce_min_sync(kFull, gw.fin ? 0x7fffffff : gw.w) < wc - 1) break;
        const int first = BWD ? span - 1 - 32 * wc : 32 * wc;
        __syncwarp();  // readers of the slot being refilled are done
        ring_fill<G, BWD>(ring, wc, first, min(32, span - 32 * wc), values, base, cull, wx0, wy0, lane);
        __syncwarp();
        ++wc;
    }
}

// Sum of NV per-lane values per group: returns, in out[k], the total of value
// row(q) over the lanes of group grp(q) for pair q = lane + 32 k, q < NV * 32/G
// (row = q / (32/G), grp = q % (32/G)); scratch = kRedRows x kRedStride floats.
template <int NV, int G>
__device__ __forceinline__ void group_reduce(const float (&v)[NV], float* scratch, int lane,
                                             float (&out)[(NV * (32 / G) + 31) / 32]) {
    constexpr int NG = 32 / G;
    constexpr int PASSES = (NV * NG + 31) / 32;
    __syncwarp();
#pragma unroll
    for (int i = 0; i < NV; ++i) scratch[i * kRedStride + lane] = v[i];
    __syncwarp();
#pragma unroll
    for (int k = 0; k < PASSES; ++k) {
        const int q = lane + 32 * k;
        float acc = 0.0f;
        if (q < NV * NG) {
            const float4* p = reinterpret_cast<const float4*>(scratch + (q / NG) * kRedStride + (q % NG) * G);
#pragma unroll
            for (int j = 0; j < G / 4; ++j) {
                const float4 a = p[j];
                acc += (a.x + a.y) + (a.z + a.w);
            }
        }
        out[k] = acc;
    }
}

// ---------------------------------------------------------------------------
// K3 forward
// ---------------------------------------------------------------------------
template <int MODE, int NT, int G>
__global__ void __launch_bounds__(256) k_forward_grp(const uint2* __restrict__ ranges,
                                                     const int32_t* __restrict__ values,
                                                     const ScreenHeader* __restrict__ hdr,
                                                     const CullRec* __restrict__ cull, const float* __restrict__ tex,
                                                     const CamConst cc, const RasterConst rc, int n_rt,
                                                     float* __restrict__ out_color, float* __restrict__ out_trans,
                                                     int32_t* __restrict__ out_last) {
    constexpr int NG = 32 / G;
    __shared__ WarpRing<G> s_ring[8];
    const int N = tex_n<NT>(n_rt);
    const int F = 3 * N * N;
    const int ts = rc.tile_size;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned gm = group_mask<G>(lane);
    const int tile = blockIdx.x;
    const uint2 range = ranges[tile];
    const int total = (int)(range.y - range.x);
    const int tx = tile % rc.tiles_x, ty = tile / rc.tiles_x;
    int x, y, wx0, wy0;
    group_pixel<G>(threadIdx.x, ts, tx, ty, x, y);
    warp_origin(threadIdx.x, ts, tx, ty, wx0, wy0);
    const bool inside = x < cc.width && y < cc.height;
    float T = 1.0f, acc0 = 0.0f, acc1 = 0.0f, acc2 = 0.0f;
    int last = -1;
    bool done = !inside;
    WarpRing<G>& ring = s_ring[warp];
    const int nwin = (total + 31) / 32;
    int wc = 0;
    GroupWalk gw{-1, 0u, __all_sync(gm, done) != 0};  // a group with no pixel in the image has nothing to do
    for (;;) {
        ring_advance<G, false>(ring, gw, wc, nwin, total, values, range.x, cull, wx0, wy0, lane);
        if (!__any_sync(kFull, gw.pend != 0)) break;
        if (gw.pend != 0) {
            const int bit = __ffs(gw.pend) - 1;
            gw.pend &= gw.pend - 1;
            if (!done) {
                const int id = ring.ids[gw.w & 1][bit];
                ScreenHeader h;
                h.h0 = __ldg(&hdr[id].h0);
                h.h1 = __ldg(&hdr[id].h1);
                h.h2 = __ldg(&hdr[id].h2);
                float u, v;
                bool hit;
                if (MODE == GB_MODE_ORTHO) {
                    hit = eval_uv_ortho(h, x, y, u, v);
                } else {
                    PinholeTerms pt;
                    hit = eval_uv_pinhole(h, x, y, u, v, pt);
                }
                if (hit) {
                    const float alpha = fminf(__fmul_rn(h.h1.z, gauss_weight(u, v)), kMaxAlphaF);  // raster.hpp:241
                    if (!(alpha < rc.alpha_skip)) {                                                  // raster.hpp:242
                        const float* t = tex + (size_t)id * F;
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
                            c0_ = __ldg(p00) * b.w00 + __ldg(p10) * b.w10 + __ldg(p00 + 3) * b.w01 +
                                  __ldg(p10 + 3) * b.w11;
                            c1_ = __ldg(p00 + 1) * b.w00 + __ldg(p10 + 1) * b.w10 + __ldg(p00 + 4) * b.w01 +
                                  __ldg(p10 + 4) * b.w11;
                            c2_ = __ldg(p00 + 2) * b.w00 + __ldg(p10 + 2) * b.w10 + __ldg(p00 + 5) * b.w01 +
                                  __ldg(p10 + 5) * b.w11;
                        }
                        const float w = alpha * T;  // raster.hpp:244-249
                        acc0 = fmaf(c0_, w, acc0);
                        acc1 = fmaf(c1_, w, acc1);
                        acc2 = fmaf(c2_, w, acc2);
                        T = __fmul_rn(T, __fsub_rn(1.0f, alpha));
                        last = 32 * gw.w + bit;
                        if (rc.early_stop > 0.0f && T < rc.early_stop) done = true;  // raster.hpp:250
                    }
                }
            }
        }
        if (__all_sync(gm, done)) {  // the whole group terminated early
            gw.fin = true;
            gw.pend = 0;
        }
    }
    if (inside) {  // raster.hpp:253-254
        const size_t q = (size_t)y * cc.width + x;
        out_color[q * 3 + 0] = fmaf(T, cc.bg[0], acc0);
        out_color[q * 3 + 1] = fmaf(T, cc.bg[1], acc1);
        out_color[q * 3 + 2] = fmaf(T, cc.bg[2], acc2);
        out_trans[q] = T;
        out_last[q] = last;
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
// adj_bilinear_accum (texture.hpp:77-111).  Writes the screen-space terms to
// red[], the 12 texel terms to tg[] (corner-major: 00, 10, 01, 11 x RGB) with
// their base offset, and advances the rewind state.  Returns false (and
// leaves red/tg untouched) when the entry is skipped for this pixel.
template <int MODE, int NT>
__device__ __forceinline__ bool bwd_px(const ScreenHeader& h, const float* __restrict__ t, int N, BwdPx& s,
                                       const RasterConst& rc, float (&red)[10], float (&tg)[12], int& tbase) {
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
    s.T = __fmul_rn(s.T, rcp_approx(om));  // raster.hpp:333
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
        red[0] = u_hat;
        red[1] = v_hat;
        red[2] = u_hat * v;
        red[3] = v_hat * u;
        red[4] = u_hat * u;
        red[5] = v_hat * v;
        red[6] = op;
    } else {
        // (u, v) = (c_x, c_y) / c_z with c = E' + dx X + dy Y (K1 header)
        const float gc0 = u_hat * pt.iz, gc1 = v_hat * pt.iz, gc2 = -(u_hat * u + v_hat * v) * pt.iz;
        red[0] = gc0;
        red[1] = gc1;
        red[2] = gc2;
        red[3] = pt.dx * gc0;
        red[4] = pt.dx * gc1;
        red[5] = pt.dx * gc2;
        red[6] = pt.dy * gc0;
        red[7] = pt.dy * gc1;
        red[8] = pt.dy * gc2;
        red[9] = op;
    }
    s.bh0 = alpha * c0 + om * s.bh0;  // raster.hpp:362
    s.bh1 = alpha * c1 + om * s.bh1;
    s.bh2 = alpha * c2 + om * s.bh2;
    return true;
}

template <int MODE, int NT, int G, bool UNI>
__global__ void __launch_bounds__(256, 4) k_backward_grp(const uint2* __restrict__ ranges,
                                                      const int32_t* __restrict__ values,
                                                      const ScreenHeader* __restrict__ hdr,
                                                      const CullRec* __restrict__ cull,
                                                      const float* __restrict__ tex, const CamConst cc,
                                                      const RasterConst rc, int n_rt,
                                                      const float* __restrict__ in_trans,
                                                      const int32_t* __restrict__ in_last,
                                                      const float* __restrict__ image_grad, float* __restrict__ accum,
                                                      float* __restrict__ grid_grad) {
    constexpr int NS = MODE == GB_MODE_ORTHO ? 7 : 10;  // screen-space sums per entry
    constexpr int NG = 32 / G;                          // groups per warp
    constexpr int PS = (NS * NG + 31) / 32;             // reduction passes (screen sums)
    constexpr int PT = (12 * NG + 31) / 32;             // reduction passes (texels)
    __shared__ __align__(16) float red_scratch[8 * kRedRows * kRedStride];
    __shared__ WarpRing<G> s_ring[8];
    const int N = tex_n<NT>(n_rt);
    const int F = 3 * N * N;
    const int ts = rc.tile_size;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned gm = group_mask<G>(lane);
    const int tile = blockIdx.x;
    const uint2 range = ranges[tile];
    const int tx = tile % rc.tiles_x, ty = tile / rc.tiles_x;
    int wx0, wy0;
    warp_origin(threadIdx.x, ts, tx, ty, wx0, wy0);
    BwdPx s;
    group_pixel<G>(threadIdx.x, ts, tx, ty, s.x, s.y);
    s.last = -1;
    s.T = 1.0f;
    s.g0 = s.g1 = s.g2 = 0.0f;
    if (s.x < cc.width && s.y < cc.height) {  // raster.hpp:313-322
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
    float* wscratch = red_scratch + warp * kRedRows * kRedStride;
    WarpRing<G>& ring = s_ring[warp];
    // the warp walks ranks [0, span) back to front; a group never needs ranks above its own largest last
    const int span = __reduce_max_sync(kFull, s.last) + 1;
    const int nwin = (span + 31) / 32;
    const int gl = __reduce_max_sync(gm, s.last);
    if (lane % G == 0) ring.glast[lane / G] = gl;
    __syncwarp();
    int wc = 0;
    GroupWalk gw{-1, 0u, false};
    for (;;) {
        ring_advance<G, true>(ring, gw, wc, nwin, span, values, range.x, cull, wx0, wy0, lane);
        if (!__any_sync(kFull, gw.pend != 0)) break;
        int id = -1;
        bool on = false;
        float red[10] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // inactive lanes add zeros
        float tg[12];
        int tbase = 0;
        if (gw.pend != 0) {
            const int bit = __ffs(gw.pend) - 1;
            gw.pend &= gw.pend - 1;
            id = ring.ids[gw.w & 1][bit];
            if (span - 1 - 32 * gw.w - bit <= s.last) {
                ScreenHeader h;
                h.h0 = __ldg(&hdr[id].h0);
                h.h1 = __ldg(&hdr[id].h1);
                h.h2 = __ldg(&hdr[id].h2);
                on = bwd_px<MODE, NT>(h, tex + (size_t)id * F, N, s, rc, red, tg, tbase);
            }
        }
        const unsigned act = __ballot_sync(kFull, on);
        if (act == 0) continue;
        {  // screen-space sums: one per (value, group), owned by distinct lanes
            float sv[NS];
#pragma unroll
            for (int i = 0; i < NS; ++i) sv[i] = red[i];
            float r2[PS];
            group_reduce<NS, G>(sv, wscratch, lane, r2);
#pragma unroll
            for (int k = 0; k < PS; ++k) {
                const int q = lane + 32 * k;
                const int src = (q % NG) * G;
                const int gid = __shfl_sync(kFull, id, src);
                if (q < NS * NG && ((act >> src) & group_mask<G>(0)))
                    red_add(accum + (size_t)gid * kAccumStride + q / NG, r2[k]);
            }
        }
        // texel terms (UNI): one reduction for the groups whose active pixels share a bilinear cell;
        // otherwise (and always without UNI) each lane adds its non-zero texels straight to HBM
        bool uni = false;
        if (UNI) {
            const unsigned gact = act & gm;
            const int b0 = __shfl_sync(kFull, tbase, gact ? __ffs(gact) - 1 : lane);
            const unsigned mixed = __ballot_sync(kFull, on && tbase != b0);
            uni = (mixed & gm) == 0 && gact != 0;
            const unsigned unimask = __ballot_sync(kFull, uni);
            if (unimask) {
                float tv[12];
#pragma unroll
                for (int i = 0; i < 12; ++i) tv[i] = (uni && on) ? tg[i] : 0.0f;
                float r2[PT];
                group_reduce<12, G>(tv, wscratch, lane, r2);
#pragma unroll
                for (int k = 0; k < PT; ++k) {
                    const int q = lane + 32 * k;
                    const int src = (q % NG) * G;
                    const int gid = __shfl_sync(kFull, id, src);
                    const int gb0 = __shfl_sync(kFull, b0, src);
                    if (q < 12 * NG && ((unimask >> src) & 1u) && (N > 1 || q / NG < 3))
                        red_add(grid_grad + (size_t)gid * F + gb0 + corner_offset(q / NG, N), r2[k]);
                }
            }
        }
        if (on && !uni) {  // mixed cells: each lane adds its (at most four) non-zero texels straight to HBM
            float* gg = grid_grad + (size_t)id * F;
            if (N == 1) {
                red3(gg, tg[0], tg[1], tg[2]);
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (tg[3 * k] != 0.0f || tg[3 * k + 1] != 0.0f || tg[3 * k + 2] != 0.0f)
                        red3(gg + tbase + corner_offset(3 * k, N), tg[3 * k], tg[3 * k + 1], tg[3 * k + 2]);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// launchers (16x16 tiles: 8 warps; 8x8 tiles: 2 warps)
// ---------------------------------------------------------------------------
bool grp_supported(int ts) { return ts == 8 || ts == 16; }

static int group_size() {  // GB_GROUP=4|8|16 (A/B); default 8
    const char* v = getenv("GB_GROUP");
    const int g = v ? atoi(v) : 8;
    return (g == 4 || g == 16) ? g : 8;
}

#define GB_GRP_DISPATCH(KERNEL, MODE, G, ...)                                      \
    switch (n) {                                                                   \
        case 1: KERNEL<MODE, 1, G><<<tiles, threads, 0, st>>>(__VA_ARGS__); break;   \
        case 2: KERNEL<MODE, 2, G><<<tiles, threads, 0, st>>>(__VA_ARGS__); break;   \
        case 4: KERNEL<MODE, 4, G><<<tiles, threads, 0, st>>>(__VA_ARGS__); break;   \
        case 8: KERNEL<MODE, 8, G><<<tiles, threads, 0, st>>>(__VA_ARGS__); break;   \
        case 16: KERNEL<MODE, 16, G><<<tiles, threads, 0, st>>>(__VA_ARGS__); break; \
        default: KERNEL<MODE, 0, G><<<tiles, threads, 0, st>>>(__VA_ARGS__); break;  \
    }

#define GB_GRP_G(KERNEL, MODE, ...)                                 \
    switch (group_size()) {                                         \
        case 4: GB_GRP_DISPATCH(KERNEL, MODE, 4, __VA_ARGS__) break;   \
        case 16: GB_GRP_DISPATCH(KERNEL, MODE, 16, __VA_ARGS__) break; \
        default: GB_GRP_DISPATCH(KERNEL, MODE, 8, __VA_ARGS__) break;  \
    }

#define GB_GRP_DISPATCH4(KERNEL, MODE, G, UNI, ...)                                      \
    switch (n) {                                                                         \
        case 1: KERNEL<MODE, 1, G, UNI><<<tiles, threads, 0, st>>>(__VA_ARGS__); break;   \
        case 2: KERNEL<MODE, 2, G, UNI><<<tiles, threads, 0, st>>>(__VA_ARGS__); break;   \
        case 4: KERNEL<MODE, 4, G, UNI><<<tiles, threads, 0, st>>>(__VA_ARGS__); break;   \
        case 8: KERNEL<MODE, 8, G, UNI><<<tiles, threads, 0, st>>>(__VA_ARGS__); break;   \
        case 16: KERNEL<MODE, 16, G, UNI><<<tiles, threads, 0, st>>>(__VA_ARGS__); break; \
        default: KERNEL<MODE, 0, G, UNI><<<tiles, threads, 0, st>>>(__VA_ARGS__); break;  \
    }

// backward: G and the texel strategy (GB_GRP_TEXEL=uni: shared-cell reductions, default: per-lane reds)
#define GB_GRP_B(KERNEL, MODE, ...)                                                                      \
    {                                                                                                    \
        const char* tv_ = getenv("GB_GRP_TEXEL");                                                         \
        const bool uni_ = tv_ && !strcmp(tv_, "uni");                                                     \
        switch (group_size() * 2 + (uni_ ? 1 : 0)) {                                                      \
            case 8: GB_GRP_DISPATCH4(KERNEL, MODE, 4, false, __VA_ARGS__) break;                          \
            case 9: GB_GRP_DISPATCH4(KERNEL, MODE, 4, true, __VA_ARGS__) break;                           \
            case 32: GB_GRP_DISPATCH4(KERNEL, MODE, 16, false, __VA_ARGS__) break;                        \
            case 33: GB_GRP_DISPATCH4(KERNEL, MODE, 16, true, __VA_ARGS__) break;                         \
            case 17: GB_GRP_DISPATCH4(KERNEL, MODE, 8, true, __VA_ARGS__) break;                          \
            default: GB_GRP_DISPATCH4(KERNEL, MODE, 8, false, __VA_ARGS__) break;                         \
        }                                                                                                \
    }

cudaError_t launch_forward_grp(int mode, int n, int tiles, int ts, const uint2* ranges, const int32_t* values,
                               const ScreenHeader* hdr, const CullRec* cull, const float* tex, const CamConst& cc,
                               const RasterConst& rc, float* color, float* trans, int32_t* last, cudaStream_t st) {
    const int threads = ts * ts;
    if (mode == GB_MODE_ORTHO) {
        GB_GRP_G(k_forward_grp, GB_MODE_ORTHO, ranges, values, hdr, cull, tex, cc, rc, n, color, trans, last)
    } else {
        GB_GRP_G(k_forward_grp, GB_MODE_PINHOLE, ranges, values, hdr, cull, tex, cc, rc, n, color, trans, last)
    }
    return cudaGetLastError();
}

cudaError_t launch_backward_grp(int mode, int n, int tiles, int ts, const uint2* ranges, const int32_t* values,
                                const ScreenHeader* hdr, const CullRec* cull, const float* tex, const CamConst& cc,
                                const RasterConst& rc, const float* trans, const int32_t* last,
                                const float* image_grad, float* accum, float* grid_grad, cudaStream_t st) {
    const int threads = ts * ts;
    if (mode == GB_MODE_ORTHO) {
        GB_GRP_B(k_backward_grp, GB_MODE_ORTHO, ranges, values, hdr, cull, tex, cc, rc, n, trans, last, image_grad,
                 accum, grid_grad)
    } else {
        GB_GRP_B(k_backward_grp, GB_MODE_PINHOLE, ranges, values, hdr, cull, tex, cc, rc, n, trans, last,
                 image_grad, accum, grid_grad)
    }
    return cudaGetLastError();
}

}  // namespace gb
