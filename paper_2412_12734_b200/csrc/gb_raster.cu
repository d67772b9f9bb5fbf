// gb_raster.cu -- K3 (per-tile forward compositor) and K4 (per-tile
// back-to-front backward), fp32, sm_100a.
//
// One CTA per tile (tile size 1..16), one thread per pixel; with 8-multiple
// tiles each warp owns an 8x4 pixel block.  Every warp walks the tile's sorted
// list on its own through L1: per 32 entries it loads ids and cull records,
// tests its pixel rectangle against each entry's exact alpha-skip ellipse (K1
// alpha_ellipse) and ballots; then it composites the passing entries one at a
// time.  No CTA barrier.  (Measured alternatives -- TMA-staged headers and
// textures, sub-warp pixel groups, one fused forward+backward kernel -- are in
// DESIGN.md §5; only compile-time variants built by tools/build_variant.sh
// remain, never a runtime switch.)
//
// K3 restates render_forward (raster.hpp:201-261) + bilinear
// (texture.hpp:49-66); K4 restates render_backward (raster.hpp:277-387) +
// adj_bilinear_accum (texture.hpp:77-111).  In the walks each entry is
// shaded in one of four texel footprint classes (bwd_shade): lanes outside the
// |u|, |v| < sigma texture square are clamped to one texel row/column, so a warp
// whose active lanes never interpolate along an axis loads and scatters 1 or 2
// texels per pixel instead of 4.  Instead of the reference's per-(tile, rank)
// partial records and ordered reduction, K4 adds each entry's per-pixel
// contributions with red.global.add into (a) the caller's texel gradients and
// (b) a 48 B per-primitive screen-space accumulator that K5 chains to the raw
// parameters: straight from every active lane when at most kDirectLanes lanes
// are active, else after a warp reduction (a shared-memory transpose, lane l
// summing half of row l/2).
#include <climits>

#include "gb_compose.cuh"

namespace gb {

// K4 warp-entries with at most this many active lanes add per lane instead of reducing first (B200 sweep
// of 0..32 at configs[3]: 0 = always reduce 575 MP/s, 8 = 605, 12 = 607, 16 = 605, 24 = 586, 32 = 453;
// re-swept after the footprint classes: 10 -> 719.1, 12 -> 718.8, 14 -> 716.1, 16 -> 712.1; with RGBA texels
// at 5 CTAs/SM: 10 -> 859.8, 12 -> 858.6, 14 -> 854.7; after the shared-memory id staging: 8 -> 888.2,
// 10 -> 892.2, 12 -> 893.3, 14 -> 891.5)
#ifndef GB_K4_DIRECT_LANES
#define GB_K4_DIRECT_LANES 12
#endif
constexpr int kDirectLanes = GB_K4_DIRECT_LANES;

#ifdef GB_DEBUG_COUNTERS
// development counters (not built by default): [0] warp-entries tested, [1] passing the box,
// [2] with an active lane, [3] active lanes, [4] uniform-cell texel groups, [5] per-lane texel groups,
// [6] active entries with both 4x4 halves active, [7] with both 8x2 halves active
__device__ unsigned long long g_dbg[8];
#define GB_DBG(i, v) atomicAdd(&g_dbg[i], (unsigned long long)(v))
extern "C" __attribute__((visibility("default"))) int gb_debug_counters(unsigned long long* out, int reset) {
    cudaMemcpyFromSymbol(out, g_dbg, sizeof(g_dbg));
    if (reset) {
        unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        cudaMemcpyToSymbol(g_dbg, z, sizeof(z));
    }
    return 0;
}
#else
#define GB_DBG(i, v)
#endif


// ---------------------------------------------------------------------------
// K4 backward
// ---------------------------------------------------------------------------
// One backward entry for the calling warp: evaluate, update the pixel's
// rewind state, reduce and scatter the gradients (raster.hpp:324-363).
// Texel footprint class of a warp-entry (texture.hpp:27-47).  A lane whose |u| >= sigma sits where the
// clamp pins u' to 0 or n-1: f_u is exactly 0 or 1, one texel row carries all the weight and the u
// adjoint is masked (texture.hpp:106-109); likewise for v.  When no active lane of the warp needs
// interpolation along u (v), the bilinear cell degenerates to a texel pair or a single texel and the
// warp skips the loads, products and reductions of the zero-weight corners.  In a configs[3] view 27 %
// of warp-entries need one texel, 48 % two, 25 % all four (62 % of active pixels are clamped in both).
enum { kCellFull = 0, kCellU = 1, kCellV = 2, kCellOne = 3 };

template <int CELL>
struct CellShape {
    static constexpr int texels = CELL == kCellFull ? 4 : CELL == kCellOne ? 1 : 2;
};

// offset of reduced texel-gradient value i (corner i / 3, channel i % 3) from the class's base texel
// texel-index offset of the class's corner k from its base texel (texel index i_u * n + i_v, core.hpp:44-48)
template <int CELL>
__device__ __forceinline__ int cell_texel(int k, int N) {
    if (CELL == kCellFull) return ((k & 1) ? N : 0) + ((k & 2) ? 1 : 0);  // 00, 10, 01, 11
    if (CELL == kCellU) return k ? N : 0;                                  // (i_u, i_v'), (i_u + 1, i_v')
    return k;                                                              // kCellV: (i_u', i_v), (i_u', i_v + 1)
}

// An entry's texels (core.hpp:44-48, texel index i_u * n + i_v): TL = 3 reads the reference layout (three
// scalar loads per texel), TL = 4 an RGBA-padded copy (one 16-B load per texel, every texel row in whole
// 16-B words; gb_context_set_texel_rgba) -- the same values either way.
template <int TL>
struct TexelRef;
template <>
struct TexelRef<3> {
    const float* t;
    __device__ __forceinline__ TexelRef(const float* tex, const float4*, int id, int NN)
        : t(tex + (size_t)id * (3 * NN)) {}
    __device__ __forceinline__ float3 operator[](int i) const {
        return make_float3(__ldg(t + 3 * i), __ldg(t + 3 * i + 1), __ldg(t + 3 * i + 2));
    }
};
template <>
struct TexelRef<4> {
    const float4* t;
    __device__ __forceinline__ TexelRef(const float*, const float4* tex4, int id, int NN) : t(tex4 + (size_t)id * NN) {}
    __device__ __forceinline__ float3 operator[](int i) const {
        const float4 q = __ldg(t + i);
        return make_float3(q.x, q.y, q.z);
    }
};
__device__ __forceinline__ float ch(const float3& q, int c) { return c == 0 ? q.x : (c == 1 ? q.y : q.z); }

// One backward entry for the calling warp, after the evaluation: rewind the pixel's state, form the
// adjoints and reduce/scatter the gradients (raster.hpp:324-363).
template <int MODE, int NT, int CELL, int S, int TL>
__device__ __forceinline__ void bwd_shade(const TexelRef<TL>& tx, int id, bool on, unsigned act, real u,
                                          real v, real G, real alpha, real araw, const PinholeTerms& pt,
                                          real& T, real g0, real g1, real g2, real& bh0, real& bh1,
                                          real& bh2, const RasterConst& rc, int N, int lane, real* wscratch,
                                          real* __restrict__ accum, real* __restrict__ grid_grad) {
    constexpr int NS = MODE == GB_MODE_ORTHO ? 7 : 10;  // screen-space sums per entry
    constexpr int NX = CellShape<CELL>::texels;
    const real sigma = rc.sigma;
    real red[16];  // screen-space sums (NS of 16 slots)
#pragma unroll
    for (int i = 0; i < 16; ++i) red[i] = (real)0;
    real tg[3 * NX];
#pragma unroll
    for (int i = 0; i < 3 * NX; ++i) tg[i] = (real)0;
    int tt = -1;  // base texel index of the entry's footprint class
    real wk[NX];  // corner weights
#pragma unroll
    for (int k = 0; k < NX; ++k) wk[k] = (real)0;
    {
        // Branch-free: every lane runs the arithmetic (the warp issues it anyway), lanes that are not on
        // skip the texel loads (predicated) and select zeros / their old state at the end -- no divergent
        // region, no BSSY/BSYNC reconvergence per entry.  Off lanes' u, v may be non-finite (a missed
        // plane): the texel addresses are clamped, and every value they reach is masked below.
        const real Tn = mul_rn(T, rcp_approx(sub_rn((real)1, alpha)));  // raster.hpp:333
        T = on ? Tn : T;
        real c0, c1, c2, fu_hat = (real)0, fv_hat = (real)0;
        const real aT = alpha * T;
        const real chat[3] = {on ? aT * g0 : (real)0, on ? aT * g1 : (real)0,
                              on ? aT * g2 : (real)0};  // c_hat (raster.hpp:338-340)
        real cc_[3];
        if (CELL == kCellFull) {
            Bilin b;
            bilin_setup(u, v, N, rc, b);
            const float3 z = make_float3(0.f, 0.f, 0.f);
            const float3 q00 = on ? tx[b.t00] : z, q10 = on ? tx[b.t00 + N] : z, q01 = on ? tx[b.t00 + 1] : z,
                         q11 = on ? tx[b.t00 + N + 1] : z;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const real c00 = ch(q00, c), c10 = ch(q10, c), c01 = ch(q01, c), c11 = ch(q11, c);
                cc_[c] = c00 * b.w00 + c10 * b.w10 + c01 * b.w01 + c11 * b.w11;
                tg[c] = chat[c] * b.w00;
                tg[3 + c] = chat[c] * b.w10;
                tg[6 + c] = chat[c] * b.w01;
                tg[9 + c] = chat[c] * b.w11;
                // texture.hpp:102-103: (C10 - C00)(1 - f_v) + (C11 - C01) f_v = du + f_v e and
                // (C01 - C00)(1 - f_u) + (C11 - C10) f_u = dv + f_u e, e = C11 - C10 - C01 + C00
                const real du = c10 - c00, dv = c01 - c00, e = (c11 - c10) - dv;
                fu_hat = fma_rn(chat[c], fma_rn(b.fv, e, du), fu_hat);
                fv_hat = fma_rn(chat[c], fma_rn(b.fu, e, dv), fv_hat);
            }
            tt = b.t00;
            wk[0] = b.w00;
            wk[1] = b.w10;
            wk[2] = b.w01;
            wk[3] = b.w11;
        } else if (CELL == kCellU || CELL == kCellV) {
            // interpolation along one axis; the other sits on texel 0 or n-1
            const real w = CELL == kCellU ? u : v;
            real sx = fma_rn(w, rc.tex_scale, rc.tex_offset);
            sx = rmin(rmax(sx, (real)0), (real)(N - 1));
            const int i0 = min((int)rfloor(sx), N - 2);
            const real f = sub_rn(sx, (real)i0);
            const real gf = (real)1 - f;
            const int other = (CELL == kCellU ? v : u) > (real)0 ? N - 1 : 0;
            tt = CELL == kCellU ? i0 * N + other : other * N + i0;
            const float3 z = make_float3(0.f, 0.f, 0.f);
            const float3 qa = on ? tx[tt] : z, qb = on ? tx[tt + (CELL == kCellU ? N : 1)] : z;
            real fh = (real)0;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const real ca = ch(qa, c), cb = ch(qb, c);
                cc_[c] = fma_rn(cb, f, ca * gf);  // = the four-corner blend with two zero weights
                tg[c] = chat[c] * gf;
                tg[3 + c] = chat[c] * f;
                fh = fma_rn(chat[c], cb - ca, fh);
            }
            if (CELL == kCellU)
                fu_hat = fh;
            else
                fv_hat = fh;
            wk[0] = gf;
            wk[1] = f;
        } else {  // kCellOne (and n = 1): a single texel with weight 1
            const int iu = N > 1 && u > (real)0 ? N - 1 : 0, iv = N > 1 && v > (real)0 ? N - 1 : 0;
            tt = iu * N + iv;
            const float3 q = on ? tx[tt] : make_float3(0.f, 0.f, 0.f);
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                cc_[c] = ch(q, c);
                tg[c] = chat[c];
            }
            wk[0] = (real)1;
        }
        GB_CHECK(!on || (tt >= 0 && tt + cell_texel<CELL>(NX - 1, N) < N * N));
        c0 = cc_[0];
        c1 = cc_[1];
        c2 = cc_[2];
        // texture.hpp:106-109 (strict mask)
        real u_hat = (CELL != kCellV && CELL != kCellOne && u > -sigma && u < sigma) ? rc.tex_scale * fu_hat : (real)0;
        real v_hat = (CELL != kCellU && CELL != kCellOne && v > -sigma && v < sigma) ? rc.tex_scale * fv_hat : (real)0;
        // raster.hpp:344-346
        const real alpha_hat = T * (g0 * (c0 - bh0) + g1 * (c1 - bh1) + g2 * (c2 - bh2));
        real op = (real)0;
        if (araw < kMaxAlpha) {  // raster.hpp:350-354
            op = alpha_hat * G;
            const real aa = alpha_hat * alpha;
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
            const real iz = pt.iz;
            const real gc0 = u_hat * iz, gc1 = v_hat * iz, gc2 = -(u_hat * u + v_hat * v) * iz;
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
#pragma unroll
        for (int i = 0; i < NS; ++i) red[i] = on ? red[i] : (real)0;
        // raster.hpp:362
        const real om = (real)1 - alpha;
        bh0 = on ? alpha * c0 + om * bh0 : bh0;
        bh1 = on ? alpha * c1 + om * bh1 : bh1;
        bh2 = on ? alpha * c2 + om * bh2 : bh2;
    }
    // S: the texel-gradient stride, 3 (reference layout (i_u, i_v, channel)) or 4 (RGBA-padded,
    // gb_context_set_texel_grad_stride: texel records 16-B aligned, one vector red each)
    real* gg = grid_grad + (size_t)id * (S * N * N);
    // this lane's non-zero texels straight to memory: one 16-B red (S = 4) or an 8-B + 4-B pair (S = 3)
    auto texel_reds = [&]() {
#pragma unroll
        for (int k = 0; k < NX; ++k)  // a zero corner weight (clamped or on-grid uv) adds nothing
            if (wk[k] != (real)0) {
                real* p = gg + S * (tt + cell_texel<CELL>(k, N));
                if (S == 4)
                    red4(p, tg[3 * k], tg[3 * k + 1], tg[3 * k + 2], (real)0);
                else
                    red3(p, tg[3 * k], tg[3 * k + 1], tg[3 * k + 2]);
            }
    };
    if (__popc(act) <= kDirectLanes) {
        // few active lanes: each adds its own terms with vector reds -- ~20 instructions for the warp
        // instead of two ~35-instruction warp reductions (12 % of warp-entries have one active lane)
        if (on) {
            real* a = accum + (size_t)id * kAccumStride;  // 48-B records: 16-B aligned
            red4(a, red[0], red[1], red[2], red[3]);
            if (NS == 10) {
                red4(a + 4, red[4], red[5], red[6], red[7]);
                red2(a + 8, red[8], red[9]);
            } else {  // slot 7 is padding in the ortho record: one 16-B red for slots 4..7
                red4(a + 4, red[4], red[5], red[6], (real)0);
            }
            texel_reds();
        }
        return;
    }
    {  // screen-space sums: lane l owns value l >> 1
        real sv[NS];
#pragma unroll
        for (int i = 0; i < NS; ++i) sv[i] = red[i];
        const real r2 = smem_reduce<NS>(sv, wscratch, lane);
        if ((lane & 1) == 0 && (lane >> 1) < NS) red_add(accum + (size_t)id * kAccumStride + (lane >> 1), r2);
    }
    if (CELL == kCellOne && NT != 1 && N > 1) {
        // one texel per lane, and it is one of the four grid corners (by the signs of u, v): one warp
        // reduction over the 4 corners x 3 channels instead of up to 32 reds on at most 4 addresses
        const int q = on ? ((u > (real)0) ? 2 : 0) + ((v > (real)0) ? 1 : 0) : -1;
        real tq[12];
#pragma unroll
        for (int i = 0; i < 12; ++i) tq[i] = (q == i / 3) ? tg[i % 3] : (real)0;
        const real r2 = smem_reduce<12>(tq, wscratch, lane);
        const int row = lane >> 1, qc = row / 3;
        if ((lane & 1) == 0 && row < 12)
            red_add(gg + S * (((qc >> 1) ? N - 1 : 0) * N + ((qc & 1) ? N - 1 : 0)) + row % 3, r2);
        return;
    }
    // texel gradients: one warp reduction when every active lane has the same base texel;
    // otherwise each lane adds its own texels -- cheaper than a reduction per distinct cell
    const int b0 = __shfl_sync(kFull, tt, __ffs(act) - 1);
    if (__all_sync(kFull, !on || tt == b0)) {
        if (lane == 0) GB_DBG(4, 1);
        const real r2 = smem_reduce<3 * NX>(tg, wscratch, lane);
        const int i = lane >> 1;
        if ((lane & 1) == 0 && i < 3 * NX) red_add(gg + S * (b0 + cell_texel<CELL>(i / 3, N)) + i % 3, r2);
    } else if (on) {
        if (lane == 0) GB_DBG(5, 1);
        texel_reds();
    }
}

// One backward entry for the calling warp: evaluate, pick the warp's texel footprint class, then
// bwd_shade (raster.hpp:324-363).
template <int MODE, int NT, int S, int TL = 3>
__device__ __forceinline__ void bwd_entry(const ScreenHeader& h, const float* __restrict__ tex, int id, int rank,
                                          int last, int x, int y, real& T, real g0, real g1, real g2,
                                          real& bh0, real& bh1, real& bh2, const RasterConst& rc, int N,
                                          int lane, real* wscratch, real* __restrict__ accum,
                                          real* __restrict__ grid_grad) {
    const real sigma = rc.sigma;
    // evaluated on every lane (branch-free; lanes past their last rank or missing the plane are masked)
    real u, v;
    PinholeTerms pt;
    bool hit;
    if (MODE == GB_MODE_ORTHO) {
        hit = eval_uv_ortho(h, x, y, u, v);
    } else {
        hit = eval_uv_pinhole(h, x, y, u, v, pt);
    }
    const real G = gauss_weight(u, v);
    const real araw = mul_rn(h.h1.z, G);
    const real alpha = rmin(araw, kMaxAlpha);
    const bool on = rank <= last && hit && !(alpha < rc.alpha_skip);
    const unsigned act = __ballot_sync(kFull, on);
    if (act == 0) return;
    if (lane == 0) {
        GB_DBG(2, 1);
        GB_DBG(3, __popc(act));
        GB_DBG(6, (act & 0x0F0F0F0Fu) && (act & 0xF0F0F0F0u));  // both 4x4 halves active
        GB_DBG(7, (act & 0x0000FFFFu) && (act & 0xFFFF0000u));  // both 8x2 halves active
    }
    const TexelRef<TL> tx(tex, rc.tex4, id, N * N);
#define GB_SHADE(CELL)                                                                                              \
    bwd_shade<MODE, NT, CELL, S, TL>(tx, id, on, act, u, v, G, alpha, araw, pt, T, g0, g1, g2, bh0, bh1, bh2, rc, N, \
                                     lane, wscratch, accum, grid_grad)
    if (N == 1) {
        GB_SHADE(kCellOne);
        return;
    }
    const bool au = __any_sync(kFull, on && u > -sigma && u < sigma);
    const bool av = __any_sync(kFull, on && v > -sigma && v < sigma);
    if (au && av)
        GB_SHADE(kCellFull);
    else if (au)
        GB_SHADE(kCellU);
    else if (av)
        GB_SHADE(kCellV);
    else
        GB_SHADE(kCellOne);
#undef GB_SHADE
}

// ---------------------------------------------------------------------------
// Direct variants (no shared-memory staging): each warp walks the tile list on
// its own, reading ids, headers and texels through L1 (__ldg).  No producer,
// no CTA-level synchronisation; warps finish independently.  The walks are
// device functions shared by the forward, the backward and the fused
// forward + loss + backward kernel, so all three run the same arithmetic.
// ---------------------------------------------------------------------------
struct WarpPixel {
    int x, y;
    bool inside;
    float bx0, bx1, by0, by1;  // the warp's pixel rectangle
};

__device__ __forceinline__ WarpPixel warp_pixel(const RasterConst& rc, const CamConst& cc, int tile) {
    WarpPixel w;
    const int ts = rc.tile_size;
    const int tx = tile % rc.tiles_x, ty = tile / rc.tiles_x;
    int lx, ly;
    tile_pixel(threadIdx.x, ts, lx, ly);
    w.x = tx * ts + lx;
    w.y = ty * ts + ly;
    w.inside = (int)threadIdx.x < ts * ts && w.x < cc.width && w.y < cc.height;
    w.bx0 = (float)__reduce_min_sync(kFull, w.x);
    w.bx1 = (float)__reduce_max_sync(kFull, w.x);
    w.by0 = (float)__reduce_min_sync(kFull, w.y);
    w.by1 = (float)__reduce_max_sync(kFull, w.y);
    return w;
}

// one lane's test of list entry `idl` against its warp's rectangle: the exact alpha-skip ellipse (K1);
// the variant build -DGB_CULL_BOX tests the alpha-box instead (A/B only)
__device__ __forceinline__ bool entry_meets_warp(const ScreenHeader* __restrict__ hdr, const CullRec* __restrict__ cull,
                                                 int idl, const WarpPixel& w) {
#ifdef GB_CULL_BOX
    return !box_miss(__ldg(&hdr[idl].h3), w.bx0, w.bx1, w.by0, w.by1);
#else
    return ellipse_meets_rect(__ldg(&cull[idl].a), __ldg(&cull[idl].b), w.bx0 - 0.05f, w.bx1 + 0.05f, w.by0 - 0.05f,
                              w.by1 + 0.05f);
#endif
}

// The warp rectangle of the lanes still in play (the forward's pixels not yet past early termination):
// entries that meet only the other pixels change nothing.
__device__ __forceinline__ WarpPixel live_rect(const WarpPixel& wp, bool live) {
    WarpPixel r = wp;
    r.bx0 = (float)__reduce_min_sync(kFull, live ? wp.x : INT_MAX);
    r.bx1 = (float)__reduce_max_sync(kFull, live ? wp.x : INT_MIN);
    r.by0 = (float)__reduce_min_sync(kFull, live ? wp.y : INT_MAX);
    r.by1 = (float)__reduce_max_sync(kFull, live ? wp.y : INT_MIN);
    return r;
}

// One forward entry for the calling warp (raster.hpp:238-250): evaluate, pick the warp's texel footprint
// class (see bwd_shade), composite into the lanes that are not done.
template <int MODE, int NT, int TL = 3, bool DERIVED_DONE = false>
__device__ __forceinline__ void fwd_entry(const ScreenHeader& h, const float* __restrict__ tex, int id, int rank, int x,
                                          int y, const RasterConst& rc, int N, real early, bool& done, real& T,
                                          real& acc0, real& acc1, real& acc2, int& last) {
    real u, v;
    bool hit;
    if (MODE == GB_MODE_ORTHO) {
        hit = eval_uv_ortho(h, x, y, u, v);
    } else {
        PinholeTerms pt;
        hit = eval_uv_pinhole(h, x, y, u, v, pt);
    }
    const real G = gauss_weight(u, v);
    const real alpha = rmin(mul_rn(h.h1.z, G), kMaxAlpha);  // raster.hpp:241
    // DERIVED_DONE: a pixel is done once it composited (last >= 0) and T fell below the threshold -- the same
    // state as the flag (T and last change only when compositing), without a flag to keep
    const bool fin = DERIVED_DONE ? (last >= 0 && T < early) : done;
    const bool comp = !fin && hit && !(alpha < rc.alpha_skip);     // raster.hpp:242
    // texel footprint class of the warp (see bwd_shade): clamped axes read one texel row
    const real sigma = rc.sigma;
    const bool au = N > 1 && __any_sync(kFull, comp && u > -sigma && u < sigma);
    const bool av = N > 1 && __any_sync(kFull, comp && v > -sigma && v < sigma);
    if (comp) {
        const TexelRef<TL> tx(tex, rc.tex4, id, N * N);
        real c0_, c1_, c2_;
        if (au && av) {
            Bilin b;
            bilin_setup(u, v, N, rc, b);
            const float3 q00 = tx[b.t00], q10 = tx[b.t00 + N], q01 = tx[b.t00 + 1], q11 = tx[b.t00 + N + 1];
            c0_ = q00.x * b.w00 + q10.x * b.w10 + q01.x * b.w01 + q11.x * b.w11;
            c1_ = q00.y * b.w00 + q10.y * b.w10 + q01.y * b.w01 + q11.y * b.w11;
            c2_ = q00.z * b.w00 + q10.z * b.w10 + q01.z * b.w01 + q11.z * b.w11;
        } else if (au || av) {  // the four-corner blend with two zero weights
            // (separate uniform branches: each keeps its index arithmetic free of selects)
            int ta, tb;
            real f;
            if (au) {
                real sx = fma_rn(u, rc.tex_scale, rc.tex_offset);
                sx = rmin(rmax(sx, (real)0), (real)(N - 1));
                const int i0 = min((int)rfloor(sx), N - 2);
                f = sub_rn(sx, (real)i0);
                ta = i0 * N + (v > (real)0 ? N - 1 : 0);
                tb = ta + N;
            } else {
                real sx = fma_rn(v, rc.tex_scale, rc.tex_offset);
                sx = rmin(rmax(sx, (real)0), (real)(N - 1));
                const int i0 = min((int)rfloor(sx), N - 2);
                f = sub_rn(sx, (real)i0);
                ta = (u > (real)0 ? N - 1 : 0) * N + i0;
                tb = ta + 1;
            }
            const real gf = (real)1 - f;
            const float3 qa = tx[ta], qb = tx[tb];
            c0_ = fma_rn(qb.x, f, qa.x * gf);
            c1_ = fma_rn(qb.y, f, qa.y * gf);
            c2_ = fma_rn(qb.z, f, qa.z * gf);
        } else {  // one texel (and n = 1)
            const float3 q = tx[N > 1 ? (u > (real)0 ? N - 1 : 0) * N + (v > (real)0 ? N - 1 : 0) : 0];
            c0_ = q.x;
            c1_ = q.y;
            c2_ = q.z;
        }
        const real w = alpha * T;  // raster.hpp:244-249
        acc0 = fma_rn(c0_, w, acc0);
        acc1 = fma_rn(c1_, w, acc1);
        acc2 = fma_rn(c2_, w, acc2);
        T = mul_rn(T, sub_rn((real)1, alpha));
        last = rank;
        if (!DERIVED_DONE && T < early) done = true;  // raster.hpp:250
    }
}

// Per-warp header staging (default; -DGB_WARP_STAGE=0 for the A/B): after the 32-entry ballot every
// passing lane copies its entry's header into the warp's shared-memory slot (structure of arrays, so the
// stores are conflict-free and each entry's read is a broadcast).  The warp then waits on the header
// loads once per chunk -- all issued together -- instead of once per entry right before its evaluation
// (the evaluation's first header use was the top stall site of K3 and K4 under ncu).  Warp-private: no CTA
// barrier, only __syncwarp.
#ifndef GB_WARP_STAGE
#define GB_WARP_STAGE 1
#endif
struct WarpHeaders {
    real4 h[3][32];
    int id[32];   // the chunk's primitive ids (read per entry instead of a shuffle of a register held through the loop)
    float4 rect;  // K4: the warp's pixel rectangle for the cull test, +-0.05 px (re-read per chunk, see bwd_walk)
};

// the warp rectangle kept in shared memory: re-read once per 32-entry chunk instead of holding four registers
// through the entry loop (at K4's 48-register cap they spilled: three local loads per warp-entry)
__device__ __forceinline__ float4 ld_rect(const float4* r) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"((uint32_t)__cvta_generic_to_shared(r)));
    return v;
}

// (slot: the lane for K3, 31 - lane for K4's back-to-front walk)
__device__ __forceinline__ void stage_headers(WarpHeaders& wh, const ScreenHeader* __restrict__ hdr, bool pass,
                                              int idl, int slot) {
    __syncwarp();  // the previous chunk's readers are done
    if (pass) {
        wh.h[0][slot] = ld_real4(&hdr[idl].h0);
        wh.h[1][slot] = ld_real4(&hdr[idl].h1);
        wh.h[2][slot] = ld_real4(&hdr[idl].h2);
        wh.id[slot] = idl;
    }
    __syncwarp();
}

__device__ __forceinline__ ScreenHeader staged_hdr(const WarpHeaders& wh, int j) {
    ScreenHeader h;
    h.h0 = wh.h[0][j];
    h.h1 = wh.h[1][j];
    h.h2 = wh.h[2][j];
    return h;
}

// render_forward's per-pixel loop (raster.hpp:237-250) for the calling warp's pixels
template <int MODE, int NT, int TL>
__device__ __forceinline__ void fwd_walk(const uint2 range, const int32_t* __restrict__ values,
                                         const ScreenHeader* __restrict__ hdr, const CullRec* __restrict__ cull,
                                         const float* __restrict__ tex, const RasterConst& rc, int N,
                                         const WarpPixel& wp, real& T, real& acc0, real& acc1, real& acc2,
                                         int& last, WarpHeaders* wh) {
    const int lane = threadIdx.x & 31;
    const int total = (int)(range.y - range.x);
    const int x = wp.x, y = wp.y;
    T = (real)1;
    acc0 = acc1 = acc2 = (real)0;
    last = -1;
    const real early = rc.early_stop;  // -1 when disabled (gb_capi.cu): T >= 0 never falls below it
    // No per-pixel done flag (a byte-packed bool cost three instructions per entry at the 32-register cap): a
    // pixel is done once it composited and T fell below the threshold (fwd_entry<..., true>).  Pixels outside
    // the image start finished -- last 0, T -2 below any threshold >= -1 -- and are never stored.  +0.5 %
    // (ab_r02 s60).
    if (!wp.inside) {
        T = (real)-2;
        last = 0;
    }
    bool done = false;  // unused by the derived test
#define GB_K3_DONE (last >= 0 && T < early)
    for (int c0 = 0; c0 < total && !__all_sync(kFull, GB_K3_DONE); c0 += 32) {
        const WarpPixel lr = live_rect(wp, !(GB_K3_DONE));
        int idl = -1;
        bool pass = false;
        if (c0 + lane < total) {
            idl = __ldg(&values[range.x + c0 + lane]);
            GB_CHECK(idl >= 0 && idl < rc.dbg_K);
            pass = entry_meets_warp(hdr, cull, idl, lr);
        }
        unsigned mask = __ballot_sync(kFull, pass);
#if GB_WARP_STAGE
        if (mask) stage_headers(*wh, hdr, pass, idl, lane);
#endif
        while (mask) {
            const int bit = __ffs(mask) - 1;
            mask &= mask - 1;
#if GB_WARP_STAGE
            const int id = wh->id[bit];
            const ScreenHeader h = staged_hdr(*wh, bit);
#else
            const int id = __shfl_sync(kFull, idl, bit);
            ScreenHeader h;
            h.h0 = ld_real4(&hdr[id].h0);
            h.h1 = ld_real4(&hdr[id].h1);
            h.h2 = ld_real4(&hdr[id].h2);
#endif
            // every lane evaluates (the warp runs the instructions anyway); finished pixels just do not composite
            // (no per-entry all-done vote: early termination is checked once per chunk by the outer loop --
            // the rest of a chunk after every pixel finished composites nothing; +0.65 %, ab_r02 s53)
            fwd_entry<MODE, NT, TL, true>(h, tex, id, c0 + bit, x, y, rc, N, early, done, T, acc0, acc1, acc2, last);
        }
    }
#undef GB_K3_DONE
}

// render_backward's per-pixel loop (raster.hpp:313-364) for the calling warp's pixels
template <int MODE, int NT, int S, int TL>
__device__ __forceinline__ void bwd_walk(const uint2 range, const int32_t* __restrict__ values,
                                         const ScreenHeader* __restrict__ hdr, const CullRec* __restrict__ cull,
                                         const float* __restrict__ tex, const CamConst& cc, const RasterConst& rc,
                                         int N, const WarpPixel& wp, int last, real T, real g0, real g1, real g2,
                                         real* wscratch, real* __restrict__ accum, real* __restrict__ grid_grad,
                                         WarpHeaders* wh) {
    const int F = 3 * N * N;
    const int lane = threadIdx.x & 31;
    if (g0 == (real)0 && g1 == (real)0 && g2 == (real)0) last = -1;  // raster.hpp:315-317
    real bh0 = cc.bg[0], bh1 = cc.bg[1], bh2 = cc.bg[2];
    const int wlast = __reduce_max_sync(kFull, last);
    const int xy = wp.x | (wp.y << 16);  // pixel coordinates < 2^16 (gb_build_binning checks the image size)
#if GB_WARP_STAGE && !defined(GB_CULL_BOX)
    if (lane == 0) wh->rect = make_float4(wp.bx0 - 0.05f, wp.bx1 + 0.05f, wp.by0 - 0.05f, wp.by1 + 0.05f);
    __syncwarp();
#endif
    for (int c0 = wlast & ~31; c0 >= 0; c0 -= 32) {
        // (a live rectangle here -- lanes with last >= c0 -- measured 1 % slower: few entries drop out)
        int idl = -1;
        bool pass = false;
        if (c0 + lane <= wlast) {
            idl = __ldg(&values[range.x + c0 + lane]);
            GB_CHECK(idl >= 0 && idl < rc.dbg_K);
#if GB_WARP_STAGE && !defined(GB_CULL_BOX)
            const float4 r = ld_rect(&wh->rect);
            pass = ellipse_meets_rect(__ldg(&cull[idl].a), __ldg(&cull[idl].b), r.x, r.y, r.z, r.w);
#else
            pass = entry_meets_warp(hdr, cull, idl, wp);
#endif
        }
        unsigned mask = __ballot_sync(kFull, pass);
        if (lane == 0) GB_DBG(1, __popc(mask));
#if GB_WARP_STAGE
        // entries staged in reverse slot order (slot 31 - lane), so the back-to-front walk takes the lowest set
        // bit of the reversed ballot: a shorter per-entry index computation (+0.3 %, ab_r02 s61)
        if (mask) stage_headers(*wh, hdr, pass, idl, 31 - lane);
        unsigned rmask = __brev(mask);
        while (rmask) {
            const int slot = __ffs(rmask) - 1;
            rmask &= rmask - 1;
            const int bit = 31 - slot;
            const int id = wh->id[slot];
            const ScreenHeader h = staged_hdr(*wh, slot);
#else
        while (mask) {
            const int bit = 31 - __clz(mask);
            mask &= ~(1u << bit);
            const int id = __shfl_sync(kFull, idl, bit);
            ScreenHeader h;
            h.h0 = ld_real4(&hdr[id].h0);
            h.h1 = ld_real4(&hdr[id].h1);
            h.h2 = ld_real4(&hdr[id].h2);
#endif
            // the pixel's x and y live packed in one register through the loop and are unpacked per entry
            // (volatile: not hoisted out of the loop) -- at the 48-register cap this removed the last
            // per-entry spill reload (+1.6 %, ab_r02 s54)
            int px, py;
            asm volatile("bfe.u32 %0, %2, 0, 16;\n\tshr.u32 %1, %2, 16;" : "=r"(px), "=r"(py) : "r"(xy));
            bwd_entry<MODE, NT, S, TL>(h, tex, id, c0 + bit, last, px, py, T, g0, g1, g2, bh0, bh1, bh2, rc, N,
                                       lane, wscratch, accum, grid_grad);
        }
    }
}

#ifdef GB_STAGE_HEADERS
#ifdef GB_PARITY_F64
#error "GB_STAGE_HEADERS is an fp32 A/B variant"
#endif
// ---------------------------------------------------------------------------
// Variant build (-DGB_STAGE_HEADERS; A/B only): CTA-cooperative staging of the list
// entries' ids, cull records and headers (84 B per entry) in a double-buffered shared-memory ring of
// 32-entry chunks.  Warp 0 copies chunk i+1 with cp.async (16-B LDGSTS, one entry per lane) while every
// warp composites chunk i from shared memory; one CTA barrier per chunk.  Texels stay on L1.  Versus the
// direct walk each entry's id/cull/header is read from L2/L1 once per tile instead of once per warp.
// ---------------------------------------------------------------------------
struct __align__(16) StageChunk {
    float4 cull[32][2];
    float4 hdr[32][3];
    int id[32];
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// warp 0: entries [c0, c0 + n) of the tile list into chunk buffer b (n <= 32)
__device__ __forceinline__ void stage_chunk(StageChunk& b, const int32_t* __restrict__ values, uint32_t base, int c0,
                                            int n, const ScreenHeader* __restrict__ hdr,
                                            const CullRec* __restrict__ cull) {
    const int lane = threadIdx.x & 31;
    const int id = lane < n ? __ldg(&values[base + c0 + lane]) : -1;
    b.id[lane] = id;
    if (id >= 0) {
        cp_async16(&b.cull[lane][0], &cull[id].a);
        cp_async16(&b.cull[lane][1], &cull[id].b);
        cp_async16(&b.hdr[lane][0], &hdr[id].h0);
        cp_async16(&b.hdr[lane][1], &hdr[id].h1);
        cp_async16(&b.hdr[lane][2], &hdr[id].h2);
    }
    cp_async_commit();
}

__device__ __forceinline__ bool staged_meets(const StageChunk& b, int j, const WarpPixel& w) {
    return ellipse_meets_rect(b.cull[j][0], b.cull[j][1], w.bx0 - 0.05f, w.bx1 + 0.05f, w.by0 - 0.05f, w.by1 + 0.05f);
}

__device__ __forceinline__ ScreenHeader staged_header(const StageChunk& b, int j) {
    ScreenHeader h;
    h.h0 = b.hdr[j][0];
    h.h1 = b.hdr[j][1];
    h.h2 = b.hdr[j][2];
    return h;
}

template <int MODE, int NT>
__device__ __forceinline__ void fwd_walk_staged(const uint2 range, const int32_t* __restrict__ values,
                                                const ScreenHeader* __restrict__ hdr, const CullRec* __restrict__ cull,
                                                const float* __restrict__ tex, const RasterConst& rc, int N,
                                                const WarpPixel& wp, real& T, real& acc0, real& acc1, real& acc2,
                                                int& last, StageChunk* ring) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int total = (int)(range.y - range.x);
    T = (real)1;
    acc0 = acc1 = acc2 = (real)0;
    last = -1;
    bool done = !wp.inside;
    const real early = rc.early_stop;
    if (total == 0) return;
    if (warp == 0) {
        stage_chunk(ring[0], values, range.x, 0, min(32, total), hdr, cull);
        cp_async_wait_all();
    }
    __syncthreads();
    int buf = 0;
    for (int c0 = 0; c0 < total; c0 += 32) {
        if (warp == 0 && c0 + 32 < total) stage_chunk(ring[buf ^ 1], values, range.x, c0 + 32, min(32, total - c0 - 32), hdr, cull);
        const StageChunk& b = ring[buf];
        if (!__all_sync(kFull, done)) {
            const WarpPixel lr = live_rect(wp, !done);
            const bool pass = c0 + lane < total && staged_meets(b, lane, lr);
            unsigned mask = __ballot_sync(kFull, pass);
            while (mask) {
                const int bit = __ffs(mask) - 1;
                mask &= mask - 1;
                fwd_entry<MODE, NT>(staged_header(b, bit), tex, b.id[bit], c0 + bit, wp.x, wp.y, rc, N, early, done, T,
                                    acc0, acc1, acc2, last);
                if (__all_sync(kFull, done)) break;
            }
        }
        if (warp == 0) cp_async_wait_all();
        if (__syncthreads_and(done)) break;  // every pixel of the tile terminated (raster.hpp:250)
        buf ^= 1;
    }
}

template <int MODE, int NT, int S>
__device__ __forceinline__ void bwd_walk_staged(const uint2 range, const int32_t* __restrict__ values,
                                                const ScreenHeader* __restrict__ hdr, const CullRec* __restrict__ cull,
                                                const float* __restrict__ tex, const CamConst& cc,
                                                const RasterConst& rc, int N, const WarpPixel& wp, int last, real T,
                                                real g0, real g1, real g2, real* wscratch, real* __restrict__ accum,
                                                real* __restrict__ grid_grad, StageChunk* ring, int* s_top) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (g0 == (real)0 && g1 == (real)0 && g2 == (real)0) last = -1;  // raster.hpp:315-317
    real bh0 = cc.bg[0], bh1 = cc.bg[1], bh2 = cc.bg[2];
    const int wlast = __reduce_max_sync(kFull, last);
    if (threadIdx.x == 0) *s_top = -1;
    __syncthreads();
    if (lane == 0 && wlast >= 0) atomicMax(s_top, wlast);
    __syncthreads();
    const int top = *s_top;  // the CTA walks ranks [0, top] back to front in 32-entry chunks
    if (top < 0) return;
    int c0 = top & ~31;
    if (warp == 0) {
        stage_chunk(ring[0], values, range.x, c0, top - c0 + 1, hdr, cull);
        cp_async_wait_all();
    }
    __syncthreads();
    int buf = 0;
    for (; c0 >= 0; c0 -= 32) {
        if (warp == 0 && c0 >= 32) stage_chunk(ring[buf ^ 1], values, range.x, c0 - 32, 32, hdr, cull);
        const StageChunk& b = ring[buf];
        if (c0 <= wlast) {
            const bool pass = c0 + lane <= wlast && staged_meets(b, lane, wp);
            unsigned mask = __ballot_sync(kFull, pass);
            while (mask) {
                const int bit = 31 - __clz(mask);
                mask &= ~(1u << bit);
                const int id = b.id[bit];
                bwd_entry<MODE, NT, S>(staged_header(b, bit), tex, id, c0 + bit, last, wp.x,
                                    wp.y, T, g0, g1, g2, bh0, bh1, bh2, rc, N, lane, wscratch, accum, grid_grad);
            }
        }
        if (warp == 0) cp_async_wait_all();
        __syncthreads();
        buf ^= 1;
    }
}
#endif  // GB_STAGE_HEADERS

// K3 at <= 32 registers: 8 CTAs (64 warps) per SM, no spills, the same instructions as the compiler's own
// 40-register choice (6 CTAs) -- measured 0.7 % faster
#ifndef GB_K3_MINB
#define GB_K3_MINB 8
#endif
template <int MODE, int NT, int TL>
__global__ void __launch_bounds__(256, GB_K3_MINB) k_forward_direct(const uint2* __restrict__ ranges,
                                                        const int32_t* __restrict__ values,
                                                        const ScreenHeader* __restrict__ hdr,
                                                        const CullRec* __restrict__ cull, const float* __restrict__ tex,
                                                        const CamConst cc, const RasterConst rc, int n_rt,
                                                        float* __restrict__ out_color, float* __restrict__ out_trans,
                                                        int32_t* __restrict__ out_last) {
    const WarpPixel wp = warp_pixel(rc, cc, blockIdx.x);
    real T, a0, a1, a2;
    int last;
#ifdef GB_STAGE_HEADERS
    __shared__ StageChunk ring[2];
    fwd_walk_staged<MODE, NT>(ranges[blockIdx.x], values, hdr, cull, tex, rc, tex_n<NT>(n_rt), wp, T, a0, a1, a2, last,
                              ring);
#else
    __shared__ WarpHeaders whs[8];
    fwd_walk<MODE, NT, TL>(ranges[blockIdx.x], values, hdr, cull, tex, rc, tex_n<NT>(n_rt), wp, T, a0, a1, a2, last,
                       &whs[threadIdx.x >> 5]);
#endif
    if (wp.inside) {  // raster.hpp:253-254
        const size_t p = (size_t)wp.y * cc.width + wp.x;
        out_color[p * 3 + 0] = fma_rn(T, cc.bg[0], a0);
        out_color[p * 3 + 1] = fma_rn(T, cc.bg[1], a1);
        out_color[p * 3 + 2] = fma_rn(T, cc.bg[2], a2);
        out_trans[p] = T;
#ifdef GB_PARITY_F64
        if (rc.trans64) rc.trans64[p] = T;
#endif
        out_last[p] = last;
    }
}

// render_forward with the photometric loss (KIND 0 = L1, 1 = MSE; K6) in its epilogue: the pixel's
// colour turns into the loss cotangent in registers, so the image is written only when asked for and
// no separate loss pass runs.  T and the last rank are always written (the backward rewinds from them).
template <int MODE, int NT, int KIND, int TL>
__global__ void __launch_bounds__(256, GB_K3_MINB) k_forward_loss(const uint2* __restrict__ ranges,
                                                      const int32_t* __restrict__ values,
                                                      const ScreenHeader* __restrict__ hdr,
                                                      const CullRec* __restrict__ cull, const float* __restrict__ tex,
                                                      const CamConst cc, const RasterConst rc, int n_rt,
                                                      const float* __restrict__ target, float scale,
                                                      float* __restrict__ out_color, float* __restrict__ out_trans,
                                                      int32_t* __restrict__ out_last, float* __restrict__ out_grad,
                                                      float* __restrict__ loss) {
    const WarpPixel wp = warp_pixel(rc, cc, blockIdx.x);
    real T, a0, a1, a2;
    int last;
#ifdef GB_STAGE_HEADERS
    __shared__ StageChunk ring[2];
    fwd_walk_staged<MODE, NT>(ranges[blockIdx.x], values, hdr, cull, tex, rc, tex_n<NT>(n_rt), wp, T, a0, a1, a2, last,
                              ring);
#else
    __shared__ WarpHeaders whs[8];
    fwd_walk<MODE, NT, TL>(ranges[blockIdx.x], values, hdr, cull, tex, rc, tex_n<NT>(n_rt), wp, T, a0, a1, a2, last,
                       &whs[threadIdx.x >> 5]);
#endif
    real l = (real)0;
    if (wp.inside) {
        const size_t p = (size_t)wp.y * cc.width + wp.x;
        const real c[3] = {fma_rn(T, cc.bg[0], a0), fma_rn(T, cc.bg[1], a1), fma_rn(T, cc.bg[2], a2)};
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {  // K6 (gb_misc.cu k_loss), per pixel
            const real d = c[ch] - target[p * 3 + ch];
            real g;
            if (KIND == 0) {
                l += rabs(d);
                g = scale * (real)((d > (real)0) - (d < (real)0));
            } else {
                l = fma_rn(d, d, l);
                g = (real)2 * scale * d;
            }
            out_grad[p * 3 + ch] = g;
            if (out_color) out_color[p * 3 + ch] = c[ch];
        }
        out_trans[p] = T;
#ifdef GB_PARITY_F64
        if (rc.trans64) rc.trans64[p] = T;
#endif
        out_last[p] = last;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(kFull, l, o);
    if ((threadIdx.x & 31) == 0 && loss && l != (real)0) atomicAdd(loss, (float)(l * scale));
}

// K4 register caps.  Reference texel layout (TL = 3): <= 64 registers, 4 CTAs (32 warps) per SM, no spills --
// with the branch-free entry, 1.0 % faster than 5 CTAs at 48 registers (16 B of spills) and 7 % faster than 6
// CTAs at 40 (56 B).  RGBA texels (TL = 4, one 16-B load per texel, fewer live registers): <= 48 registers,
// 5 CTAs per SM (16 B of spills) -- 2.7 % faster than 4 CTAs, 7 % faster than 6 (profiles/ab_r02.md s44).
#ifndef GB_K4_MINB
#define GB_K4_MINB 4
#endif
#ifndef GB_K4_MINB_RGBA
#define GB_K4_MINB_RGBA 5
#endif
template <int MODE, int NT, int S, int TL>
__global__ void __launch_bounds__(256, TL == 4 ? GB_K4_MINB_RGBA : GB_K4_MINB) k_backward_direct(const uint2* __restrict__ ranges,
                                                         const int32_t* __restrict__ values,
                                                         const ScreenHeader* __restrict__ hdr,
                                                         const CullRec* __restrict__ cull, const float* __restrict__ tex,
                                                         const CamConst cc, const RasterConst rc, int n_rt,
                                                         const float* __restrict__ in_trans,
                                                         const int32_t* __restrict__ in_last,
                                                         const float* __restrict__ image_grad,
                                                         real* __restrict__ accum, real* __restrict__ grid_grad) {
    extern __shared__ __align__(16) real red_scratch[];
    const WarpPixel wp = warp_pixel(rc, cc, blockIdx.x);
    int last = -1;
    real T = (real)1, g0 = (real)0, g1 = (real)0, g2 = (real)0;
    if (wp.inside) {  // raster.hpp:313-322
        const size_t p = (size_t)wp.y * cc.width + wp.x;
        last = in_last[p];
        g0 = image_grad[p * 3 + 0];
        g1 = image_grad[p * 3 + 1];
        g2 = image_grad[p * 3 + 2];
        T = in_trans[p];
#ifdef GB_PARITY_F64
        if (rc.trans64) T = rc.trans64[p];
#endif
    }
#ifdef GB_STAGE_HEADERS
    __shared__ StageChunk ring[2];
    __shared__ int s_top;
    bwd_walk_staged<MODE, NT, S>(ranges[blockIdx.x], values, hdr, cull, tex, cc, rc, tex_n<NT>(n_rt), wp, last, T, g0, g1,
                              g2, red_scratch + (threadIdx.x >> 5) * kRedRows * kRedStride, accum, grid_grad, ring,
                              &s_top);
#else
    __shared__ WarpHeaders whs[8];
    bwd_walk<MODE, NT, S, TL>(ranges[blockIdx.x], values, hdr, cull, tex, cc, rc, tex_n<NT>(n_rt), wp, last, T, g0, g1,
                          g2, red_scratch + (threadIdx.x >> 5) * kRedRows * kRedStride, accum, grid_grad,
                          &whs[threadIdx.x >> 5]);
#endif
}

#ifdef GB_FUSED_SINGLE_KERNEL
// Variant build only (measured slower).
// render_forward + the photometric loss (KIND 0 = L1, 1 = MSE; K6) + render_backward of one view in one
// kernel.  Every warp composites its pixels, turns them into the loss cotangent in registers and walks the
// same entries back to front while their headers and texels are still in L1/L2; colour, transmittance,
// last rank and the cotangent are stored only when asked for.
template <int MODE, int NT, int KIND>
__global__ void __launch_bounds__(256) k_fused_direct(const uint2* __restrict__ ranges,
                                                      const int32_t* __restrict__ values,
                                                      const ScreenHeader* __restrict__ hdr,
                                                      const CullRec* __restrict__ cull, const float* __restrict__ tex,
                                                      const CamConst cc, const RasterConst rc, int n_rt,
                                                      const float* __restrict__ target, float scale,
                                                      float* __restrict__ out_color, float* __restrict__ out_trans,
                                                      int32_t* __restrict__ out_last, float* __restrict__ out_grad,
                                                      float* __restrict__ loss, real* __restrict__ accum,
                                                      real* __restrict__ grid_grad) {
    extern __shared__ __align__(16) real red_scratch[];
    const int N = tex_n<NT>(n_rt);
    const WarpPixel wp = warp_pixel(rc, cc, blockIdx.x);
    const uint2 range = ranges[blockIdx.x];
    real T, a0, a1, a2;
    int last;
    __shared__ WarpHeaders whs[8];
    fwd_walk<MODE, NT, 3>(range, values, hdr, cull, tex, rc, N, wp, T, a0, a1, a2, last, &whs[threadIdx.x >> 5]);
    real g0 = (real)0, g1 = (real)0, g2 = (real)0, l = (real)0;
    if (wp.inside) {
        const size_t p = (size_t)wp.y * cc.width + wp.x;
        const real c[3] = {fma_rn(T, cc.bg[0], a0), fma_rn(T, cc.bg[1], a1), fma_rn(T, cc.bg[2], a2)};
        real g[3];
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {  // K6 (gb_misc.cu k_loss), per pixel
            const real d = c[ch] - target[p * 3 + ch];
            if (KIND == 0) {
                l += rabs(d);
                g[ch] = scale * (real)((d > (real)0) - (d < (real)0));
            } else {
                l = fma_rn(d, d, l);
                g[ch] = (real)2 * scale * d;
            }
        }
        g0 = g[0];
        g1 = g[1];
        g2 = g[2];
        if (out_color) {
            out_color[p * 3 + 0] = c[0];
            out_color[p * 3 + 1] = c[1];
            out_color[p * 3 + 2] = c[2];
            out_trans[p] = T;
#ifdef GB_PARITY_F64
        if (rc.trans64) rc.trans64[p] = T;
#endif
            out_last[p] = last;
        }
        if (out_grad) {
            out_grad[p * 3 + 0] = g0;
            out_grad[p * 3 + 1] = g1;
            out_grad[p * 3 + 2] = g2;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(kFull, l, o);
    if ((threadIdx.x & 31) == 0 && loss && l != (real)0) atomicAdd(loss, (float)(l * scale));
    bwd_walk<MODE, NT, 3, 3>(range, values, hdr, cull, tex, cc, rc, N, wp, last, T, g0, g1, g2,
                       red_scratch + (threadIdx.x >> 5) * kRedRows * kRedStride, accum, grid_grad,
                       &whs[threadIdx.x >> 5]);
}
#endif  // GB_FUSED_SINGLE_KERNEL

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
#define GB_DISPATCH_N(FN, MODE, ...)               \
    switch (n) {                                   \
        case 1: return FN<MODE, 1>(__VA_ARGS__);   \
        case 2: return FN<MODE, 2>(__VA_ARGS__);   \
        case 4: return FN<MODE, 4>(__VA_ARGS__);   \
        case 8: return FN<MODE, 8>(__VA_ARGS__);   \
        case 16: return FN<MODE, 16>(__VA_ARGS__); \
        default: return FN<MODE, 0>(__VA_ARGS__);  \
    }

static int tile_threads(int ts) { return ((ts * ts + 31) / 32) * 32; }
static size_t red_smem(int threads) { return (size_t)(threads / 32) * kRedRows * kRedStride * sizeof(real); }

template <int MODE, int NT>
static cudaError_t fwdd_t(int tiles, int threads, cudaStream_t st, const uint2* ranges, const int32_t* values,
                          const ScreenHeader* hdr, const CullRec* cull, const float* tex, const CamConst& cc,
                          const RasterConst& rc, int n, float* color, float* trans, int32_t* last) {
    if (rc.tex4)  // RGBA-padded texels (gb_context_set_texel_rgba)
        k_forward_direct<MODE, NT, 4><<<tiles, threads, 0, st>>>(ranges, values, hdr, cull, tex, cc, rc, n, color, trans,
                                                                 last);
    else
        k_forward_direct<MODE, NT, 3><<<tiles, threads, 0, st>>>(ranges, values, hdr, cull, tex, cc, rc, n, color, trans,
                                                                 last);
    return cudaGetLastError();
}

template <int MODE, int NT>
static cudaError_t bwdd_t(int tiles, int threads, cudaStream_t st, const uint2* ranges, const int32_t* values,
                          const ScreenHeader* hdr, const CullRec* cull, const float* tex, const CamConst& cc,
                          const RasterConst& rc, int n, const float* trans, const int32_t* last,
                          const float* image_grad, real* accum, real* grid_grad) {
    // the fp64 parity build's scratch (static header slots + dynamic reduction rows) exceeds the 48 KB default;
    // (texel-gradient stride, texel layout) in {(3, 3), (4, 3), (4, 4)}
    static const cudaError_t opt_in = [] {
        const int bytes = (int)red_smem(256);
        cudaError_t e = cudaFuncSetAttribute(k_backward_direct<MODE, NT, 3, 3>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(k_backward_direct<MODE, NT, 4, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     bytes);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(k_backward_direct<MODE, NT, 4, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     bytes);
        return e;
    }();
    if (opt_in != cudaSuccess) return opt_in;
    if (rc.tex4 && rc.tgs != 4) return cudaErrorNotSupported;  // RGBA texels come with RGBA texel gradients
    const size_t smem = red_smem(threads);
    if (rc.tex4)
        k_backward_direct<MODE, NT, 4, 4><<<tiles, threads, smem, st>>>(ranges, values, hdr, cull, tex, cc, rc, n, trans,
                                                                        last, image_grad, accum, grid_grad);
    else if (rc.tgs == 4)
        k_backward_direct<MODE, NT, 4, 3><<<tiles, threads, smem, st>>>(ranges, values, hdr, cull, tex, cc, rc, n, trans,
                                                                        last, image_grad, accum, grid_grad);
    else
        k_backward_direct<MODE, NT, 3, 3><<<tiles, threads, smem, st>>>(ranges, values, hdr, cull, tex, cc, rc, n, trans,
                                                                        last, image_grad, accum, grid_grad);
    return cudaGetLastError();
}

cudaError_t launch_forward(int mode, int n, int tiles, int ts, const uint2* ranges, const int32_t* values,
                           const ScreenHeader* hdr, const CullRec* cull, const float* tex, const CamConst& cc,
                           const RasterConst& rc, float* color, float* trans, int32_t* last, cudaStream_t st) {
    if (tiles == 0) return cudaSuccess;
    const int threads = tile_threads(ts);
    if (mode == GB_MODE_ORTHO) {
        GB_DISPATCH_N(fwdd_t, GB_MODE_ORTHO, tiles, threads, st, ranges, values, hdr, cull, tex, cc, rc, n, color,
                      trans, last)
    } else {
        GB_DISPATCH_N(fwdd_t, GB_MODE_PINHOLE, tiles, threads, st, ranges, values, hdr, cull, tex, cc, rc, n, color,
                      trans, last)
    }
}

cudaError_t launch_backward(int mode, int n, int tiles, int ts, const uint2* ranges, const int32_t* values,
                            const ScreenHeader* hdr, const CullRec* cull, const float* tex, const CamConst& cc,
                            const RasterConst& rc, const float* trans, const int32_t* last, const float* image_grad,
                            real* accum, real* grid_grad, cudaStream_t st) {
    if (tiles == 0) return cudaSuccess;
    const int threads = tile_threads(ts);
    if (mode == GB_MODE_ORTHO) {
        GB_DISPATCH_N(bwdd_t, GB_MODE_ORTHO, tiles, threads, st, ranges, values, hdr, cull, tex, cc, rc, n, trans, last,
                      image_grad, accum, grid_grad)
    } else {
        GB_DISPATCH_N(bwdd_t, GB_MODE_PINHOLE, tiles, threads, st, ranges, values, hdr, cull, tex, cc, rc, n, trans,
                      last, image_grad, accum, grid_grad)
    }
}

template <int MODE, int NT>
static cudaError_t fwdl_t(int tiles, int threads, cudaStream_t st, const uint2* ranges, const int32_t* values,
                          const ScreenHeader* hdr, const CullRec* cull, const float* tex, const CamConst& cc,
                          const RasterConst& rc, int n, int kind, const float* target, float scale, float* color,
                          float* trans, int32_t* last, float* image_grad, float* loss) {
#define GB_FWDL(KIND_, TL_)                                                                                     \
    k_forward_loss<MODE, NT, KIND_, TL_><<<tiles, threads, 0, st>>>(ranges, values, hdr, cull, tex, cc, rc, n, target, \
                                                                    scale, color, trans, last, image_grad, loss)
    if (kind == 0) {
        if (rc.tex4)
            GB_FWDL(0, 4);
        else
            GB_FWDL(0, 3);
    } else {
        if (rc.tex4)
            GB_FWDL(1, 4);
        else
            GB_FWDL(1, 3);
    }
#undef GB_FWDL
    return cudaGetLastError();
}

// K3 + K6: trans, last and image_grad are required, color optional
cudaError_t launch_forward_loss(int mode, int n, int tiles, int ts, const uint2* ranges, const int32_t* values,
                                const ScreenHeader* hdr, const CullRec* cull, const float* tex, const CamConst& cc,
                                const RasterConst& rc, int kind, const float* target, float scale, float* color,
                                float* trans, int32_t* last, float* image_grad, float* loss, cudaStream_t st) {
    if (tiles == 0) return cudaSuccess;
    const int threads = tile_threads(ts);
    if (mode == GB_MODE_ORTHO) {
        GB_DISPATCH_N(fwdl_t, GB_MODE_ORTHO, tiles, threads, st, ranges, values, hdr, cull, tex, cc, rc, n, kind,
                      target, scale, color, trans, last, image_grad, loss)
    } else {
        GB_DISPATCH_N(fwdl_t, GB_MODE_PINHOLE, tiles, threads, st, ranges, values, hdr, cull, tex, cc, rc, n, kind,
                      target, scale, color, trans, last, image_grad, loss)
    }
}

#ifdef GB_FUSED_SINGLE_KERNEL
template <int MODE, int NT>
static cudaError_t fused_t(int tiles, int threads, cudaStream_t st, const uint2* ranges, const int32_t* values,
                           const ScreenHeader* hdr, const CullRec* cull, const float* tex, const CamConst& cc,
                           const RasterConst& rc, int n, int kind, const float* target, float scale, float* color,
                           float* trans, int32_t* last, float* image_grad, float* loss, real* accum,
                           real* grid_grad) {
    if (kind == 0)
        k_fused_direct<MODE, NT, 0><<<tiles, threads, red_smem(threads), st>>>(
            ranges, values, hdr, cull, tex, cc, rc, n, target, scale, color, trans, last, image_grad, loss, accum,
            grid_grad);
    else
        k_fused_direct<MODE, NT, 1><<<tiles, threads, red_smem(threads), st>>>(
            ranges, values, hdr, cull, tex, cc, rc, n, target, scale, color, trans, last, image_grad, loss, accum,
            grid_grad);
    return cudaGetLastError();
}

cudaError_t launch_fused(int mode, int n, int tiles, int ts, const uint2* ranges, const int32_t* values,
                         const ScreenHeader* hdr, const CullRec* cull, const float* tex, const CamConst& cc,
                         const RasterConst& rc, int kind, const float* target, float scale, float* color, float* trans,
                         int32_t* last, float* image_grad, float* loss, real* accum, real* grid_grad,
                         cudaStream_t st) {
    if (tiles == 0) return cudaSuccess;
    const int threads = tile_threads(ts);
    if (mode == GB_MODE_ORTHO) {
        GB_DISPATCH_N(fused_t, GB_MODE_ORTHO, tiles, threads, st, ranges, values, hdr, cull, tex, cc, rc, n, kind,
                      target, scale, color, trans, last, image_grad, loss, accum, grid_grad)
    } else {
        GB_DISPATCH_N(fused_t, GB_MODE_PINHOLE, tiles, threads, st, ranges, values, hdr, cull, tex, cc, rc, n, kind,
                      target, scale, color, trans, last, image_grad, loss, accum, grid_grad)
    }
}
#endif  // GB_FUSED_SINGLE_KERNEL

}  // namespace gb
