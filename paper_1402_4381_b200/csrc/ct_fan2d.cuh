// ct_fan2d.cuh — 2D fan-beam projector pair (K1 fwd2d, K2 back2d), sm_100a, fp32.
//
// Same SF-TR/A1 weights as ct_common.cuh (reading O2 / G1), organised around
// the pixel-corner ("vertex") grid: a pixel's trapezoid breakpoints are the arc
// positions of its four corners, and each corner is shared by four pixels.  Both
// kernels evaluate the vertex positions with the ONE routine `vertex_ch` below and
// the pixel footprint with `pixel_foot` / `foot_weights`, so a_ij is the same fp32
// expression in A and A' (matched pair).
//
//   back2d: CTA = 32x8 pixel tile; per batch of views the CTA evaluates the tile's
//           33x9 vertex positions into shared memory (1.16 atan per pixel-view
//           instead of 5), then thread = pixel gathers its 2-6 sinogram bins per view.
//   fwd2d:  CTA = (32x32 pixel tile, chunk of views); the same vertex table; lane =
//           pixel, warp = row or column; a deterministic shared-memory reduction per
//           tile and an exact 64-bit fixed-point sum over tiles (see fwd2d_tile_kernel).
#pragma once
#include "ct_common.cuh"

namespace ct {

// Pixel-corner ("vertex") coordinates: vertex (vx, vy) is the lower-left corner of
// pixel (ix, iy) = (vx, vy).  Every kernel derives them with these two expressions.
__device__ __forceinline__ float vertex_px(const DevGeom& g, int vx) { return fmaf((float)vx, g.dx, g.x0 - 0.5f * g.dx); }
__device__ __forceinline__ float vertex_py(const DevGeom& g, int vy) { return fmaf((float)vy, g.dy, g.y0 - 0.5f * g.dy); }

// Centred channel coordinate (channel units, fan angle 0 -> 0) of the point (px, py).
// Explicit fmaf/__fmul_rn pin the rounding, so every kernel gets identical bits.
__device__ __forceinline__ float vertex_ch(const DevGeom& g, float sb, float cb, float px, float py) {
    const float along = fmaf(px, sb, fmaf(-py, cb, g.dso));   // > 0: the image is inside the orbit
    const float perp = fmaf(px, cb, __fmul_rn(py, sb));
    return __fmul_rn(fast_atan(__fdividef(perp, along)), g.dsd_ds);
}

// Vertex positions relative to a reference ray (vrel = 1).  The vertex grid is cut into
// kVB x kVB blocks; vertices (kVB bx + i, kVB by + j), i, j in [0, kVB), belong to block
// (bx, by), whose reference is the ray through its vertex (kVB bx + kVB/2, kVB by + kVB/2).
// For a vertex at index offset (di, dj) from the reference, the angle between the two
// source rays is atan(cross / dot) with cross = di Cx + dj Cy and dot = r2 + di Cy - dj Cx
// (square pixels), |cross / dot| <= 0.1 (validated at create; c2: 0.03), so the odd series
// q - q^3/3 + q^5/5 (error < 1.5e-8 rad at the bound) replaces the full atan: one
// reference atan per (block, view).  Forward and back use the same owner block for every
// vertex, so both see identical vertex values.
constexpr int kVB = 8;   // reference block edge (vertices)
constexpr int kVBShift = 3;
static_assert((1 << kVBShift) == kVB, "kVB must be 1 << kVBShift (vertex_tab's block index)");

struct VRef {
    float G;                  // reference arc position (centred channel units)
    float Cx, Cy, r2;
};

__device__ __forceinline__ VRef make_vref(const DevGeom& g, float sb, float cb, int bx, int by) {
    const float px = vertex_px(g, kVB * bx + kVB / 2), py = vertex_py(g, kVB * by + kVB / 2);
    const float A = fmaf(px, sb, fmaf(-py, cb, g.dso));
    const float P = fmaf(px, cb, __fmul_rn(py, sb));
    VRef R;
    R.G = __fmul_rn(fast_atan(__fdividef(P, A)), g.dsd_ds);
    R.Cx = __fmul_rn(g.dx, fmaf(cb, A, -__fmul_rn(sb, P)));
    R.Cy = __fmul_rn(g.dx, fmaf(sb, A, __fmul_rn(cb, P)));
    R.r2 = fmaf(A, A, __fmul_rn(P, P));
    return R;
}

__device__ __forceinline__ float vertex_rel(const DevGeom& g, const VRef& R, float di, float dj) {
    const float cross = fmaf(di, R.Cx, __fmul_rn(dj, R.Cy));
    const float dot = fmaf(di, R.Cy, fmaf(-dj, R.Cx, R.r2));
    const float q = __fdividef(cross, dot), t = __fmul_rn(q, q);
    const float p = fmaf(fmaf(t, 1.0f / 5.0f, -1.0f / 3.0f), t, 1.0f);
    return fmaf(__fmul_rn(q, p), g.dsd_ds, R.G);
}

// Vertex (vx, vy) (global vertex indices) from the reference table of a tile whose first
// block is (bx0, by0); RT[(by - by0) * NBX + (bx - bx0)].
template <int NBX>
__device__ __forceinline__ float vertex_tab(const DevGeom& g, const VRef* RT, int bx0, int by0, int vx, int vy) {
    const VRef& R = RT[((vy >> kVBShift) - by0) * NBX + ((vx >> kVBShift) - bx0)];
    return vertex_rel(g, R, (float)((vx & (kVB - 1)) - kVB / 2), (float)((vy & (kVB - 1)) - kVB / 2));
}

// Footprint of one pixel for one view (centred channel units).
struct Foot2 {
    float t0, t1, t2, t3;   // sorted breakpoints
    float lphi;             // A1 amplitude dx / max(|cos phi0|, |sin phi0|)
    int cA, n;              // first channel, channel count (n <= 0: off the detector)
    bool clL, clR;          // footprint clipped by the detector's left / right edge
};

// CLAMP = false (forward tiles): cA / n describe the unclipped footprint (bins may lie off
// the detector; the caller drops them).  On-detector bin edges are evaluated exactly
// (Trap2), so the weights are bit-identical to the clamped ones.
template <bool CLAMP = true>
__device__ __forceinline__ void pixel_foot(const DevGeom& g, float sb, float cb, float xc, float yc, float v00, float v10,
                                           float v01, float v11, Foot2& f) {
    // The projections of the two diagonals overlap (they cross inside the pixel), so
    // sorting each diagonal's pair gives the breakpoints with 4 more min/max.
    const float a0 = fminf(v00, v11), a1 = fmaxf(v00, v11);
    const float b0 = fminf(v10, v01), b1 = fmaxf(v10, v01);
    f.t0 = fminf(a0, b0); f.t1 = fmaxf(a0, b0);
    f.t2 = fminf(a1, b1); f.t3 = fmaxf(a1, b1);
    const float dirx = fabsf(fmaf(g.dso, sb, xc)), diry = fabsf(fmaf(-g.dso, cb, yc));
    const float lo = fminf(dirx, diry), hi = fmaxf(dirx, diry);
    const float r = __fdividef(lo, hi);
    f.lphi = __fmul_rn(g.dx, sqrt_approx(fmaf(r, r, 1.0f)));
    int a = __float2int_rd(__fadd_rn(f.t0, g.cedge));
    int b = __float2int_rd(__fadd_rn(f.t3, g.cedge));
    if (CLAMP) {
        f.clL = a < 0;
        f.clR = b > g.ns - 1;
        a = max(a, 0);
        b = min(b, g.ns - 1);
    } else {
        f.clL = f.clR = false;
    }
    f.cA = a;
    f.n = b - a + 1;
}

// Unit-height trapezoid CDF in coordinates u = s - t0 (branch-free, degenerate widths
// safe).  F(u) = a^2/(2 w1) + m + b - b^2/(2 w3) with a, m, b the clamped pieces.
// Bin edges: with t0a = t0 + cedge (absolute channel coordinate of t0) and c0 =
// max(cA, 0) the first on-detector bin, u(c) = (c0 - t0a) + (c - c0).  c0 - t0a is exact
// (Sterbenz: c0 = floor(t0a) >= t0a / 2, or c0 = 0), and adding small integers keeps it
// exact, so the clipped (back) and unclipped (forward) footprints evaluate every
// on-detector edge from the same float — bit-identical weights — with one add per edge.
struct Trap2 {
    float w1, t2r, t3r, h0, h3, mass, u0;
    int c0;
    __device__ __forceinline__ Trap2(const DevGeom& g, const Foot2& f) {
        w1 = __fsub_rn(f.t1, f.t0);
        t2r = __fsub_rn(f.t2, f.t0);
        t3r = __fsub_rn(f.t3, f.t0);
        h0 = __fdividef(0.5f, fmaxf(w1, 1e-20f));
        h3 = __fdividef(0.5f, fmaxf(__fsub_rn(t3r, t2r), 1e-20f));
        mass = __fmul_rn(0.5f, __fsub_rn(__fadd_rn(t3r, t2r), w1));   // (t3 + t2 - t1 - t0) / 2
        c0 = max(f.cA, 0);
        u0 = __fsub_rn((float)c0, __fadd_rn(f.t0, g.cedge));
    }
    // Evaluated only at edges with u > 0 (interior edges, and the clipped edge at channel
    // 0 or ns: u0 = c0 - t0a > 0 there), so the rise piece needs no lower clamp; the fall
    // piece keeps both clamps (u may exceed t3r by rounding, and w3 may be ~0).
    // m + b = clamp(u, w1, t3r) - w1 for the flat and fall pieces together.
    __device__ __forceinline__ float F(float u) const {
        const float a = fminf(u, w1);
        const float mb = __fsub_rn(fminf(fmaxf(u, w1), t3r), w1);
        const float b = __fsub_rn(fminf(fmaxf(u, t2r), t3r), t2r);
        return fmaf(-__fmul_rn(b, b), h3, fmaf(__fmul_rn(a, a), h0, mb));
    }
};

// sum_j lphi F_s(cA + j) yk[j]: the n - 1 interior bin edges are evaluated once each.
constexpr int kPre = 4;   // prefetched bins
__device__ __forceinline__ float foot_dot(const DevGeom& g, const Foot2& f, const float* __restrict__ yk) {
    // issue the bin loads before the CDF arithmetic (latency hiding)
    float yv[kPre];
#pragma unroll
    for (int j = 0; j < kPre; j++) yv[j] = (j + 1 < f.n) ? ld_dep(&yk[j]) : 0.0f;
    const float ylast = ld_dep(&yk[f.n - 1]);
    const Trap2 T(g, f);   // clamped footprint: c0 = cA
    // F = 0 left of t0 and F = mass right of t3: only clipped ends need an evaluation
    float Fp = f.clL ? T.F(T.u0) : 0.0f, s = 0.0f;
#pragma unroll
    for (int j = 0; j < kMaxFoot - 1; j++) {
        if (j + 1 >= f.n) break;
        const float Fn = T.F(__fadd_rn(T.u0, (float)(j + 1)));
        s = fmaf(__fsub_rn(Fn, Fp), j < kPre ? yv[j < kPre ? j : 0] : ld_dep(&yk[j]), s);
        Fp = Fn;
    }
    const float Fend = f.clR ? T.F(__fadd_rn(T.u0, (float)f.n)) : T.mass;
    s = fmaf(__fsub_rn(Fend, Fp), ylast, s);
    return f.lphi * s;
}

// ---------------------------------------------------------------------------
// K1 (2D fan): pixel-driven forward projection with a deterministic reduction
// ---------------------------------------------------------------------------
// CTA = (32x32 pixel tile, chunk of kF2VC views).  Per view:
//  (a) the tile's 33x33 vertex positions go to shared memory (1.06 atan per pixel);
//  (b) warp = one pixel row (or column, whichever the rays cross more steeply), lane =
//      pixel; round j (warp-uniform) adds lane l's weight of bin cA_l + j times x_l into
//      the warp's shared channel buffer l % P.  Lanes l and l + P have different cA
//      (consecutive pixels advance >= 1/P channel, validated at create), so every add in
//      one instruction goes to a distinct address: no atomics, fixed order;
//  (c) the 8 x P buffers are summed in fixed order over the tile's channel span and
//      added to the 64-bit fixed-point accumulator acc[k][c] (2^-40 units) with integer
//      atomics, which are exact and order-independent: the result is bit-reproducible.
//      fwd2d_finalize converts, applies the residual epilogue r = scale W (Ax - y) and
//      re-zeroes acc.
#ifndef CT_FWD2D_MINB
#define CT_FWD2D_MINB 1   // min resident CTAs per SM for the register budget (tuning: -D; 4-6 measured slower)
#endif
#ifndef CT_BACK2D_MINB
#define CT_BACK2D_MINB 1
#endif
constexpr int kF2T = 32;      // tile edge (pixels)
constexpr int kF2VC = 8;      // views per CTA
// Fixed-point unit 2^-40: absolute quantum 9.1e-13 per tile partial, range |partial|,
// |A x| < 2^23 = 8.4e6 per detector cell (include/ct_oslalm.h, ct_fwd_proj), i.e. x from
// ~1e-7 to ~1e5 times attenuation scale (0.02 mm^-1) keeps 1e-6 relative accuracy.
constexpr float kFix = 1099511627776.0f;   // 2^40
constexpr double kFixInv = 1.0 / 1099511627776.0;

// NR rounds of the forward tile (NR = warp max of the lanes' bin counts n): round j adds
// lane's bin cA + j.  Bins j >= n add exactly 0 (Fn = Fp = mass); the last round needs no CDF
// (every lane is at or past its right edge).  The CDF is evaluated on every lane and
// selected, so the rounds are branch-free.
template <int NR>
__device__ __forceinline__ void fwd_rounds(float* bp, const Trap2& T, float koff, int n, bool act, float lx,
                                           const float* wb_lo = nullptr, const float* wb_hi = nullptr) {
    float Fp = 0.0f;   // unclipped: F = 0 at the left edge of bin cA
#pragma unroll
    for (int j = 0; j < NR; j++) {
        float Fn = T.mass;
        if (j + 1 < NR) {
            const float Fv = T.F(__fadd_rn(T.u0, koff + (float)(j + 1)));
            Fn = (j + 1 < n) ? Fv : T.mass;
        }
#if CT_DEBUG_CHECKS
        {   // the round's read-modify-writes must hit distinct addresses (no lost update) in range
            const int lane = threadIdx.x & 31;
            const unsigned long long a = act ? (unsigned long long)(bp + j) : ~(unsigned long long)lane;
            CT_DCHECK(__match_any_sync(0xffffffffu, a) == (1u << lane));
            CT_DCHECK(!act || (bp + j >= wb_lo && bp + j < wb_hi));
        }
#endif
        if (act) bp[j] += lx * __fsub_rn(Fn, Fp);
        Fp = Fn;
        __syncwarp();   // round j's stores are visible to round j + 1's loads
    }
}

// PT: the lane-parity buffer count P as a compile-time constant (0: runtime g.fpar)
template <bool VREL, int PT>
__global__ void __launch_bounds__(256, CT_FWD2D_MINB) fwd2d_tile_kernel(DevGeom g, int first, int stride, int count,
                                                        const float* __restrict__ x,
                                                        unsigned long long* __restrict__ acc) {
    extern __shared__ float wb[];                 // [8 warps][P][SPAN]
    __shared__ float xs[kF2T][kF2T + 1];
    __shared__ float V[kF2T + 1][kF2T + 1];
    const int P = PT ? PT : g.fpar, SPAN = g.fspan;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int vx0 = blockIdx.x * kF2T, vy0 = blockIdx.y * kF2T;
    const int nvx = min(kF2T, g.nx - vx0), nvy = min(kF2T, g.ny - vy0);   // valid pixels in the tile
    pdl_trigger();
    pdl_wait();   // x is the previous kernel's output
    x = pdl_after(x);
    bool any = false;
    for (int e = tid; e < kF2T * kF2T; e += 256) {
        const int j = e >> 5, i = e & 31;
        const float v = (i < nvx && j < nvy) ? ld_dep(&x[(vy0 + j) * g.nx + vx0 + i]) : 0.0f;
        xs[j][i] = v;
        any |= v != 0.0f;
    }
    // reference rays of the 5 x 5 vertex blocks that own the tile's 33 x 33 vertices, for
    // every view of the chunk
    constexpr int NBF = kF2T / kVB + 1;
    __shared__ VRef RF[kF2VC][NBF * NBF];
    const int k0 = blockIdx.z * kF2VC, k1 = min(count, k0 + kF2VC);
    const int bx0 = vx0 / kVB, by0 = vy0 / kVB;
    if (VREL)
        for (int e = tid; e < (k1 - k0) * NBF * NBF; e += 256) {
            const int kk = e / (NBF * NBF), b = e - kk * (NBF * NBF);
            const float4 vw = __ldg(&g.views[first + (k0 + kk) * stride]);
            RF[kk][b] = make_vref(g, vw.x, vw.y, bx0 + b % NBF, by0 + b / NBF);
        }
    if (!__syncthreads_or(any)) return;   // nothing to project from this tile
    for (int e = tid; e < 8 * P * SPAN; e += 256) wb[e] = 0.0f;
    float* mybuf = wb + (w * P + lane % P) * SPAN;
    const float xcen = g.x0 + (vx0 + 0.5f * (nvx - 1)) * g.dx, ycen = g.y0 + (vy0 + 0.5f * (nvy - 1)) * g.dy;
    // this thread's vertex coordinates (view-independent)
    const float pxl = vertex_px(g, vx0 + lane), pxe = vertex_px(g, vx0 + kF2T);
    const float pyl = vertex_py(g, vy0 + lane), pye = vertex_py(g, vy0 + kF2T);
    float pyr[4];
#pragma unroll
    for (int r = 0; r < 4; r++) pyr[r] = vertex_py(g, vy0 + w + 8 * r);
    for (int k = k0; k < k1; k++) {
        const float4 vw = __ldg(&g.views[first + k * stride]);
        const float sb = vw.x, cb = vw.y;
        if (VREL) {   // relative to the owner blocks' reference rays (no per-vertex atan)
            const VRef* R = RF[k - k0];
#pragma unroll
            for (int r = 0; r < 4; r++)
                if (lane <= nvx && w + 8 * r <= nvy)
                    V[w + 8 * r][lane] = vertex_tab<NBF>(g, R, bx0, by0, vx0 + lane, vy0 + w + 8 * r);
            if (w == 0 && lane <= nvx && nvy == kF2T) V[kF2T][lane] = vertex_tab<NBF>(g, R, bx0, by0, vx0 + lane, vy0 + kF2T);
            else if (w == 1 && lane <= nvy && nvx == kF2T) V[lane][kF2T] = vertex_tab<NBF>(g, R, bx0, by0, vx0 + kF2T, vy0 + lane);
            else if (w == 2 && lane == 0 && nvx == kF2T && nvy == kF2T)
                V[kF2T][kF2T] = vertex_tab<NBF>(g, R, bx0, by0, vx0 + kF2T, vy0 + kF2T);
        } else if (nvx == kF2T && nvy == kF2T) {   // full tile (uniform branch): no bounds checks
#pragma unroll
            for (int r = 0; r < 4; r++) V[w + 8 * r][lane] = vertex_ch(g, sb, cb, pxl, pyr[r]);
            if (w == 0) V[kF2T][lane] = vertex_ch(g, sb, cb, pxl, pye);          // top vertex row
            else if (w == 1) V[lane][kF2T] = vertex_ch(g, sb, cb, pxe, pyl);     // right vertex column
            else if (w == 2 && lane == 0) V[kF2T][kF2T] = vertex_ch(g, sb, cb, pxe, pye);
        } else {
#pragma unroll
            for (int r = 0; r < 4; r++)
                if (lane <= nvx && w + 8 * r <= nvy) V[w + 8 * r][lane] = vertex_ch(g, sb, cb, pxl, pyr[r]);
            if (w == 0 && lane <= nvx) V[nvy][lane] = vertex_ch(g, sb, cb, pxl, vertex_py(g, vy0 + nvy));
            else if (w == 1 && lane <= nvy) V[lane][nvx] = vertex_ch(g, sb, cb, vertex_px(g, vx0 + nvx), pyl);
        }
        __syncthreads();
        // channel span of the tile: u -> perp/along is linear-fractional, so the arc position is
        // quasi-linear and its extremes over the (convex) tile are at the corners; the margin
        // covers the fp32 error of the vertex values (< 1e-4 channel)
        const float q0 = V[0][0], q1 = V[0][nvx], q2 = V[nvy][0], q3 = V[nvy][nvx];
        const float tmin = fminf(fminf(q0, q1), fminf(q2, q3)) - 2e-3f, tmax = fmaxf(fmaxf(q0, q1), fmaxf(q2, q3)) + 2e-3f;
        const int cLoU = __float2int_rd(__fadd_rn(tmin, g.cedge));   // unclipped span
        const int cHiU = __float2int_rd(__fadd_rn(tmax, g.cedge));
        const bool hit = cHiU >= 0 && cLoU <= g.ns - 1;
        if (hit) {
            // rays cross rows steeply (|d_y| >= |d_x|): warps walk rows, lanes = ix
            const bool rowmode = fabsf(ycen - g.dso * cb) >= fabsf(xcen + g.dso * sb);
#pragma unroll 1
            for (int q = 0; q < kF2T / 8; q++) {
                const int il = rowmode ? lane : w + 8 * q, jl = rowmode ? w + 8 * q : lane;
                const float xv = xs[jl][il];
                const bool act = xv != 0.0f;
                Foot2 f;
                int n = 0;
                if (act) {
                    pixel_foot<false>(g, sb, cb, fmaf((float)(vx0 + il), g.dx, g.x0), fmaf((float)(vy0 + jl), g.dy, g.y0),
                                      V[jl][il], V[jl][il + 1], V[jl + 1][il], V[jl + 1][il + 1], f);
                    n = f.n;
                }
                const int nmax = __reduce_max_sync(0xffffffffu, n);
                if (nmax == 0) continue;
                const Trap2 T(g, f);
                const float lx = f.lphi * xv;
                float* bp = mybuf + (f.cA - cLoU);
                // edge cA + j + 1 = c0 + k, k = (cA - c0) + j + 1 an exact small integer in fp32:
                // u = u0 + k rounds exactly as in the back-projector (edges left of channel 0
                // only feed dropped bins)
                const float koff = (float)(f.cA - T.c0);
                // warp-uniform round count: straight-line rounds, no per-round branches
                switch (nmax) {
                    case 1: fwd_rounds<1>(bp, T, koff, n, act, lx, wb, wb + 8 * P * SPAN); break;
                    case 2: fwd_rounds<2>(bp, T, koff, n, act, lx, wb, wb + 8 * P * SPAN); break;
                    case 3: fwd_rounds<3>(bp, T, koff, n, act, lx, wb, wb + 8 * P * SPAN); break;
                    case 4: fwd_rounds<4>(bp, T, koff, n, act, lx, wb, wb + 8 * P * SPAN); break;
                    case 5: fwd_rounds<5>(bp, T, koff, n, act, lx, wb, wb + 8 * P * SPAN); break;
                    case 6: fwd_rounds<6>(bp, T, koff, n, act, lx, wb, wb + 8 * P * SPAN); break;
                    case 7: fwd_rounds<7>(bp, T, koff, n, act, lx, wb, wb + 8 * P * SPAN); break;
                    default: fwd_rounds<kMaxFoot>(bp, T, koff, n, act, lx, wb, wb + 8 * P * SPAN); break;
                }
            }
        }
        __syncthreads();
        if (hit) {
            const int span = cHiU - cLoU + 1;
            unsigned long long* ak = acc + (size_t)k * g.ns;
            for (int t = tid; t < span; t += 256) {
                float s = 0.0f;
                for (int b = 0; b < 8 * P; b++) {
                    s += wb[b * SPAN + t];
                    wb[b * SPAN + t] = 0.0f;
                }
                const int c = cLoU + t;
                if (s != 0.0f && c >= 0 && c < g.ns) atomicAdd(ak + c, (unsigned long long)__float2ll_rn(s * kFix));
            }
        }
        // the next view's vertex phase writes V only after every warp passed this barrier
        __syncthreads();
    }
}

// out[k][c] = acc * 2^-40 (RESID: scale W (Ax - y)); acc is re-zeroed for the next launch.
template <bool RESID>
__global__ void __launch_bounds__(256) fwd2d_finalize_kernel(DevGeom g, int first, int stride, int count,
                                                            unsigned long long* __restrict__ acc, float* __restrict__ out,
                                                            const float* __restrict__ yobs, const float* __restrict__ wts,
                                                            float scale) {
    pdl_trigger();
    pdl_wait();
    acc = pdl_after(acc);
    const int i = blockIdx.x * 256 + threadIdx.x;
    if (i >= count * g.ns) return;
    const long long q = (long long)acc[i];
    acc[i] = 0ull;
    const float s = (float)((double)q * kFixInv);
    if (RESID) {
        const int k = i / g.ns, c = i - k * g.ns;
        const size_t gi = (size_t)(first + k * stride) * g.ns + c;
        const float yo = yobs ? __ldg(&yobs[gi]) : 0.0f;
        out[i] = scale * __ldg(&wts[gi]) * (s - yo);
    } else {
        out[i] = s;
    }
}

// ---------------------------------------------------------------------------
// K2 (2D fan): voxel-driven back projection, one thread per pixel
// ---------------------------------------------------------------------------
// CTA = 32x8 pixel tile.  Per batch of kB2VB views the warps fill the tile's 33x9
// vertex table for every view (warp w: vertex row w; the top row and right column of
// view kk by warp kk % 8), then thread = pixel walks the batch's views.
constexpr int kB2VB = 16;   // views per vertex-table batch
static_assert(2 * (32 / kVB + 1) * kB2VB <= 256, "back2d: one thread per (view, reference block) of a batch");

template <int EPI, bool VREL>
__global__ void __launch_bounds__(256, CT_BACK2D_MINB) back2d_kernel(DevGeom g, int first, int stride, int count,
                                                    const float* __restrict__ y, float* __restrict__ x, GupdArgs ga) {
    __shared__ float V[kB2VB][9][33];
    __shared__ float2 SC[kB2VB];
    constexpr int NBB = 32 / kVB + 1;   // vertex blocks across the tile's 33 vertex columns
    __shared__ VRef RB[kB2VB][2 * NBB];   // vrel: reference rays of the owner blocks (see VRef)
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int ix = blockIdx.x * 32 + lane;
    const int iy = blockIdx.y * 8 + w;
    const bool valid = ix < g.nx && iy < g.ny;
    const size_t jv = (size_t)(valid ? iy : 0) * g.nx + (valid ? ix : 0);
    // voxels outside the support S are not needed by OS-LALM / D_L: skip their views
    const bool act = valid && (ga.mask == nullptr || ga.mask[jv]);   // the mask is static
    float acc = 0.0f;
    pdl_trigger();
    if (__syncthreads_or(act)) {
        const int vx0 = blockIdx.x * 32, vy0 = blockIdx.y * 8;
        const float pxl = vertex_px(g, vx0 + lane), pxe = vertex_px(g, vx0 + 32);
        const float pyw = vertex_py(g, vy0 + w), pye = vertex_py(g, vy0 + 8), pyl = vertex_py(g, vy0 + min(lane, 8));
        const float xc = fmaf((float)ix, g.dx, g.x0), yc = fmaf((float)iy, g.dy, g.y0);
        // vrel: the tile's 9 vertex rows lie in vertex-block rows by0 (rows 0-7) and by0 + 1 (row 8)
        const int bx0 = vx0 / kVB, by0 = vy0 / kVB;
        for (int kb = 0; kb < count; kb += kB2VB) {
            const int nb = min(kB2VB, count - kb);
            if (VREL) {
                if (threadIdx.x < 2 * NBB * nb) {
                    const int kk = threadIdx.x / (2 * NBB), q = threadIdx.x - kk * (2 * NBB);
                    const float4 vw = __ldg(&g.views[first + (kb + kk) * stride]);
                    RB[kk][q] = make_vref(g, vw.x, vw.y, bx0 + q % NBB, by0 + q / NBB);
                }
                __syncthreads();
                for (int kk = 0; kk < nb; kk++) {
                    const VRef* R = RB[kk];
                    V[kk][w][lane] = vertex_tab<NBB>(g, R, bx0, by0, vx0 + lane, vy0 + w);
                    if ((kk & 7) == w) {
                        V[kk][8][lane] = vertex_tab<NBB>(g, R, bx0, by0, vx0 + lane, vy0 + 8);   // top row
                        if (lane <= 8)                                                            // right column
                            V[kk][lane][32] = vertex_tab<NBB>(g, R, bx0, by0, vx0 + 32, vy0 + lane);
                        if (lane == 0) {
                            const float4 vw = __ldg(&g.views[first + (kb + kk) * stride]);
                            SC[kk] = make_float2(vw.x, vw.y);
                        }
                    }
                }
            } else {
                for (int kk = 0; kk < nb; kk++) {
                    const float4 vw = __ldg(&g.views[first + (kb + kk) * stride]);
                    V[kk][w][lane] = vertex_ch(g, vw.x, vw.y, pxl, pyw);
                    if ((kk & 7) == w) {
                        V[kk][8][lane] = vertex_ch(g, vw.x, vw.y, pxl, pye);                   // top row
                        if (lane <= 8) V[kk][lane][32] = vertex_ch(g, vw.x, vw.y, pxe, pyl);   // right column
                        if (lane == 0) SC[kk] = make_float2(vw.x, vw.y);
                    }
                }
            }
            if (kb == 0) pdl_wait();   // the vertex tables depend on the geometry only; y is the predecessor's
            y = pdl_after(y);
            __syncthreads();
            if (act) {
                for (int kk = 0; kk < nb; kk++) {
                    const float2 sc = SC[kk];
                    Foot2 f;
                    pixel_foot(g, sc.x, sc.y, xc, yc, V[kk][w][lane], V[kk][w][lane + 1], V[kk][w + 1][lane],
                               V[kk][w + 1][lane + 1], f);
                    if (f.n <= 0) continue;
                    acc += foot_dot(g, f, y + (size_t)(kb + kk) * g.ns + f.cA);
                }
            }
            __syncthreads();
        }
    }
    pdl_wait();   // (tiles outside S skipped the loop) the epilogue writes G+, g
    ga.G_old = pdl_after(ga.G_old);
    ga.gs = pdl_after(ga.gs);
    ga.rho = pdl_after(ga.rho);
    ga.gbar = pdl_after(ga.gbar);
    const size_t j = (size_t)iy * g.nx + ix;
    const double xi = back_epilogue<EPI>(j, valid, acc, x, ga);
    if (EPI == EPI_GUPD) {
        block_sum_store<256>(xi, &ga.xi_part[blockIdx.y * gridDim.x + blockIdx.x]);
        xi_arrive<256>(ga, gridDim.x * gridDim.y);
    }
}

}  // namespace ct
