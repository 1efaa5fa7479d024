// ct_kernels.cuh — sm_100a kernels of the OS-LALM hot path.
//
//   K1  fwd3d (fwd2d in ct_fan2d.cuh): y_k = A_v x (+ fused weighted residual r = s W (A x - y))
//   K2  back3d (back2d in ct_fan2d.cuh): x = A_v' y  (+ fused g-update / restart-indicator epilogue) P:391-395
//   K3  sqs_update      : rho-scaled non-negative SQS step with the Fair stencil
//   K4  xi_finalize     : fixed-order fp64 sum of xi, counter l and rho_l update
//   K5  (setup)         : D_L = A'(W A 1_S) from K1/K2 + mask finalisation
//   K6  reg_grad        : standalone Fair gradient / Huber curvature
//
// Every projection is a gather: no global or shared float atomics, so results are
// deterministic run to run.  See DESIGN.md §Kernels for the tiling and rooflines.
#pragma once
#include "ct_common.cuh"
#include <type_traits>

namespace ct {

// ---------------------------------------------------------------------------
// Sweep-line wedge of a channel tile (shared by fwd2d / fwd3d)
// ---------------------------------------------------------------------------
// For one view and a tile of channels [c0, c0 + TC), the voxel columns whose
// footprint can reach the tile lie, on each image row (or column), inside the
// interval cut by the tile's two edge rays, widened by the footprint half-width.
struct Wedge {
    bool rows;        // true: lines are image rows (iy fixed, ix varies)
    int nlines;       // ny or nx
    float Sx, Sy;     // source position
    float ka, kb;     // slopes (dx/dy for row lines, dy/dx for column lines) of the edge rays
    float margin;     // in pixels
    bool increasing;  // channel coordinate increases with the in-line index
};

__device__ __forceinline__ void ray_dir(float sb, float cb, float gam, float& dx, float& dy) {
    float cg = __cosf(gam), sg = __sinf(gam);   // |gam| < pi/2; only bounds the wedge
    // d = cos(g) e_c + sin(g) e_perp, e_c = (sb, -cb), e_perp = (cb, sb)
    dx = cg * sb + sg * cb;
    dy = -cg * cb + sg * sb;
}

__device__ __forceinline__ Wedge make_wedge(const DevGeom& g, float sb, float cb, int c0, int tc) {
    Wedge w;
    w.Sx = -g.dso * sb;
    w.Sy = g.dso * cb;
    float ga = ((float)c0 - 0.5f - g.cbase) / g.dsd_ds;
    float gb = ((float)(c0 + tc) - 0.5f - g.cbase) / g.dsd_ds;
    float ax, ay, bx, by, mx, my;
    ray_dir(sb, cb, ga, ax, ay);
    ray_dir(sb, cb, gb, bx, by);
    ray_dir(sb, cb, 0.5f * (ga + gb), mx, my);
    w.rows = fabsf(my) >= fabsf(mx);
    if (w.rows) {
        w.nlines = g.ny;
        w.ka = ax / ay;
        w.kb = bx / by;
        // channel (fan angle) increases with x iff d gamma/dx = -dir.y/rho^2 > 0
        w.increasing = my < 0.0f;
    } else {
        w.nlines = g.nx;
        w.ka = ay / ax;
        w.kb = by / bx;
        // d gamma/dy = dir.x / rho^2
        w.increasing = mx > 0.0f;
    }
    w.margin = 1.0f + 0.5f * fmaxf(fabsf(w.ka), fabsf(w.kb));
    return w;
}

// In-line index range [lo, hi] of line L (clamped); empty if lo > hi.
__device__ __forceinline__ void wedge_line(const DevGeom& g, const Wedge& w, int L, int& lo, int& hi) {
    float a, b;
    if (w.rows) {
        float y = g.y0 + L * g.dy;
        a = w.Sx + (y - w.Sy) * w.ka;
        b = w.Sx + (y - w.Sy) * w.kb;
        float u0 = (fminf(a, b) - g.x0) / g.dx - w.margin, u1 = (fmaxf(a, b) - g.x0) / g.dx + w.margin;
        lo = max(0, __float2int_ru(u0));
        hi = min(g.nx - 1, __float2int_rd(u1));
    } else {
        float x = g.x0 + L * g.dx;
        a = w.Sy + (x - w.Sx) * w.ka;
        b = w.Sy + (x - w.Sx) * w.kb;
        float u0 = (fminf(a, b) - g.y0) / g.dy - w.margin, u1 = (fmaxf(a, b) - g.y0) / g.dy + w.margin;
        lo = max(0, __float2int_ru(u0));
        hi = min(g.ny - 1, __float2int_rd(u1));
    }
}

// ---------------------------------------------------------------------------
// Footprint of one (voxel column, view), computed lane-parallel and broadcast
// to the warp with shuffles (the column's transaxial part is shared by all its
// voxels and, in the forward projector, by all detector rows).
// ---------------------------------------------------------------------------
struct __align__(16) Foot {
    float w[kMaxFoot];      // lphi * F_s(cA + j)
    int cA, n;              // first channel and channel count (n <= 0: misses the detector)
    Axial ax;               // 5 words
    int rows;               // back3d: first active slice | (slice count << 16); fwd3d: 32-bit column base
};
static_assert(sizeof(Foot) == 64, "Foot must be 64 bytes");

__device__ __forceinline__ void load_foot(const Foot* src, Foot& d) {
    const float4* p = reinterpret_cast<const float4*>(src);
    float4 a = p[0], b = p[1], c = p[2], e = p[3];
    d.w[0] = a.x; d.w[1] = a.y; d.w[2] = a.z; d.w[3] = a.w;
    d.w[4] = b.x; d.w[5] = b.y; d.w[6] = b.z; d.w[7] = b.w;
    d.cA = __float_as_int(c.x); d.n = __float_as_int(c.y); d.ax.qi = __float_as_int(c.z); d.ax.qf = c.w;
    d.ax.kz = e.x; d.ax.inv_kz = e.y; d.ax.dz_rho = e.z; d.rows = __float_as_int(e.w);
}

// [clo, chi): channel window the footprint is clipped to (the forward projector's tile;
// the back-projector passes the whole detector).
__device__ __forceinline__ void column_footprint(const DevGeom& g, float4 vw, float xc, float yc, Foot& f,
                                                 int clo = 0, int chi = 0x7fffffff) {
    Trans tr;
    transaxial(g, vw.x, vw.y, xc, yc, tr);
    foot_range(g, tr, f.cA, f.n);
    {
        const int a = max(f.cA, clo), b = min(f.cA + f.n, chi);
        f.cA = a;
        f.n = b - a;
    }
    TrapCdf F(tr);
    float e = (float)f.cA - 0.5f - tr.cc;
    float Fp = F(e);
#pragma unroll
    for (int j = 0; j < kMaxFoot; j++) {
        float Fn = F(e + (float)(j + 1));
        f.w[j] = (j < f.n) ? tr.lphi * (Fn - Fp) : 0.0f;
        Fp = Fn;
    }
    axial(g, vw, tr.rho, f.ax);
}

// ---------------------------------------------------------------------------
// K1 (3D cone): forward projection of one (view, channel tile, all rows)
// ---------------------------------------------------------------------------
// CTA = (tile of TC channels, view k); NTHR threads = G groups of NTP row-threads.
// Group gi walks sweep lines gi, gi+G, ...; the footprints of a line's wedge
// columns are computed group-parallel (one column per thread) into a shared
// table; then, for each column, thread r computes the column's axial sum
//   A(r) = sum_iz x[iz] l_theta(iz) F_t(iz, r)      (z-fastest layout: coalesced)
// and adds lphi F_s(c) A(r) to its own row of the group's shared accumulator
// [channel][row] (thread r is the only writer of row r: no atomics, fixed order).
// Lines are trimmed to the columns that hold a nonzero voxel (fwd3d_extent_kernel).
// Axial sum of one column for detector row r (forward projector):
//   A(r) = sum_iz x[iz] l_theta(iz) F_t(iz, r),  F_t = overlap / kz.
// Table fields (set in the footprint phase): ax.qf = lower edge of row 0's extent
// (voxel units relative to qi), rows = 32-bit index of (column, iz = qi).
// Fast form for kz < 2 (a row meets at most three slices), predicated loads only.
__device__ __forceinline__ float fwd_axial3(const Foot& f, const float* __restrict__ x, int r, int nz, float rbase) {
    if (f.n <= 0) return 0.0f;
    const float lo = fmaf((float)r, f.ax.kz, f.ax.qf);
    const float hi = lo + f.ax.kz;
    const int i0 = __float2int_rd(lo);
    const float z0 = (float)i0;
    const float o0 = fminf(z0 + 1.0f, hi) - lo;
    const float o1 = fminf(fmaxf(hi - (z0 + 1.0f), 0.0f), 1.0f);
    const float o2 = fmaxf(hi - (z0 + 2.0f), 0.0f);
    const float qf = f.ax.qf + (0.5f + rbase) * f.ax.kz;
    const float tz0 = (z0 + 0.5f - qf) * f.ax.dz_rho;
    const float tz1 = tz0 + f.ax.dz_rho, tz2 = tz1 + f.ax.dz_rho;
    const int iz = i0 + f.ax.qi;
    const int idx = f.rows + i0;
    const float v0 = ((unsigned)iz < (unsigned)nz) ? __ldg(x + idx) : 0.0f;
    const float v1 = ((unsigned)(iz + 1) < (unsigned)nz && o1 > 0.0f) ? __ldg(x + idx + 1) : 0.0f;
    const float v2 = ((unsigned)(iz + 2) < (unsigned)nz && o2 > 0.0f) ? __ldg(x + idx + 2) : 0.0f;
    return (v0 * sqrt_approx(fmaf(tz0, tz0, 1.0f)) * o0 + v1 * sqrt_approx(fmaf(tz1, tz1, 1.0f)) * o1 +
            v2 * sqrt_approx(fmaf(tz2, tz2, 1.0f)) * o2) * f.ax.inv_kz;
}

__device__ __forceinline__ float fwd_axial_any(const Foot& f, const float* __restrict__ x, int r, int nz, float rbase) {
    if (f.n <= 0) return 0.0f;
    Axial ax = f.ax;
    ax.qf = f.ax.qf + (0.5f + rbase) * f.ax.kz;
    const float qr = fmaf((float)r, f.ax.kz, f.ax.qf) + 0.5f * f.ax.kz;
    int iz0, iz1;
    row_voxels(ax, qr, iz0, iz1);
    const float* xc = x + (f.rows - f.ax.qi);
    float A = 0.0f;
    for (int iz = max(iz0, 0); iz <= min(iz1, nz - 1); iz++) A += __ldg(&xc[iz]) * ltheta(ax, iz) * axial_weight(ax, qr, iz);
    return A;
}

// Accumulator channels of a tile: a column overlapping the tile starts at most
// kMaxFoot - 1 channels left of it and spans at most kMaxFoot channels.
template <int TC>
__host__ __device__ constexpr int fwd3d_tcp() { return TC + 2 * kMaxFoot - 2; }

// Pair-row forward: footprints are clipped to the tile, so the accumulator holds the tile's
// channels plus the 3 slots the unconditional first-4-channel updates (acc_one) may touch.
#ifndef CT_FWD3D2_CLIP
#define CT_FWD3D2_CLIP 1
#endif
template <int TC>
__host__ __device__ constexpr int fwd3d2_tcp() { return CT_FWD3D2_CLIP ? TC + 3 : fwd3d_tcp<TC>(); }
__host__ __device__ constexpr int fwd3d2_base() { return CT_FWD3D2_CLIP ? 0 : kMaxFoot - 1; }

#ifndef CT_FWD3D_MINB
#define CT_FWD3D_MINB 4   // min resident CTAs per SM for the register budget (A/B: 4 beats 1 by 1.3-1.5x)
#endif


template <int TC, int NTP, int NTHR, bool RESID>
__global__ void __launch_bounds__(NTHR, CT_FWD3D_MINB) fwd3d_kernel(DevGeom g, int first, int stride, const float* __restrict__ x,
                                                     float* __restrict__ out, const float* __restrict__ yobs,
                                                     const float* __restrict__ wts, float scale,
                                                     const int2* __restrict__ ext) {
    constexpr int G = NTHR / NTP;
    constexpr int TCP = fwd3d_tcp<TC>();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* Pacc = reinterpret_cast<float*>(smem_raw);                                    // [G][TCP][NTP]
    Foot* table = reinterpret_cast<Foot*>(smem_raw + sizeof(float) * G * TCP * NTP);     // [G][NTP]
    const int c0 = blockIdx.x * TC;
    const int k = blockIdx.y;
    const int v = first + k * stride;
    const float4 vw = g.views[v];
    const float sb = vw.x, cb = vw.y;
    const int gi = threadIdx.x / NTP, r = threadIdx.x % NTP;
    const bool row_ok = r < g.nt;
    Foot* tab = table + gi * NTP;
    // thread r owns row r of its group's accumulator (stride NTP: distinct banks, no sharing)
    float* Pg = Pacc + gi * TCP * NTP + r;
#pragma unroll
    for (int c = 0; c < TCP; c++) Pg[c * NTP] = 0.0f;
    const Wedge w = make_wedge(g, sb, cb, c0, TC);
    const int nz = g.nz;
    for (int L = gi; L < w.nlines; L += G) {
        int lo, hi;
        wedge_line(g, w, L, lo, hi);
        if (ext) {   // columns of this line that hold a nonzero voxel (fwd3d_extent_kernel)
            const int2 e = __ldg(&ext[w.rows ? L : g.ny + L]);
            lo = max(lo, e.x);
            hi = min(hi, e.y);
        }
        if (lo > hi) continue;
        const int n_in = hi - lo + 1;
        for (int cb0 = 0; cb0 < n_in; cb0 += NTP) {
            // group-parallel footprints of up to NTP columns of this line
            const int q = cb0 + r;
            if (q < n_in) {
                const int u = lo + q;
                const int ix = w.rows ? u : L, iy = w.rows ? L : u;
                Foot f;
                column_footprint(g, vw, g.x0 + ix * g.dx, g.y0 + iy * g.dy, f);
                if (!(f.n > 0 && f.cA + f.n > c0 && f.cA < c0 + TC)) f.n = 0;   // misses the tile
                // forward-projector table: qf -> lower edge of row 0's extent; rows -> 32-bit column base
                f.ax.qf = f.ax.qf - 0.5f * f.ax.kz - g.rbase * f.ax.kz;
                f.rows = (iy * g.nx + ix) * nz + f.ax.qi;
                tab[r] = f;
            }
            asm volatile("bar.sync %0, %1;" ::"r"(gi + 1), "r"(NTP) : "memory");
            const int nq = min(NTP, n_in - cb0);
            // two columns per step: both columns' loads are in flight before either's FMAs
            for (int j = 0; j < nq; j += 2) {
                Foot f0, f1;
                load_foot(&tab[j], f0);
                if (j + 1 < nq) load_foot(&tab[j + 1], f1); else f1.n = 0;
                if (f0.n <= 0 && f1.n <= 0) continue;
                float A0 = 0.0f, A1 = 0.0f;
                if (row_ok) {
                    if (f0.ax.kz < 2.0f && f1.ax.kz < 2.0f) {
                        A0 = fwd_axial3(f0, x, r, nz, g.rbase);
                        A1 = fwd_axial3(f1, x, r, nz, g.rbase);
                    } else {
                        A0 = fwd_axial_any(f0, x, r, nz, g.rbase);
                        A1 = fwd_axial_any(f1, x, r, nz, g.rbase);
                    }
                }
                // lphi F_s(c) A(r) into channels cA..cA+n-1 (warp-uniform n: no divergence)
                if (f0.n > 0) {
                    float* p = Pg + (f0.cA - c0 + kMaxFoot - 1) * NTP;
#pragma unroll
                    for (int jj = 0; jj < kMaxFoot; jj++) {
                        if (jj >= f0.n) break;
                        p[jj * NTP] = fmaf(f0.w[jj], A0, p[jj * NTP]);
                    }
                }
                if (f1.n > 0) {
                    float* p = Pg + (f1.cA - c0 + kMaxFoot - 1) * NTP;
#pragma unroll
                    for (int jj = 0; jj < kMaxFoot; jj++) {
                        if (jj >= f1.n) break;
                        p[jj * NTP] = fmaf(f1.w[jj], A1, p[jj * NTP]);
                    }
                }
            }
            asm volatile("bar.sync %0, %1;" ::"r"(gi + 1), "r"(NTP) : "memory");
        }
    }
    __syncthreads();
    // fixed-order sum over groups; thread (c, r) pairs cover the tile, r fastest
    for (int idx = threadIdx.x; idx < TC * NTP; idx += NTHR) {
        const int c = idx / NTP, rr = idx % NTP;
        if (rr >= g.nt || c0 + c >= g.ns) continue;
        float s = 0.0f;
#pragma unroll
        for (int q = 0; q < G; q++) s += Pacc[(q * TCP + c + kMaxFoot - 1) * NTP + rr];
        const size_t oi = ((size_t)k * g.ns + c0 + c) * g.nt + rr;
        if (RESID) {
            const size_t gidx = ((size_t)v * g.ns + c0 + c) * g.nt + rr;
            const float yo = yobs ? __ldg(&yobs[gidx]) : 0.0f;
            out[oi] = scale * __ldg(&wts[gidx]) * (s - yo);
        } else {
            out[oi] = s;
        }
    }
}

template <int TC, int NTP, int NTHR>
constexpr size_t fwd3d_smem() {
    return sizeof(float) * (NTHR / NTP) * fwd3d_tcp<TC>() * NTP + sizeof(Foot) * NTHR;
}

// ---------------------------------------------------------------------------
// K1 (3D cone), pair-row form for nt <= 64: lane l of a column's LW = 32 / H lanes owns
// detector rows 2l and 2l + 1.  H = 1 (32 < nt <= 64, c3 / c5): warp = one group of
// fwd3d_kernel; H = 2 (nt <= 32, c4): each half-warp is a group with its own accumulator,
// and both halves walk the same line (two columns per half per step).
// ---------------------------------------------------------------------------
// Same wedge walk, column trimming and per-group shared accumulators as fwd3d_kernel;
// the per-column work that does not depend on the row (table loads, branches,
// accumulator addressing) is shared by two rows, the accumulator update is one float2
// read-modify-write, and the two rows' slices are formed once: rows 2l, 2l + 1 cover
// [lo, lo + 2 kz] (voxel units), i.e. slices z0 .. z0 + 4 when kz < 2.
// Table fields (footprint phase): w[j] = lphi F_s(cA + j) / kz (F_t = overlap / kz folded
// in); ax.qf = lower edge of row 0 relative to qi; ax.inv_kz holds tzc, the l_theta
// offset tz(slice qi + m) = m dz_rho + tzc; rows = 32-bit index of (column, slice qi).
#ifndef CT_FWD3D2_UNPRED
#define CT_FWD3D2_UNPRED 0
#endif
#ifndef CT_FWD3D2_INTERIOR
#define CT_FWD3D2_INTERIOR 1   // interior columns (every touched slice inside the volume) skip the volume predicates
#endif
#ifndef CT_FWD3D2_KS
#define CT_FWD3D2_KS 1     // per-column slice-window specialisation (3 / 4 / 5 slices per row pair)
#endif
// Resident CTAs per SM (register budget) is a template parameter: 5 CTAs of 4 warps for
// axial scans (A/B: c3 2.32 -> 2.12 ms vs 4), 6 for helical ones (with 26-channel tiles:
// c5 12.01 -> 11.41, c4 3.72 -> 3.31 ms vs 22 channels / 5 CTAs; c3 prefers the latter).

// KS = slices a lane's row pair can meet: rows 2l, 2l + 1 cover [lo, lo + 2 kz] with
// lo in [z0, z0 + 1), i.e. slices z0 .. z0 + KS - 1 when 1 + 2 kz <= KS (KS = 3: kz <= 1,
// KS = 4: kz <= 1.5, KS = 5: kz < 2); chosen per column (warp-uniform), so near-source
// columns (small kz) do not pay for the far side's longer windows.
// INTERIOR: every slice the column's row pairs can touch lies inside the volume (flagged in
// the table by a negative kz), so only the slices past hi need a predicate.
#ifndef CT_FWD3D2_XHINT
#define CT_FWD3D2_XHINT 0   // 1: x slice loads carry an L2 evict_last policy, the epilogue's y / W / out evict_first
#endif
template <int KS, bool INTERIOR, bool LP>
__device__ __forceinline__ float2 fwd_axial_pair(const Foot& f, const float* __restrict__ x, int l, int nz,
                                                 unsigned long long pol = 0) {
    const float kz = fabsf(f.ax.kz);
    const float lo = fmaf((float)(2 * l), kz, f.ax.qf);
    const float mid = lo + kz, hi = mid + kz;
    const int i0 = __float2int_rd(lo);
    const float z0 = (float)i0;
    const float tz0 = fmaf(z0, f.ax.dz_rho, f.ax.inv_kz);
    const int iz0 = i0 + f.ax.qi;
    const float* xp = x + (f.rows + i0);
    float xl[KS];   // x l_theta of slices z0 .. z0 + KS - 1 (0 outside the volume)
#pragma unroll
    for (int m = 0; m < KS; m++) {
        const float tz = fmaf((float)m, f.ax.dz_rho, tz0);
        // slices past hi get weight 0 below; skipping their loads saves L1 traffic (CT_FWD3D2_UNPRED = 1: load them)
        const bool in = (INTERIOR || (unsigned)(iz0 + m) < (unsigned)nz) && (CT_FWD3D2_UNPRED || m < 2 || z0 + (float)m < hi);
        const float v = in ? (CT_FWD3D2_XHINT ? ldg_pol(xp + m, pol) : __ldg(xp + m)) : 0.0f;
        xl[m] = v * ltheta_of<LP>(tz);
    }
    // row 2l: [lo, mid] meets slices z0 .. z0 + 2 (lo >= z0, kz < 2)
    const float a1 = fminf(z0 + 1.0f, mid), a2 = fminf(z0 + 2.0f, mid);
    float A = xl[0] * (a1 - lo);
    A = fmaf(xl[1], a2 - a1, A);
    A = fmaf(xl[2], mid - a2, A);
    // row 2l + 1: [mid, hi], clamped slice boundaries b(m) = clamp(z0 + m, mid, hi)
    float B = 0.0f, pb = mid;
#pragma unroll
    for (int m = 0; m < KS; m++) {
        const float nb = m < KS - 1 ? fminf(fmaxf(z0 + (float)(m + 1), mid), hi) : hi;
        B = fmaf(xl[m], nb - pb, B);
        pb = nb;
    }
    return make_float2(A, B);
}

// General form (kz >= 2, rarely: very fine slices): one row [lo, hi].
template <bool LP>
__device__ __forceinline__ float fwd_axial_row(const Foot& f, const float* __restrict__ x, float lo, float hi, int nz) {
    float A = 0.0f;
    const int m0 = max(__float2int_rd(lo), -f.ax.qi), m1 = min(__float2int_rd(hi), nz - 1 - f.ax.qi);
    for (int m = m0; m <= m1; m++) {
        const float tz = fmaf((float)m, f.ax.dz_rho, f.ax.inv_kz);
        const float ov = fminf((float)m + 1.0f, hi) - fmaxf((float)m, lo);
        A = fmaf(__ldg(x + f.rows + m) * ltheta_of<LP>(tz), fmaxf(ov, 0.0f), A);
    }
    return A;
}

// Empty column of the pair-row forward's table (misses the tile, or past the batch): kz = 0 and a
// walk that reads x[0 .. 4] (CT_FWD3D2_BOTH evaluates both columns of a pair without branches,
// so that their slice loads issue together; the sums of an empty column are never accumulated).
// nx ny nz >= 5 whenever an interior column exists (its window has >= 5 slices).
__device__ __forceinline__ void empty_foot(Foot& f) {
    f.n = 0;
    f.rows = 0;
    f.ax.kz = 0.0f;
    f.ax.qf = 0.0f;
    f.ax.qi = 0;
    f.ax.dz_rho = 0.0f;
    f.ax.inv_kz = 0.0f;
}
#ifndef CT_FWD3D2_BOTH
#define CT_FWD3D2_BOTH 1   // both columns of a pair evaluated unconditionally (their loads issue together)
#endif

// Accumulator updates of the pair-row forward: p points at the first channel's row pair.
#ifndef CT_FWD3D2_ACC4
#define CT_FWD3D2_ACC4 1   // the first 4 channels unconditionally (their weights past n are exactly 0)
#endif
template <int LW>
__device__ __forceinline__ void acc_one(float2* p, const Foot& f, float2 A, const float2* lo = nullptr,
                                        const float2* hi = nullptr) {
#pragma unroll
    for (int jj = 0; jj < kMaxFoot; jj++) {
        CT_DCHECK(lo == nullptr || (p + jj * LW >= lo && p + jj * LW < hi) || (jj >= f.n && !(CT_FWD3D2_ACC4 && jj < 4)));
        // w[jj] = 0 for jj >= n (column_footprint), and the accumulator has kMaxFoot slots past
        // any first channel, so the first CT_FWD3D2_ACC4 * 4 updates need no count test
        if (!(CT_FWD3D2_ACC4 && jj < 4) && jj >= f.n) break;
        float2 t = p[jj * LW];
        t.x = fmaf(f.w[jj], A.x, t.x);
        t.y = fmaf(f.w[jj], A.y, t.y);
        p[jj * LW] = t;
    }
}

// Two columns whose first channels are D0 / D1 channels past p's (one of D0, D1 is 0).
template <int D0, int D1, int LW>
__device__ __forceinline__ void acc_pair(float2* p, const Foot& f0, float2 A0, const Foot& f1, float2 A1,
                                         const float2* lo = nullptr, const float2* hi = nullptr) {
    constexpr int DM = D0 > D1 ? D0 : D1;
    const int nu = max(D0 + f0.n, D1 + f1.n);
#pragma unroll
    for (int jj = 0; jj < kMaxFoot + DM; jj++) {
        if (jj >= nu) break;
        CT_DCHECK(lo == nullptr || (p + jj * LW >= lo && p + jj * LW < hi));
        float2 t = p[jj * LW];
        if (jj >= D0 && jj - D0 < kMaxFoot && jj - D0 < f0.n) {
            t.x = fmaf(f0.w[jj - D0], A0.x, t.x);
            t.y = fmaf(f0.w[jj - D0], A0.y, t.y);
        }
        if (jj >= D1 && jj - D1 < kMaxFoot && jj - D1 < f1.n) {
            t.x = fmaf(f1.w[jj - D1], A1.x, t.x);
            t.y = fmaf(f1.w[jj - D1], A1.y, t.y);
        }
        p[jj * LW] = t;
    }
}

template <int TC, int NW, int H, bool RESID, int MINB, bool LP>
// [ya, yb): the image rows (iy) this launch projects (the y-split forward projects the two
// halves in two launches so that each launch's working set of x is half a view's slice
// window; `addend` (nullable) holds the first half's sums, added before the epilogue).
__global__ void __launch_bounds__(NW * 32, MINB) fwd3d2_kernel(DevGeom g, int first, int stride,
                                                                     const float* __restrict__ x, float* __restrict__ out,
                                                                     const float* __restrict__ yobs,
                                                                     const float* __restrict__ wts, float scale,
                                                                     const int2* __restrict__ ext, int ya, int yb,
                                                                     const float* __restrict__ addend) {
    constexpr int TCP = fwd3d2_tcp<TC>(), CB = fwd3d2_base();
    constexpr int LW = 32 / H;   // lanes per column (row pairs)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float2* Pacc = reinterpret_cast<float2*>(smem_raw);                                   // [NW][H][TCP][LW]
    Foot* table = reinterpret_cast<Foot*>(smem_raw + sizeof(float2) * NW * TCP * 32);     // [NW][32]
    const int c0 = blockIdx.x * TC;
    const int k = blockIdx.y;
    const int v = first + k * stride;
    const float4 vw = g.views[v];
    const int gi = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int hf = lane / LW, ll = lane % LW;   // half (column stream) and row pair
    Foot* tab = table + gi * 32;
    float2* Pg = Pacc + (gi * H + hf) * TCP * LW + ll;   // rows 2 ll, 2 ll + 1 of stream hf
    const float2* PgLo = CT_DEBUG_CHECKS ? Pacc + (gi * H + hf) * TCP * LW : nullptr;   // this stream's accumulator
    const float2* PgHi = PgLo + TCP * LW;
#pragma unroll
    for (int c = 0; c < TCP; c++) Pg[c * LW] = make_float2(0.0f, 0.0f);
    const Wedge w = make_wedge(g, vw.x, vw.y, c0, TC);
    const int nz = g.nz;
    const unsigned long long xpol = CT_FWD3D2_XHINT ? l2_evict_last() : 0ull;
    // lines: image rows [ya, yb), or every image column trimmed to rows [ya, yb)
    for (int L = (w.rows ? ya : 0) + gi; L < (w.rows ? yb : w.nlines); L += NW) {
        int lo, hi;
        wedge_line(g, w, L, lo, hi);
        if (ext) {
            const int2 e = __ldg(&ext[w.rows ? L : g.ny + L]);
            lo = max(lo, e.x);
            hi = min(hi, e.y);
        }
        if (!w.rows) {
            lo = max(lo, ya);
            hi = min(hi, yb - 1);
        }
        if (lo > hi) continue;
        const int n_in = hi - lo + 1;
        for (int cb0 = 0; cb0 < n_in; cb0 += 32) {
            const int q = cb0 + lane;
            if (q < n_in) {
                const int u = lo + q;
                const int ix = w.rows ? u : L, iy = w.rows ? L : u;
                Foot f;
                if (CT_FWD3D2_CLIP) {
                    column_footprint(g, vw, g.x0 + ix * g.dx, g.y0 + iy * g.dy, f, c0, c0 + TC);   // n <= 0: misses the tile
                } else {
                    column_footprint(g, vw, g.x0 + ix * g.dx, g.y0 + iy * g.dy, f);
                    if (!(f.n > 0 && f.cA + f.n > c0 && f.cA < c0 + TC)) f.n = 0;   // misses the tile
                }
#pragma unroll
                for (int j = 0; j < kMaxFoot; j++) f.w[j] *= f.ax.inv_kz;
                const float qf = f.ax.qf;
                f.ax.qf = qf - 0.5f * f.ax.kz - g.rbase * f.ax.kz;
                f.ax.dz_rho *= lt_scale<LP>();             // (ltheta_of)
                f.ax.inv_kz = (0.5f - qf) * f.ax.dz_rho;   // tzc
                f.rows = (iy * g.nx + ix) * nz + f.ax.qi;
                // interior column: the slices of every lane's row pair (up to 5 past floor(lo)) lie
                // in the volume -> flagged by a negative kz (its uses take |kz|)
                if (CT_FWD3D2_INTERIOR && f.ax.kz < 2.0f) {
                    const int zlo = f.ax.qi + __float2int_rd(f.ax.qf);
                    const int zhi = f.ax.qi + __float2int_rd(fmaf((float)(2 * (LW - 1)), f.ax.kz, f.ax.qf)) + 4;
                    if (zlo >= 0 && zhi <= nz - 1) f.ax.kz = -f.ax.kz;
                }
                if (f.n <= 0) empty_foot(f);   // kz = 0: the pair dispatch below needs no count test
                tab[lane] = f;
            }
            __syncwarp();
            const int nq = min(32, n_in - cb0);
            for (int j0 = 0; j0 < nq; j0 += 2 * H) {
                const int j = j0 + 2 * hf;   // this stream's two columns
                Foot f0, f1;
                if (j < nq) load_foot(&tab[j], f0); else empty_foot(f0);
                if (j + 1 < nq) load_foot(&tab[j + 1], f1); else empty_foot(f1);
                if (f0.n <= 0 && f1.n <= 0) continue;
                float2 A0 = make_float2(0.0f, 0.0f), A1 = A0;
                const float kz0 = fabsf(f0.ax.kz), kz1 = fabsf(f1.ax.kz);
                const float kzm = fmaxf(kz0, kz1);   // empty columns carry kz = 0
                // interior pair (or a single interior column; empty ones carry kz = 0): no volume predicates
                const bool inter = f0.ax.kz <= 0.0f && f1.ax.kz <= 0.0f;
#define CT_FWD3D2_AXIAL(KS_)                                                                   \
    if (CT_FWD3D2_BOTH && inter) {                                                             \
        A0 = fwd_axial_pair<KS_, true, LP>(f0, x, ll, nz, xpol);                                   \
        A1 = fwd_axial_pair<KS_, true, LP>(f1, x, ll, nz, xpol);                                   \
    } else if (CT_FWD3D2_BOTH) {                                                               \
        A0 = fwd_axial_pair<KS_, false, LP>(f0, x, ll, nz, xpol);                                  \
        A1 = fwd_axial_pair<KS_, false, LP>(f1, x, ll, nz, xpol);                                  \
    } else if (inter) {                                                                        \
        if (f0.n > 0) A0 = fwd_axial_pair<KS_, true, LP>(f0, x, ll, nz, xpol);                     \
        if (f1.n > 0) A1 = fwd_axial_pair<KS_, true, LP>(f1, x, ll, nz, xpol);                     \
    } else {                                                                                   \
        if (f0.n > 0) A0 = fwd_axial_pair<KS_, false, LP>(f0, x, ll, nz, xpol);                    \
        if (f1.n > 0) A1 = fwd_axial_pair<KS_, false, LP>(f1, x, ll, nz, xpol);                    \
    }
                if (CT_FWD3D2_KS && kzm <= 0.999f) {
                    CT_FWD3D2_AXIAL(3)
                } else if (CT_FWD3D2_KS && kzm <= 1.499f) {
                    CT_FWD3D2_AXIAL(4)
                } else if (kzm < 2.0f) {
                    CT_FWD3D2_AXIAL(5)
                } else {
                    if (f0.n > 0) {
                        const float l0 = fmaf((float)(2 * ll), kz0, f0.ax.qf);
                        A0 = make_float2(fwd_axial_row<LP>(f0, x, l0, l0 + kz0, nz),
                                         fwd_axial_row<LP>(f0, x, l0 + kz0, l0 + 2.0f * kz0, nz));
                    }
                    if (f1.n > 0) {
                        const float l1 = fmaf((float)(2 * ll), kz1, f1.ax.qf);
                        A1 = make_float2(fwd_axial_row<LP>(f1, x, l1, l1 + kz1, nz),
                                         fwd_axial_row<LP>(f1, x, l1 + kz1, l1 + 2.0f * kz1, nz));
                    }
                }
#undef CT_FWD3D2_AXIAL
                const int dd = f1.cA - f0.cA;
                if (H == 2 && f0.n > 0 && f1.n > 0 && dd >= -3 && dd <= 3) {
                    // adjacent columns' footprints overlap: one read-modify-write per channel of
                    // the union (f0's term first, then f1's, as in the separate loops).  A/B: c4
                    // (half-warp streams) 4.09 -> 3.82 ms; c3 / c5 (H = 1) 1-2 % slower, not used

                    float2* p = Pg + (min(f0.cA, f1.cA) - c0 + CB) * LW;
                    switch (dd) {
                        case -3: acc_pair<3, 0, LW>(p, f0, A0, f1, A1, PgLo, PgHi); break;
                        case -2: acc_pair<2, 0, LW>(p, f0, A0, f1, A1, PgLo, PgHi); break;
                        case -1: acc_pair<1, 0, LW>(p, f0, A0, f1, A1, PgLo, PgHi); break;
                        case 0: acc_pair<0, 0, LW>(p, f0, A0, f1, A1, PgLo, PgHi); break;
                        case 1: acc_pair<0, 1, LW>(p, f0, A0, f1, A1, PgLo, PgHi); break;
                        case 2: acc_pair<0, 2, LW>(p, f0, A0, f1, A1, PgLo, PgHi); break;
                        default: acc_pair<0, 3, LW>(p, f0, A0, f1, A1, PgLo, PgHi); break;
                    }
                } else {
                    if (f0.n > 0) acc_one<LW>(Pg + (f0.cA - c0 + CB) * LW, f0, A0, PgLo, PgHi);
                    if (f1.n > 0) acc_one<LW>(Pg + (f1.cA - c0 + CB) * LW, f1, A1, PgLo, PgHi);
                }
            }
            __syncwarp();
        }
    }
    __syncthreads();
    // fixed-order sum over the NW * H groups; (c, r) pairs cover the tile, r fastest
    constexpr int RW = 2 * LW;   // rows per group
    const float* Pf = reinterpret_cast<const float*>(Pacc);
    for (int idx = threadIdx.x; idx < TC * RW; idx += NW * 32) {
        const int c = idx / RW, rr = idx % RW;
        if (rr >= g.nt || c0 + c >= g.ns) continue;
        float s = 0.0f;
#pragma unroll
        for (int q = 0; q < NW * H; q++) s += Pf[(q * TCP + c + CB) * RW + rr];
        const size_t oi = ((size_t)k * g.ns + c0 + c) * g.nt + rr;
        if (addend) s += addend[oi];
        if (CT_FWD3D2_XHINT) {   // streamed once: evict first
            const unsigned long long ef = l2_evict_first();
            if (RESID) {
                const size_t gidx = ((size_t)v * g.ns + c0 + c) * g.nt + rr;
                const float yo = yobs ? ldg_pol(&yobs[gidx], ef) : 0.0f;
                stg_pol(&out[oi], scale * ldg_pol(&wts[gidx], ef) * (s - yo), ef);
            } else {
                stg_pol(&out[oi], s, ef);
            }
        } else if (RESID) {
            const size_t gidx = ((size_t)v * g.ns + c0 + c) * g.nt + rr;
            const float yo = yobs ? __ldg(&yobs[gidx]) : 0.0f;
            out[oi] = scale * __ldg(&wts[gidx]) * (s - yo);
        } else {
            out[oi] = s;
        }
    }
}

template <int TC, int NW>
constexpr size_t fwd3d2_smem() {
    return sizeof(float2) * NW * fwd3d2_tcp<TC>() * 32 + sizeof(Foot) * NW * 32;
}

// Per image line, the range of columns holding a nonzero voxel (forward-projection
// trimming): ext[iy] = [min ix, max ix] over row iy, ext[ny + ix] = [min iy, max iy].
// Integer atomics: order-independent.  Warp = one column (lanes walk z, coalesced).
__global__ void fwd3d_extent_init(int2* ext, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) ext[i] = make_int2(0x7fffffff, -1);
}

__global__ void __launch_bounds__(256) fwd3d_extent_kernel(DevGeom g, const float* __restrict__ x, int2* ext) {
    const int col = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (col >= g.nx * g.ny) return;
    bool any = false;
    const float* xc = x + (size_t)col * g.nz;
    for (int iz = lane; iz < g.nz; iz += 32) any |= __ldg(&xc[iz]) != 0.0f;
    if (__any_sync(0xffffffffu, any) && lane == 0) {
        const int ix = col % g.nx, iy = col / g.nx;
        atomicMin(&ext[iy].x, ix);
        atomicMax(&ext[iy].y, ix);
        atomicMin(&ext[g.ny + ix].x, iy);
        atomicMax(&ext[g.ny + ix].y, iy);
    }
}

// ---------------------------------------------------------------------------
// Back-projection epilogues
// ---------------------------------------------------------------------------
enum BackEpi { EPI_STORE = 0, EPI_ACCUM = 1, EPI_GUPD = 2, EPI_INIT = 3 };

struct Scalars {
    double rho;        // rho for the next inner step
    long long l;       // continuation counter
    long long step;    // inner steps taken
    unsigned int arrive;   // blocks of the current back-projection that have stored their xi partial
    int pad;
    double alpha;      // Barzilai-Borwein scale of the SQS Hessian, H = alpha D_L (1 without BB)
    long long kiter;   // outer iterations completed (BB secant bookkeeping)
    unsigned int arrive_bb;
    int pad2;
};

__device__ __forceinline__ double rho_l(long long l, double rho_min) {
    // rho_0 = 1; rho_l = max{ pi/(l+1) sqrt(1 - (pi/(2l+2))^2), rho_min }
    if (l == 0) return 1.0;
    const double pi = 3.14159265358979323846;
    double a = pi / (double)(l + 1), b = pi / (2.0 * (double)l + 2.0);
    double r = a * sqrt(1.0 - b * b);
    return r > rho_min ? r : rho_min;
}

struct GupdArgs {
    float* G_new;          // G+  (EPI_GUPD) / G (EPI_INIT)
    const float* G_old;    // G   (EPI_GUPD)
    float* gs;             // split gradient g, updated in place
    const uint8_t* mask;   // support S
    const double* rho;     // rho of this inner step (device scalar)
    double* xi_part;       // per-block fp64 partials of xi
    // K4 fused: the last block to finish sums the partials in fixed order and
    // applies the restart rule / rho_l update
    Scalars* sc;
    int mode;
    double rho_fixed, rho_min;
    double* log3;
    int log_slot;
    float* gbar;           // BB (nullable): running mean of the iteration's subset gradients
    float inv_M;
    double* xi_out;        // z-slab ranks (nullable): the last block stores this rank's xi sum here
                           // (all-reduced, then xi_rule_kernel applies K4) instead of finalizing
};

// xi = fixed-order fp64 sum of the partials; l <- (xi > 0) ? 0 : l + 1; rho <- rho_l.
template <int NTHR>
__device__ void xi_finalize_block(const double* part, int nparts, const GupdArgs& ga) {
    __shared__ double red[NTHR];
    double s = 0.0;
    for (int i = threadIdx.x; i < nparts; i += NTHR) s += __ldcg(&part[i]);
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = NTHR / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        Scalars* sc = ga.sc;
        double xi = red[0];
        int restart = xi > 0.0;
        double rho_used = sc->rho;
        if (ga.mode == 1) {
            sc->l = restart ? 0 : sc->l + 1;
            sc->rho = rho_l(sc->l, ga.rho_min);
        } else {
            sc->rho = ga.rho_fixed;
        }
        sc->step += 1;
        if (ga.log3 && ga.log_slot >= 0) {
            ga.log3[3 * ga.log_slot + 0] = rho_used;
            ga.log3[3 * ga.log_slot + 1] = xi;
            ga.log3[3 * ga.log_slot + 2] = restart;
        }
        sc->arrive = 0;   // ready for the next launch (stream order)
    }
}

// Called by every block after its partial is stored: the last arriving block finalises.
template <int NTHR>
__device__ __forceinline__ void xi_arrive(const GupdArgs& ga, int nblocks) {
    __shared__ int last;
    if (threadIdx.x == 0) {
        __threadfence();
        unsigned prev = atomicAdd(&ga.sc->arrive, 1u);
        last = (prev == (unsigned)nblocks - 1u);
    }
    __syncthreads();
    if (last) {
        __threadfence();
        if (ga.xi_out) {
            __shared__ double red[NTHR];
            double s = 0.0;
            for (int i = threadIdx.x; i < nblocks; i += NTHR) s += __ldcg(&ga.xi_part[i]);
            red[threadIdx.x] = s;
            __syncthreads();
            for (int o = NTHR / 2; o > 0; o >>= 1) {
                if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
                __syncthreads();
            }
            if (threadIdx.x == 0) {
                *ga.xi_out = red[0];
                ga.sc->arrive = 0;
            }
        } else {
            xi_finalize_block<NTHR>(ga.xi_part, nblocks, ga);
        }
    }
}

template <int NTHR>
__device__ __forceinline__ void block_sum_store(double val, double* dst) {
    __shared__ double red[NTHR / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) val += __shfl_down_sync(0xffffffffu, val, o);
    int lane = threadIdx.x % 32, wid = threadIdx.x / 32;
    if (lane == 0) red[wid] = val;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < NTHR / 32; i++) s += red[i];
        *dst = s;
    }
}

template <int EPI>
__device__ __forceinline__ double back_epilogue(size_t j, bool valid, float acc, float* x, const GupdArgs& ga) {
    if (!valid) return 0.0;
    if (EPI == EPI_STORE) {
        x[j] = acc;
    } else if (EPI == EPI_ACCUM) {
        x[j] += acc;
    } else if (EPI == EPI_INIT) {
        ga.G_new[j] = acc;
        ga.gs[j] = acc;
    } else {
        float rho = (float)*ga.rho;
        float Gp = acc, G = ga.G_old[j], gg = ga.gs[j];
        ga.G_new[j] = Gp;
        ga.gs[j] = (rho * Gp + gg) / (1.0f + rho);
        if (ga.gbar) ga.gbar[j] += Gp * ga.inv_M;
        if (ga.mask[j]) return (double)(gg - Gp) * (double)(Gp - G);
    }
    return 0.0;
}

// ---------------------------------------------------------------------------
// K2 (3D cone): voxel-driven back projection; warp = one whole voxel column
// ---------------------------------------------------------------------------
// Block = 4x2 columns (8 warps); each warp owns one column's nz slices as
// shared-memory accumulators.  Views are processed in batches of 32: lane l
// computes the column's footprint for view vb + l (and the view's active slice
// range, i.e. the slices its cone meets) into the warp's shared table.  For each
// view the warp then
//  (1) forms the transaxially filtered detector rows  Q(r) = sum_c lphi F_s(c) y[k][c][r]
//      (lanes = rows: unit-stride loads) and their prefix sums (warp scan), and
//  (2) walks only the active slices (lanes = slices): sum_r F_t(iz, r) Q(r) is the
//      integral of the row-wise constant Q over the slice's extent on the detector,
//      PF(u(iz + 1)) - PF(u(iz)) with PF the piecewise-linear cumulative sum.
// Work per (column, view) is proportional to the slices the cone actually meets,
// which matters for helical scans (a view sees ~20-30 % of a long volume).
#ifndef CT_BACK3D_PAIR
#define CT_BACK3D_PAIR 0   // 1: two views per slice walk (one accumulator update per slice for both); A/B: slower (64 registers, 4 CTAs/SM: c5 11.25 -> 12.38 ms)
#endif
// two views per rows phase (half-warps): A/B 32-row detector c4 4.04 -> 3.90 ms (on), 64-row
// detector c5 10.73 -> 10.85 ms without view groups; with view groups (r43) c5 10.18 -> 10.10,
// c3 1.594 -> 1.580 ms (on)
#ifndef CT_BACK3D_ROWS2V_32
#define CT_BACK3D_ROWS2V_32 1
#endif
#ifndef CT_BACK3D_ROWS2V_64
#define CT_BACK3D_ROWS2V_64 1
#endif
#ifndef CT_BACK3D_PREFETCH
#define CT_BACK3D_PREFETCH 0   // 1: L1 prefetch of the next view's detector rows (A/B: c5 11.32 -> 13.08 ms, off)
#endif
#ifndef CT_BACK3D_MINB
// one view per walk: 5 CTAs/SM (A/B c3, c5: beats 4 by 2-3 %; 3 is 12 % slower); two views per
// walk need 64 registers (48 spill ~200 bytes)
#define CT_BACK3D_MINB (CT_BACK3D_PAIR ? 4 : 5)
#endif

constexpr int kBackRows = 128;   // >= nt (validated)
constexpr int kBackPad = 32;     // per-warp accumulator padding past nz (slice-loop tail lanes add 0 there)

__host__ __device__ constexpr size_t back3d_smem_fixed() {
    return sizeof(Foot) * 8 * 32 + sizeof(float2) * 8 * (CT_BACK3D_PAIR ? 2 : 1) * (kBackRows + 4);
}

// Two filtered detector rows (float2) of one view: q = sum_{c < n} w[c] y[c][r..r+1].
template <int NC>
__device__ __forceinline__ void filt_rows2(const float2* __restrict__ yr, int pitch2, bool inr, const Foot& f, float& q0,
                                           float& q1) {
    float2 vv[NC];
#pragma unroll
    for (int c = 0; c < NC; c++) vv[c] = (inr && c < f.n) ? __ldg(yr + c * pitch2) : make_float2(0.0f, 0.0f);
#pragma unroll
    for (int c = 0; c < NC; c++) {
        q0 = fmaf(f.w[c], vv[c].x, q0);
        q1 = fmaf(f.w[c], vv[c].y, q1);
    }
}

template <int NC>
__device__ __forceinline__ void filt_rows1(const float* __restrict__ yr, int pitch, bool inr, const Foot& f, float& q0) {
    float vv[NC];
#pragma unroll
    for (int c = 0; c < NC; c++) vv[c] = (inr && c < f.n) ? __ldg(yr + c * pitch) : 0.0f;
#pragma unroll
    for (int c = 0; c < NC; c++) q0 = fmaf(f.w[c], vv[c], q0);
}

// Filtered detector rows of one (column, view) and their prefix sums into QP (step (1) below).
// QP[k] = (PF[k], Q(r_lo + k)) for k < nr, QP[nr] = (total, 0); returns r_lo, nr.
template <int NTM>
__device__ __forceinline__ void back3d_rows(const DevGeom& g, const Foot& f, const float* __restrict__ yv0, int lane,
                                            float2* QP, int& r_lo, int& nr) {
    const int nt = NTM ? NTM : g.nt;
    r_lo = 0;
    nr = nt;
    if (NTM == 64) {
        // the common 64-row detector: one pass over every row, two rows per lane
        // (the rows the active slices miss are cheap to include)
        const float2* yr = reinterpret_cast<const float2*>(yv0) + lane;
        float q0 = 0.0f, q1 = 0.0f;
        if (f.n <= 3) filt_rows2<3>(yr, 32, true, f, q0, q1);
        else if (f.n <= 4) filt_rows2<4>(yr, 32, true, f, q0, q1);
        else filt_rows2<kMaxFoot>(yr, 32, true, f, q0, q1);
        const float s2 = q0 + q1;
        float inc = s2;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const float t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        const float ex = inc - s2;
        reinterpret_cast<float4*>(QP)[lane] = make_float4(ex, q0, ex + q0, q1);
        if (lane == 31) QP[64] = make_float2(inc, 0.0f);
    } else if (NTM == 32) {
        // 32-row detector: one pass over every row, one row per lane
        const float* yr = yv0 + lane;
        float q0 = 0.0f;
        if (f.n <= 3) filt_rows1<3>(yr, 32, true, f, q0);
        else if (f.n <= 4) filt_rows1<4>(yr, 32, true, f, q0);
        else filt_rows1<kMaxFoot>(yr, 32, true, f, q0);
        float inc = q0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const float t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        QP[lane] = make_float2(inc - q0, q0);
        if (lane == 31) QP[32] = make_float2(inc, 0.0f);
    } else {
        // rows met by the active slices, from an even row (float2 loads)
        const int za = f.rows & 0xffff, nzs = f.rows >> 16;
        const float ub = g.rbase + 0.5f;
        const float zq = (float)(za - f.ax.qi) - f.ax.qf;
        // two rows per lane (float2) for tall detectors; float2 rows need an even row pitch
        const bool even = (nt & 1) == 0 && nt > 32;
        r_lo = min(max(__float2int_rd(fmaf(zq, f.ax.inv_kz, ub)), 0), nt - 1) & (even ? ~1 : ~0);
        const int r_hi = min(max(__float2int_rd(fmaf(zq + (float)nzs, f.ax.inv_kz, ub)), 0), nt - 1);
        nr = r_hi - r_lo + 1;
        const float* yv = yv0 + r_lo;   // < 2^31 (validated at create)
        float carry = 0.0f;
        const int RPL = even ? 2 : 1;
        for (int p0 = 0; p0 < nr; p0 += 32 * RPL) {
            const int p = p0 + RPL * lane;
            const bool inr = p < nr;
            float q0 = 0.0f, q1 = 0.0f;
            if (even) {
                const float2* yr = reinterpret_cast<const float2*>(yv + (inr ? p : 0));
                // warp-uniform channel count: issue all loads, then the FMAs
                if (f.n <= 3) filt_rows2<3>(yr, nt >> 1, inr, f, q0, q1);
                else if (f.n <= 4) filt_rows2<4>(yr, nt >> 1, inr, f, q0, q1);
                else filt_rows2<kMaxFoot>(yr, nt >> 1, inr, f, q0, q1);
                if (p + 1 >= nr) q1 = 0.0f;   // row past r_hi (odd count)
            } else {
                const float* yr = yv + (inr ? p : 0);
                if (f.n <= 3) filt_rows1<3>(yr, nt, inr, f, q0);
                else if (f.n <= 4) filt_rows1<4>(yr, nt, inr, f, q0);
                else filt_rows1<kMaxFoot>(yr, nt, inr, f, q0);
            }
            const float s2 = q0 + q1;
            float inc = s2;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const float t = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += t;
            }
            const float ex = carry + inc - s2;
            if (inr) {
                QP[p] = make_float2(ex, q0);
                if (even) QP[p + 1] = make_float2(ex + q0, q1);
                if (p + RPL >= nr) QP[p + RPL] = make_float2(ex + s2, 0.0f);   // upper edge of the last row
            }
            carry += __shfl_sync(0xffffffffu, inc, 31);
        }
    }
}

// Prefix table of two filtered rows per lane (64-row detector): warp scan of the row pairs.
__device__ __forceinline__ void back3d_qp64(float q0, float q1, int lane, float2* QP) {
    const float s2 = q0 + q1;
    float inc = s2;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const float t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    const float ex = inc - s2;
    reinterpret_cast<float4*>(QP)[lane] = make_float4(ex, q0, ex + q0, q1);
    if (lane == 31) QP[64] = make_float2(inc, 0.0f);
}

// Per-view constants of the slice walk (step (2)): the slice edge zi (voxel units relative to
// the view's qi, minus qf) maps to the detector-row coordinate u = zi inv_kz + ubl in [0, nr].
template <bool LP>
struct SliceWalk {
    float zbase;     // edge of the walk's first slice z0 (voxel units relative to qi, minus qf)
    float zl;        // this lane's edge in pass 0 of a walk starting at slice z0
    float inv_kz, ubl, fnr, dz_rho, hdz;
    const float2* QP;
    // flane = (float)lane (computed once per thread)
    __device__ __forceinline__ void init(const Foot& f, const DevGeom& g, int z0, float flane, int r_lo, int nr,
                                         const float2* qp) {
        zbase = (float)(z0 - f.ax.qi) - f.ax.qf;
        zl = zbase + flane;
        inv_kz = f.ax.inv_kz;
        ubl = g.rbase + 0.5f - (float)r_lo;
        fnr = (float)nr;
        dz_rho = f.ax.dz_rho * lt_scale<LP>();   // (ltheta_of)
        hdz = 0.5f * dz_rho;
        QP = qp;
    }
    // l_theta-weighted integral of the row-wise constant Q over this lane's slice in the pass at
    // offset sf: PF(u(zi + 1)) - PF(u(zi)), the upper edge taken from the next lane.  Edges
    // outside the view's rows clamp to 0 / nr, so slices outside its window contribute 0.
    __device__ __forceinline__ float contrib(float sf) const {
        const float zi = zl + sf;
        const float u = fminf(fmaxf(fmaf(zi, inv_kz, ubl), 0.0f), fnr);
        const int k = __float2int_rd(u);
        const float2 qp = QP[k];
        const float pf = fmaf(u - (float)k, qp.y, qp.x);
        const float up = __shfl_down_sync(0xffffffffu, pf, 1);
        const float tz = fmaf(zi, dz_rho, hdz);
        return ltheta_of<LP>(tz) * (up - pf);
    }
    // PF at the slice edge zi (clamped to the view's rows)
    __device__ __forceinline__ float pf_at(float zi) const {
        const float u = fminf(fmaxf(fmaf(zi, inv_kz, ubl), 0.0f), fnr);
        const int k = __float2int_rd(u);
        const float2 qp = QP[k];
        return fmaf(u - (float)k, qp.y, qp.x);
    }
    // Blocked walk, one pass: lane l takes the S consecutive slices S l .. S l + S - 1 of the walk
    // (edges S l .. S l + S, the last from lane l + 1's first edge), i.e. 32 S - 1 slices with
    // one shuffle per lane instead of S passes of 31 (the per-pass work: loop, shuffle, edge
    // bookkeeping is paid once).  Lane 31's last slice has no upper edge: it adds 0.  acc0 =
    // accumulator of the walk's first slice.
    template <int S>
    __device__ __forceinline__ void walk_blocked(float* acc0, int lane, float flane) const {
        const float zb = fmaf((float)S, flane, zbase);   // this lane's first edge
        float pf[S];
#pragma unroll
        for (int e = 0; e < S; e++) pf[e] = pf_at(zb + (float)e);
        const float up = __shfl_down_sync(0xffffffffu, pf[0], 1);
        float* a = acc0 + S * lane;
#pragma unroll
        for (int e = 0; e < S; e++) {
            const float hi = e + 1 < S ? pf[e + 1] : (lane < 31 ? up : pf[e]);
            const float tz = fmaf(zb + (float)e, dz_rho, hdz);
            a[e] = fmaf(ltheta_of<LP>(tz), hi - pf[e], a[e]);
        }
    }
    // The same pass accumulating into registers (a[e]: slice S lane + e of the walk), for a
    // group of views that share the walk origin (CT_BACK3D_GROUP).
    template <int S>
    __device__ __forceinline__ void walk_reg(float* a, int lane, float flane) const {
        const float zb = fmaf((float)S, flane, zbase);
        float pf[S];
#pragma unroll
        for (int e = 0; e < S; e++) pf[e] = pf_at(zb + (float)e);
        const float up = __shfl_down_sync(0xffffffffu, pf[0], 1);
#pragma unroll
        for (int e = 0; e < S; e++) {
            const float hi = e + 1 < S ? pf[e + 1] : (lane < 31 ? up : pf[e]);
            const float tz = fmaf(zb + (float)e, dz_rho, hdz);
            a[e] = fmaf(ltheta_of<LP>(tz), hi - pf[e], a[e]);
        }
    }
};

#ifndef CT_BACK3D_GROUP
// views per register-accumulated group (power of two <= 32; 0: off): the group's views walk the
// union of their slice windows from one origin, a lane's S slices accumulate in registers and
// reach the shared-memory accumulator once per group instead of once per view
#define CT_BACK3D_GROUP 16   // A/B c5 back: off 10.70, 8 -> 10.25, 16 -> 10.18, 32 -> 10.49 ms (c3 1.66 / 1.61 / 1.59 / 1.60)
#endif
#ifndef CT_BACK3D_GROUP_R2V
#define CT_BACK3D_GROUP_R2V 1   // also in the two-view rows path (32-row detectors)
#endif
#ifndef CT_BACK3D_GROUP_SMEM
#define CT_BACK3D_GROUP_SMEM 1   // the group unions live in the table (0: in registers across the batch; spills)
#endif
#ifndef CT_BACK3D_BLOCKED
#define CT_BACK3D_BLOCKED 1   // one blocked pass (S = 2..4 slices per lane) for windows of 32..127 slices (A/B: c5 11.31 -> 10.88, c3 1.75 -> 1.69 ms)
#endif

// NTM: detector-row specialisation, 64 or 32 (every row in one pass, nt a compile-time
// constant) or 0 (general nt: the rows the active slices meet).
template <int EPI, int NTM, bool LP>
// Image rows [row0, row1) (the multi-rank band exchange back-projects one destination row slab
// per launch so that each slab's blocks travel while the next slab is computed).
__global__ void __launch_bounds__(256, CT_BACK3D_MINB) back3d_kernel(DevGeom g, int first, int stride, int count,
                                                    const float* __restrict__ y, float* __restrict__ x, GupdArgs ga,
                                                    int row0, int row1) {
    extern __shared__ __align__(16) unsigned char sm_raw[];
    constexpr int NQ = CT_BACK3D_PAIR ? 2 : 1;
    Foot* table = reinterpret_cast<Foot*>(sm_raw);
    float2* QPs = reinterpret_cast<float2*>(sm_raw + sizeof(Foot) * 8 * 32);
    float* ACC = reinterpret_cast<float*>(QPs + 8 * NQ * (kBackRows + 4));
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const float flane = (float)lane;
    const int ix = blockIdx.x * 4 + (wid & 3);
    const int iy = row0 + blockIdx.y * 2 + (wid >> 2);
    const bool colok = ix < g.nx && iy < row1;
    const int nt = NTM ? NTM : g.nt, ns = g.ns, nz = g.nz;
    const int col = ((colok ? iy : 0) * g.nx + (colok ? ix : 0)) * nz;
    Foot* tab = table + wid * 32;
    // QP[k] = (PF[k], Q(r_lo + k)): prefix sum of the filtered rows below row r_lo + k and the
    // row itself (one 8-byte load per slice edge); QP[nr] = (total, 0).  Two tables with
    // CT_BACK3D_PAIR (the two views of a slice walk).
    float2* QPA = QPs + wid * NQ * (kBackRows + 4);
    float2* QPB = QPA + (NQ - 1) * (kBackRows + 4);
    float* acc = ACC + wid * (nz + kBackPad);   // + kBackPad: the slice loop's unpredicated tail
    bool any = false;
    for (int iz = lane; iz < nz; iz += 32) {
        acc[iz] = 0.0f;
        // voxels outside the support S are not needed by OS-LALM / D_L
        any |= colok && (ga.mask == nullptr || ga.mask[col + iz]);
    }
    any = __any_sync(0xffffffffu, any);
    if (any) {
        const float xc = g.x0 + ix * g.dx, yc = g.y0 + iy * g.dy;
        for (int vb = 0; vb < count; vb += 32) {
            const int kk = vb + lane;
            int gz0 = 0x7fffffff, gz1 = -1;   // this view's active slices [gz0, gz1) (empty: none)
            if (kk < count) {
                Foot f;
                column_footprint(g, g.views[first + kk * stride], xc, yc, f);
                // slices met by rows [-1/2, nt - 1/2]:  q = qf + (r - rbase) kz  (+ qi)
                const float qa = f.ax.qf + (-0.5f - g.rbase) * f.ax.kz;
                const float qb = f.ax.qf + ((float)nt - 0.5f - g.rbase) * f.ax.kz;
                const int za = max(__float2int_rd(qa) + f.ax.qi, 0);
                const int zb = min(__float2int_rd(qb) + f.ax.qi, nz - 1);
                if (!(f.n > 0 && zb >= za)) f.n = 0;
                f.rows = za | ((zb - za + 1) << 16);
                if (f.n > 0) {
                    gz0 = za;
                    gz1 = zb + 1;
                }
                tab[lane] = f;
            }
#if CT_BACK3D_GROUP
            // union of the slice windows of each group of CT_BACK3D_GROUP consecutive views, kept in
            // the group's first record (its ax.kz field, unused after this phase: origin | count << 16)
#pragma unroll
            for (int o = 1; o < CT_BACK3D_GROUP; o <<= 1) {
                gz0 = min(gz0, __shfl_xor_sync(0xffffffffu, gz0, o));
                gz1 = max(gz1, __shfl_xor_sync(0xffffffffu, gz1, o));
            }
            if (CT_BACK3D_GROUP_SMEM && (lane & (CT_BACK3D_GROUP - 1)) == 0 && kk < count)
                tab[lane].ax.kz = __int_as_float(gz1 > gz0 ? gz0 | ((gz1 - gz0) << 16) : 0);
#endif
            __syncwarp();
            const int nb = min(32, count - vb);
            const float* yb = y + (size_t)vb * ns * nt;   // this batch's views
#if CT_BACK3D_ROWS2V_32 || CT_BACK3D_ROWS2V_64
            if (((NTM == 64 && CT_BACK3D_ROWS2V_64) || (NTM == 32 && CT_BACK3D_ROWS2V_32)) && NQ == 1) {
                // 64- / 32-row detector, two views per rows phase: half-warp h filters view j + h
                // (lane = NTM / 16 rows: float4 / float2 loads), a 16-lane scan per half; then each
                // view's slice walk on the whole warp.  Per view this halves the row loads and the
                // scan steps.
                constexpr int RL = NTM / 16 > 0 ? NTM / 16 : 1, QS = NTM + 2;   // rows per lane, table stride
                const int h = lane >> 4, l16 = lane & 15;
                float2* QPh = QPA + h * QS;   // two (NTM + 1)-entry tables in the warp's 132 slots
                // rows phase of views j, j + 1 into their prefix tables (false: neither meets the column)
                auto rows_pair = [&](int j) -> bool {
                    Foot fh;
                    load_foot(&tab[min(j + h, nb - 1)], fh);   // (a finite record for the idle half)
                    if (j + h >= nb) fh.n = 0;
                    const int nmax = __reduce_max_sync(0xffffffffu, fh.n > 0 ? fh.n : 0);
                    if (nmax <= 0) return false;
                    float q[4] = {0.0f, 0.0f, 0.0f, 0.0f};
                    {
                        const float* yrow = yb + ((j + h) * ns + fh.cA) * NTM + RL * l16;
#define CT_B3_ROWS(NC_)                                                                                       \
    {                                                                                                         \
        float4 vv[NC_];                                                                                       \
        _Pragma("unroll") for (int c = 0; c < NC_; c++) {                                                     \
            if (RL == 4)                                                                                      \
                vv[c] = c < fh.n ? __ldg(reinterpret_cast<const float4*>(yrow + c * NTM)) : make_float4(0, 0, 0, 0); \
            else {                                                                                            \
                const float2 t2 = c < fh.n ? __ldg(reinterpret_cast<const float2*>(yrow + c * NTM)) : make_float2(0, 0); \
                vv[c] = make_float4(t2.x, t2.y, 0.0f, 0.0f);                                                  \
            }                                                                                                 \
        }                                                                                                     \
        _Pragma("unroll") for (int c = 0; c < NC_; c++) {                                                     \
            q[0] = fmaf(fh.w[c], vv[c].x, q[0]);                                                              \
            q[1] = fmaf(fh.w[c], vv[c].y, q[1]);                                                              \
            if (RL == 4) {                                                                                    \
                q[2] = fmaf(fh.w[c], vv[c].z, q[2]);                                                          \
                q[3] = fmaf(fh.w[c], vv[c].w, q[3]);                                                          \
            }                                                                                                 \
        }                                                                                                     \
    }
                        if (nmax <= 3) CT_B3_ROWS(3)
                        else if (nmax <= 4) CT_B3_ROWS(4)
                        else CT_B3_ROWS(kMaxFoot)
#undef CT_B3_ROWS
                    }
                    const float sl = RL == 4 ? (q[0] + q[1]) + (q[2] + q[3]) : q[0] + q[1];
                    float inc = sl;
#pragma unroll
                    for (int o = 1; o < 16; o <<= 1) {
                        const float t = __shfl_up_sync(0xffffffffu, inc, o, 16);
                        if (l16 >= o) inc += t;
                    }
                    const float ex = inc - sl, e1 = ex + q[0];
                    if (RL == 4) {
                        const float e2 = e1 + q[1], e3 = e2 + q[2];
                        reinterpret_cast<float4*>(QPh)[2 * l16] = make_float4(ex, q[0], e1, q[1]);
                        reinterpret_cast<float4*>(QPh)[2 * l16 + 1] = make_float4(e2, q[2], e3, q[3]);
                    } else {
                        reinterpret_cast<float4*>(QPh)[l16] = make_float4(ex, q[0], e1, q[1]);
                    }
                    if (l16 == 15) QPh[NTM] = make_float2(inc, 0.0f);
                    __syncwarp();
                    return true;
                };
                // per-view walks of views j, j + 1 into the shared-memory accumulator
                auto walk_pair = [&](int j) {
#pragma unroll 1
                    for (int v2 = 0; v2 < 2 && j + v2 < nb; v2++) {
                        Foot fw;
                        load_foot(&tab[j + v2], fw);
                        if (fw.n <= 0) continue;
                        const int z0 = fw.rows & 0xffff, nzs = fw.rows >> 16;
                        SliceWalk<LP> w1;
                        w1.init(fw, g, z0, flane, 0, NTM, QPA + v2 * QS);
                        if (CT_BACK3D_BLOCKED && nzs > 31 && nzs <= 63) w1.walk_blocked<2>(acc + z0, lane, flane);
                        else if (CT_BACK3D_BLOCKED && nzs > 63 && nzs <= 95) w1.walk_blocked<3>(acc + z0, lane, flane);
                        else if (CT_BACK3D_BLOCKED && nzs > 95 && nzs <= 127) w1.walk_blocked<4>(acc + z0, lane, flane);
                        else {
                            float* accl = acc + z0 + lane;
                            float sf = 0.0f;
#pragma unroll 1
                            for (int s0 = 0; s0 < nzs; s0 += 31, sf += 31.0f) accl[s0] += w1.contrib(sf);
                        }
                        __syncwarp();
                    }
                };
#if CT_BACK3D_GROUP && CT_BACK3D_GROUP_R2V
                static_assert(CT_BACK3D_GROUP % 2 == 0, "view groups hold whole view pairs");
                for (int g0 = 0; g0 < nb; g0 += CT_BACK3D_GROUP) {
                    const int g1 = min(g0 + CT_BACK3D_GROUP, nb);
#if CT_BACK3D_GROUP_SMEM
                    const int un = __float_as_int(tab[g0].ax.kz);
                    const int uz0 = un & 0xffff, nzu = un >> 16;
#else
                    const int uz0 = __shfl_sync(0xffffffffu, gz0, g0), nzu = __shfl_sync(0xffffffffu, gz1, g0) - uz0;
#endif
                    if (nzu <= 0) continue;
                    auto group = [&](auto SC) {
                        constexpr int S = decltype(SC)::value;
                        float a[S];
#pragma unroll
                        for (int e = 0; e < S; e++) a[e] = 0.0f;
                        for (int j = g0; j < g1; j += 2) {
                            if (!rows_pair(j)) continue;
#pragma unroll 1
                            for (int v2 = 0; v2 < 2 && j + v2 < nb; v2++) {
                                Foot fw;
                                load_foot(&tab[j + v2], fw);
                                if (fw.n <= 0) continue;
                                SliceWalk<LP> w;
                                w.init(fw, g, uz0, flane, 0, NTM, QPA + v2 * QS);
                                w.template walk_reg<S>(a, lane, flane);
                                __syncwarp();
                            }
                        }
                        float* p = acc + uz0 + S * lane;
#pragma unroll
                        for (int e = 0; e < S; e++) p[e] += a[e];
                    };
                    if (nzu <= 31) group(std::integral_constant<int, 1>());
                    else if (nzu <= 63) group(std::integral_constant<int, 2>());
                    else if (nzu <= 95) group(std::integral_constant<int, 3>());
                    else if (nzu <= 127) group(std::integral_constant<int, 4>());
                    else
                        for (int j = g0; j < g1; j += 2)
                            if (rows_pair(j)) walk_pair(j);
                }
#else
                for (int j = 0; j < nb; j += 2)
                    if (rows_pair(j)) walk_pair(j);
#endif
                continue;
            }
#endif
#if CT_BACK3D_GROUP
            if (NQ == 1) {
                for (int g0 = 0; g0 < nb; g0 += CT_BACK3D_GROUP) {
                    const int g1 = min(g0 + CT_BACK3D_GROUP, nb);
#if CT_BACK3D_GROUP_SMEM
                    const int un = __float_as_int(tab[g0].ax.kz);
                    const int uz0 = un & 0xffff, nzu = un >> 16;
#else
                    const int uz0 = __shfl_sync(0xffffffffu, gz0, g0), nzu = __shfl_sync(0xffffffffu, gz1, g0) - uz0;
#endif
                    if (nzu <= 0) continue;   // no view of the group meets the column
                    // the group's views walk [uz0, uz0 + 32 S - 1) (slices outside a view's own window
                    // clamp to the same u: exactly 0); a lane's S slices accumulate in registers
                    auto group = [&](auto SC) {
                        constexpr int S = decltype(SC)::value;
                        float a[S];
#pragma unroll
                        for (int e = 0; e < S; e++) a[e] = 0.0f;
                        for (int j = g0; j < g1; j++) {
                            Foot fa;
                            load_foot(&tab[j], fa);
                            if (fa.n <= 0) continue;
                            int rla = 0, nra = 0;
                            back3d_rows<NTM>(g, fa, yb + (j * ns + fa.cA) * nt, lane, QPA, rla, nra);
                            __syncwarp();
                            SliceWalk<LP> w;
                            w.init(fa, g, uz0, flane, rla, nra, QPA);
                            w.template walk_reg<S>(a, lane, flane);
                            __syncwarp();
                        }
                        float* p = acc + uz0 + S * lane;   // < uz0 + 32 S <= nz + kBackPad
#pragma unroll
                        for (int e = 0; e < S; e++) p[e] += a[e];
                    };
                    if (nzu <= 31) group(std::integral_constant<int, 1>());
                    else if (nzu <= 63) group(std::integral_constant<int, 2>());
                    else if (nzu <= 95) group(std::integral_constant<int, 3>());
                    else if (nzu <= 127) group(std::integral_constant<int, 4>());
                    else {
                        // windows wider than one 4-slice blocked pass: per view, passes of 31 slices
                        for (int j = g0; j < g1; j++) {
                            Foot fa;
                            load_foot(&tab[j], fa);
                            if (fa.n <= 0) continue;
                            int rla = 0, nra = 0;
                            back3d_rows<NTM>(g, fa, yb + (j * ns + fa.cA) * nt, lane, QPA, rla, nra);
                            __syncwarp();
                            const int z0 = fa.rows & 0xffff, nzs = fa.rows >> 16;
                            SliceWalk<LP> w;
                            w.init(fa, g, z0, flane, rla, nra, QPA);
                            float* accl = acc + z0 + lane;
                            float sf = 0.0f;
#pragma unroll 1
                            for (int s0 = 0; s0 < nzs; s0 += 31, sf += 31.0f) accl[s0] += w.contrib(sf);
                            __syncwarp();
                        }
                    }
                }
                continue;
            }
#endif
            for (int j = 0; j < nb; j += NQ) {
#if CT_BACK3D_PREFETCH
                // L1 prefetch of the next view's detector rows ([channel][row] block of n * nt
                // floats, contiguous): their loads in step (1) then hit L1 instead of waiting on L2
                if (j + NQ < nb) {
                    const int* tn = reinterpret_cast<const int*>(&tab[j + NQ]);
                    const int cn = tn[kMaxFoot], nn = tn[kMaxFoot + 1];
                    const int lines = (nn * nt * 4 + 127) >> 7;
                    if (nn > 0 && lane < lines) {
                        const float* pp = y + ((size_t)(vb + j + NQ) * ns + cn) * nt + lane * 32;
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(pp));
                    }
                }
#endif
                Foot fa, fb;
                load_foot(&tab[j], fa);
                if (NQ == 2 && j + 1 < nb) load_foot(&tab[j + 1], fb); else fb.n = 0;
                const bool va = fa.n > 0, vbv = NQ == 2 && fb.n > 0;
                if (!va && !vbv) continue;
                // (1) filtered rows Q(r) = sum_c lphi F_s(c) y[k][c][r] and their prefix sums
                int rla = 0, nra = 0, rlb = 0, nrb = 0;
                // (32-bit offsets within the batch: count * ns * nt < 2^31, validated at create)
                if (va) back3d_rows<NTM>(g, fa, yb + (j * ns + fa.cA) * nt, lane, QPA, rla, nra);
                if (vbv) back3d_rows<NTM>(g, fb, yb + ((j + 1) * ns + fb.cA) * nt, lane, QPB, rlb, nrb);
                __syncwarp();
                // (2) the union of the views' active slices (lanes = slices): per view the integral
                //     of the row-wise constant Q over the slice's extent on the detector,
                //     PF(u(iz + 1)) - PF(u(iz)); lanes evaluate PF at consecutive slice edges and
                //     slice iz takes its upper edge from the next lane, so a pass of 32 edges
                //     completes 31 slices (u = nr, the top edge, reads QP[nr] = (total, 0);
                //     l_theta of slice iz from its lower edge's zi: tz = (zi + 1/2) dz / rho)
                const int zaA = fa.rows & 0xffff, zeA = zaA + (fa.rows >> 16);
                const int zaB = fb.rows & 0xffff, zeB = zaB + (fb.rows >> 16);
                const int z0 = va ? (vbv ? min(zaA, zaB) : zaA) : zaB;
                const int nzs = (va ? (vbv ? max(zeA, zeB) : zeA) : zeB) - z0;
                SliceWalk<LP> wa, wb;
                if (va) wa.init(fa, g, z0, flane, rla, nra, QPA);
                if (vbv) wb.init(fb, g, z0, flane, rlb, nrb, QPB);
                float* accl = acc + z0 + lane;
                float sf = 0.0f;   // (float)s0
#if CT_DEBUG_CHECKS
                for (int s0 = 0; s0 < nzs; s0 += 31) {
                    const float c = (va ? wa.contrib((float)s0) : 0.0f) + (vbv ? wb.contrib((float)s0) : 0.0f);
                    CT_DCHECK(z0 + s0 + lane < nz + kBackPad);
                    // tail lanes add exactly 0, except past the volume's last slice (window clamped
                    // to nz - 1), where they land in the discarded padding slots
                    CT_DCHECK((s0 + lane < nzs && lane < 31) || c == 0.0f || z0 + s0 + lane >= nz);
                }
#endif
                if (va && vbv) {
#pragma unroll 1
                    for (int s0 = 0; s0 < nzs; s0 += 31, sf += 31.0f) {
                        // no predicate: lanes past the union window (and lane 31, whose up = pf) add
                        // exactly 0 (both edges clamp to the same u), or, past a window clamped to the
                        // volume's last slice, land in the padding slots [nz, nz + kBackPad)
                        const float c = wa.contrib(sf) + wb.contrib(sf);
                        accl[s0] += c;
                    }
                } else {
                    const SliceWalk<LP>& w1 = va ? wa : wb;
                    // one blocked pass covers 32 S - 1 slices (tail lanes clamp to 0 or land in the
                    // padding: z0 + 32 S - 1 <= nz + kBackPad - 1 since nzs >= 32 (S - 1))
                    if (CT_BACK3D_BLOCKED && nzs > 31 && nzs <= 63) w1.walk_blocked<2>(acc + z0, lane, flane);
                    else if (CT_BACK3D_BLOCKED && nzs > 63 && nzs <= 95) w1.walk_blocked<3>(acc + z0, lane, flane);
                    else if (CT_BACK3D_BLOCKED && nzs > 95 && nzs <= 127) w1.walk_blocked<4>(acc + z0, lane, flane);
                    else {
#pragma unroll 1   // (A/B: the compiler's unrolled version needs more registers, -5 %)
                        for (int s0 = 0; s0 < nzs; s0 += 31, sf += 31.0f) accl[s0] += w1.contrib(sf);
                    }
                }
                __syncwarp();
            }
        }
    }
    __syncwarp();
    double xi = 0.0;
    for (int iz = lane; iz < nz; iz += 32) xi += back_epilogue<EPI>((size_t)(col + iz), colok, acc[iz], x, ga);
    if (EPI == EPI_GUPD) {
        block_sum_store<256>(xi, &ga.xi_part[blockIdx.y * gridDim.x + blockIdx.x]);
        xi_arrive<256>(ga, gridDim.x * gridDim.y);
    }
}

// ---------------------------------------------------------------------------
// K3: rho-scaled non-negative SQS update with the Fair stencil (one FISTA step)
// ---------------------------------------------------------------------------
// x_new = max(0, x - (rho G + (1-rho) g + grad R(x)) / (rho D_L + D_R(x)))  on S, 0 off S.
// With `grad` != nullptr (K6 standalone) it writes grad R and D_R instead.
template <int NBR>
__device__ __forceinline__ void fair_stencil(const DevGeom& g, const float* __restrict__ x, const uint8_t* __restrict__ m,
                                             int iy, int ix, int iz, float xj, float inv_delta, float& gr, float& cu) {
    const int nx = g.nx, ny = g.ny, nz = g.nz;
    gr = 0.0f;
    cu = 0.0f;
#pragma unroll
    for (int oy = -1; oy <= 1; oy++)
#pragma unroll
        for (int ox = -1; ox <= 1; ox++)
#pragma unroll
            for (int oz = (NBR == 26 ? -1 : 0); oz <= (NBR == 26 ? 1 : 0); oz++) {
                if (oy == 0 && ox == 0 && oz == 0) continue;
                int ky = iy + oy, kx = ix + ox, kz = iz + oz;
                if (ky < 0 || ky >= ny || kx < 0 || kx >= nx || kz < 0 || kz >= nz) continue;
                size_t kk = ((size_t)ky * nx + kx) * nz + kz;
                if (!__ldg(&m[kk])) continue;
                constexpr float r2 = 0.70710678118654752f, r3 = 0.57735026918962576f;
                const int d2 = oy * oy + ox * ox + oz * oz;
                const float wgt = d2 == 1 ? 1.0f : (d2 == 2 ? r2 : r3);
                float dpsi, om;
                fair(xj - __ldg(&x[kk]), inv_delta, dpsi, om);
                gr += wgt * dpsi;
                cu += wgt * om;
            }
}

template <int NBR>
__global__ void __launch_bounds__(256) sqs_update_kernel(DevGeom g, const float* __restrict__ x, float* __restrict__ xn,
                                                        const float* __restrict__ G, const float* __restrict__ gs,
                                                        const float* __restrict__ dl, const uint8_t* __restrict__ m,
                                                        const double* __restrict__ rho_p, const double* __restrict__ alpha_p,
                                                        float beta, float inv_delta, size_t j0, size_t N) {
    // updates voxels [j0, N) (multi-rank: this rank's slab of rows; x is the full image)
    size_t j = j0 + (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= N) return;
    if (!m[j]) {
        xn[j] = 0.0f;
        return;
    }
    const int nz = g.nz;
    int iz = (int)(j % nz);
    size_t c = j / nz;
    int ix = (int)(c % g.nx), iy = (int)(c / g.nx);
    float xj = x[j];
    float gr, cu;
    fair_stencil<NBR>(g, x, m, iy, ix, iz, xj, inv_delta, gr, cu);
    float rho = (float)*rho_p;
    const float ra = rho * (float)*alpha_p;   // rho alpha: H = alpha D_L (BB; alpha = 1 otherwise)
    float s = rho * G[j] + (1.0f - rho) * gs[j];
    float den = ra * dl[j] + 2.0f * beta * cu;
    float v = xj - __fdividef(s + beta * gr, den);
    xn[j] = fmaxf(v, 0.0f);
}

// Boundary slices of the neighbouring z-slab ranks (nullable pointers: no neighbour).
struct ZHalo {
    const float* lo;
    const float* hi;
    const uint8_t* mlo;
    const uint8_t* mhi;
};

// z-slab ranks: out[c] = x[c nz + z] (one slice of every column; c < ncols).
template <class T>
__global__ void zslice_pack_kernel(const T* __restrict__ x, int nz, int z, T* __restrict__ out, int ncols) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c < ncols) out[c] = x[(size_t)c * nz + z];
}

// Sinogram-domain residual (z-slab ranks, after the all-reduce of the partial projections):
// s <- scale W (s - y) in place (y nullable: s <- scale W s, the D_L setup).
__global__ void __launch_bounds__(256) resid_kernel(float* __restrict__ s, const float* __restrict__ yobs,
                                                   const float* __restrict__ wts, int first, int stride, int count,
                                                   int cells_per_view, float scale) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (size_t)count * cells_per_view) return;
    const int k = (int)(i / cells_per_view);
    const size_t gi = (size_t)(first + k * stride) * cells_per_view + (i - (size_t)k * cells_per_view);
    const float yo = yobs ? __ldg(&yobs[gi]) : 0.0f;
    s[i] = scale * __ldg(&wts[gi]) * (s[i] - yo);
}

// 3D (26-neighbour) K3 with shared-memory planes: block = 8 (ix) x 32 (z) voxels
// marching along iy; three planes of x (with a one-voxel halo) rotate through
// shared memory, voxels outside S (or outside the grid) are stored as +inf so the
// "both voxels in S" pair rule costs no branch (fair_masked) and the stencil needs no
// bounds checks.  Streams G, g, D_L once and writes x' once (21 B/voxel of HBM).
constexpr int kK3Y = 8;
#ifndef CT_K3_PIPE
#define CT_K3_PIPE 0   // 1: software-pipelined planes (4 rotating buffers, one barrier per step; A/B c5 0.670 -> 0.683 ms, off)
#endif
#ifndef CT_K3_CLASS
#define CT_K3_CLASS 1   // per-distance-class Fair sums in the 26-neighbour K3 (A/B c5 0.689 -> 0.679 ms)
#endif

template <bool HALO>
__global__ void __launch_bounds__(256) sqs_update3d_kernel(DevGeom g, const float* __restrict__ x, float* __restrict__ xn,
                                                          const float* __restrict__ G, const float* __restrict__ gs,
                                                          const float* __restrict__ dl, const uint8_t* __restrict__ m,
                                                          const double* __restrict__ rho_p,
                                                          const double* __restrict__ alpha_p, float beta, float inv_delta,
                                                          int iy_begin, int iy_end, ZHalo hz) {
    // updates rows [iy_begin, iy_end) (multi-rank: this rank's slab; x is the full image).
    // HALO (z-slab ranks): hz holds the neighbours' boundary slices (z = -1, z = nz) and their mask.
    __shared__ float Pl[CT_K3_PIPE ? 4 : 3][10][34];
    const int tz = threadIdx.x & 31, tx = threadIdx.x >> 5;
    const int ix0 = blockIdx.x * 8, z0 = blockIdx.y * 32, iy0 = iy_begin + blockIdx.z * kK3Y;
    const int nx = g.nx, ny = g.ny, nz = g.nz;
    const float rho = (float)*rho_p;
    const float ra = rho * (float)*alpha_p;   // rho alpha (BB)
    // this thread's (at most two) halo-plane elements: slot, in-plane offset and in-grid flag
    // do not depend on the plane (computed once).  The loads are unconditional (clamped to
    // element 0 outside the grid) and selected afterwards: no branches per plane.
    int pe[2], pj[2], pc[2], ph[2];
    bool pin[2];
#pragma unroll
    for (int q = 0; q < 2; q++) {
        const int e = threadIdx.x + 256 * q;
        const int a = e / 34, b = e - a * 34;
        const int ex = ix0 - 1 + a, ez = z0 - 1 + b;
        const bool inx = e < 340 && ex >= 0 && ex < nx;
        pe[q] = e < 340 ? e : 0;
        pin[q] = inx && ez >= 0 && ez < nz;
        pj[q] = pin[q] ? ex * nz + ez : 0;
        pc[q] = inx ? ex : 0;
        ph[q] = !HALO || !inx ? 0 : (ez == -1 ? 1 : (ez == nz ? 2 : 0));   // halo slice below / above
    }
    const bool two = threadIdx.x + 256 < 340;   // warp-uniform except in one warp
    // a plane's elements in two phases: fetch (global loads into registers) and store (the
    // S / grid selection, the z-slab halo, the shared-memory store), so that a plane's loads
    // can be in flight while the previous planes' stencils are computed
    struct PlaneRaw {
        float xv[2];
        uint8_t mm[2];
    };
    auto fetch_plane = [&](int iy, PlaneRaw& r) {
        const bool rowok = iy >= 0 && iy < ny;
        const int rb = rowok ? iy * nx * nz : 0;
#pragma unroll
        for (int q = 0; q < 2; q++) {
            if (q == 1 && !two) break;
            const int j = rowok && pin[q] ? rb + pj[q] : 0;
            r.mm[q] = __ldg(&m[j]);
            r.xv[q] = __ldg(&x[j]);
        }
    };
    auto store_plane = [&](float* P, int iy, const PlaneRaw& r) {
        const bool rowok = iy >= 0 && iy < ny;
#pragma unroll
        for (int q = 0; q < 2; q++) {
            if (q == 1 && !two) break;
            const bool ok = rowok && pin[q];
            float v = ok && r.mm[q] ? r.xv[q] : __uint_as_float(kOffS);   // not in S
            if (HALO && rowok && ph[q]) {
                const int c = iy * nx + pc[q];
                if (ph[q] == 1 && hz.lo && hz.mlo[c]) v = hz.lo[c];
                if (ph[q] == 2 && hz.hi && hz.mhi[c]) v = hz.hi[c];
            }
            P[pe[q]] = v;
        }
    };
    auto load_plane = [&](float* P, int iy) {
        PlaneRaw r;
        fetch_plane(iy, r);
        store_plane(P, iy, r);
    };
    // rotating planes iy - 1, iy, iy + 1 (pointer rotation instead of slot arithmetic)
    float* Pp = &Pl[0][0][0];
    float* Pc = &Pl[1][0][0];
    float* Pn = &Pl[2][0][0];
#if CT_K3_PIPE
    float* Pf = &Pl[3][0][0];   // plane iy + 2, written during step iy
    load_plane(Pp, iy0 - 1);
    load_plane(Pc, iy0);
    load_plane(Pn, iy0 + 1);
    __syncthreads();
#else
    load_plane(Pp, iy0 - 1);
    load_plane(Pc, iy0);
#endif
    const int ix = ix0 + tx, iz = z0 + tz;
    const bool inb = ix < nx && iz < nz;
    constexpr float r2 = 0.70710678118654752f, r3 = 0.57735026918962576f;
    const int own = (tx + 1) * 34 + tz + 1;   // this voxel's offset in a plane
    for (int t = 0; t < kK3Y; t++) {
        const int iy = iy0 + t;
        if (iy >= iy_end) break;
#if CT_K3_PIPE
        // one barrier per step: plane iy + 2 is fetched now and stored after the stencil into the
        // buffer plane iy - 2 occupied (read in step iy - 1, before the last barrier)
        const bool more = t + 1 < kK3Y && iy + 1 < iy_end;   // CTA-uniform
        PlaneRaw nxt;
        if (more) fetch_plane(iy + 2, nxt);
#else
        load_plane(Pn, iy + 1);
        __syncthreads();
#endif
        if (inb) {
            const int j = (iy * nx + ix) * nz + iz;
            const float xj = Pc[own];
            if (xj == __uint_as_float(kOffS)) {
                xn[j] = 0.0f;   // off S
            } else {
                const float Gj = __ldg(&G[j]), gsj = __ldg(&gs[j]), dlj = __ldg(&dl[j]);   // (in flight during the stencil)
                float gr = 0.0f, cu = 0.0f;
#if CT_K3_CLASS
                // per distance class (6 faces, 12 edges, 8 corners) sum t omega and omega, weight
                // the three class sums at the end: one FFMA and one FADD per neighbour instead of
                // FMUL + 2 FFMA (the weights are common to a class)
                float gs3[3] = {0.0f, 0.0f, 0.0f}, cs3[3] = {0.0f, 0.0f, 0.0f};
#pragma unroll
                for (int oy = -1; oy <= 1; oy++) {
                    const float* Ps = oy < 0 ? Pp : (oy == 0 ? Pc : Pn);
#pragma unroll
                    for (int ox = -1; ox <= 1; ox++)
#pragma unroll
                        for (int oz = -1; oz <= 1; oz++) {
                            if (oy == 0 && ox == 0 && oz == 0) continue;
                            const int cl = oy * oy + ox * ox + oz * oz - 1;
                            fair_masked_acc(xj, Ps[own + ox * 34 + oz], inv_delta, gs3[cl], cs3[cl]);   // 0 off S
                        }
                }
                gr = fmaf(r3, gs3[2], fmaf(r2, gs3[1], gs3[0]));
                cu = fmaf(r3, cs3[2], fmaf(r2, cs3[1], cs3[0]));
#else
#pragma unroll
                for (int oy = -1; oy <= 1; oy++) {
                    const float* Ps = oy < 0 ? Pp : (oy == 0 ? Pc : Pn);
#pragma unroll
                    for (int ox = -1; ox <= 1; ox++)
#pragma unroll
                        for (int oz = -1; oz <= 1; oz++) {
                            if (oy == 0 && ox == 0 && oz == 0) continue;
                            const int d2 = oy * oy + ox * ox + oz * oz;
                            const float wgt = d2 == 1 ? 1.0f : (d2 == 2 ? r2 : r3);
                            float dpsi, om;
                            fair_masked(xj, Ps[own + ox * 34 + oz], inv_delta, dpsi, om);   // 0 off S
                            gr += wgt * dpsi;
                            cu += wgt * om;
                        }
                }
#endif
                const float sdir = rho * Gj + (1.0f - rho) * gsj;
                const float den = ra * dlj + 2.0f * beta * cu;
                xn[j] = fmaxf(xj - __fdividef(sdir + beta * gr, den), 0.0f);
            }
        }
#if CT_K3_PIPE
        if (more) store_plane(Pf, iy + 2, nxt);
        __syncthreads();
        float* tp = Pp;   // iy + 1 becomes the centre plane, iy + 2 the next one
        Pp = Pc;
        Pc = Pn;
        Pn = Pf;
        Pf = tp;
#else
        __syncthreads();
        float* tp = Pp;   // iy + 1 becomes the centre plane
        Pp = Pc;
        Pc = Pn;
        Pn = tp;
#endif
    }
}

// 2D (8-neighbour) K3 with a shared-memory tile: block = 32 (ix) x 8 (iy) pixels, the
// 34 x 10 halo tile of x holds +inf outside S or the grid (pair rule without a branch).
__global__ void __launch_bounds__(256) sqs_update2d_kernel(DevGeom g, const float* __restrict__ x, float* __restrict__ xn,
                                                          const float* __restrict__ G, const float* __restrict__ gs,
                                                          const float* __restrict__ dl, const uint8_t* __restrict__ m,
                                                          const double* __restrict__ rho_p,
                                                          const double* __restrict__ alpha_p, float beta, float inv_delta,
                                                          int iy_begin, int iy_end) {
    // updates rows [iy_begin, iy_end) (multi-rank: this rank's slab; x is the full image)
    __shared__ float T[10][34];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int ix0 = blockIdx.x * 32, iy0 = iy_begin + blockIdx.y * 8;
    const int nx = g.nx;
    const int ix = ix0 + tx, iy = iy0 + ty;
    const bool own = ix < nx && iy < iy_end;
    const int j = own ? iy * nx + ix : 0;
    // halo tile elements e0 = tid, e1 = tid + 256 (< 340); the mask and D_L are static, so
    // they are read before the wait for the previous kernels, and x is read unconditionally
    // next to its mask bit (two independent loads instead of a dependent pair)
    int je[2];
    bool ok[2], me[2];
#pragma unroll
    for (int q = 0; q < 2; q++) {
        const int e = threadIdx.x + 256 * q;
        const int a = e / 34, b = e - a * 34;
        const int ey = iy0 - 1 + a, ex = ix0 - 1 + b;
        ok[q] = e < 340 && ey >= 0 && ey < g.ny && ex >= 0 && ex < nx;
        je[q] = ok[q] ? ey * nx + ex : 0;
        me[q] = ok[q] && __ldg(&m[je[q]]);
    }
    const float dlj = own ? __ldg(&dl[j]) : 0.0f;
    pdl_trigger();
    pdl_wait();   // x, G, g, rho are the previous kernels' outputs
    x = pdl_after(x);
    G = pdl_after(G);
    gs = pdl_after(gs);
    rho_p = pdl_after(rho_p);
    alpha_p = pdl_after(alpha_p);
    float xe[2];
#pragma unroll
    for (int q = 0; q < 2; q++) xe[q] = ok[q] ? ld_dep(&x[je[q]]) : 0.0f;
    const float Gj = own ? ld_dep(&G[j]) : 0.0f, gj = own ? ld_dep(&gs[j]) : 0.0f;
    const float rho = (float)ld_dep(rho_p);
    const float ra = rho * (float)ld_dep(alpha_p);   // rho alpha: H = alpha D_L (BB; alpha = 1 otherwise)
#pragma unroll
    for (int q = 0; q < 2; q++) {
        const int e = threadIdx.x + 256 * q;
        if (e < 340) (&T[0][0])[e] = me[q] ? xe[q] : __uint_as_float(kOffS);   // not in S
    }
    __syncthreads();
    if (!own) return;
    const float xj = T[ty + 1][tx + 1];
    if (xj == __uint_as_float(kOffS)) {
        xn[j] = 0.0f;   // off S
        return;
    }
    constexpr float r2 = 0.70710678118654752f;
    float gr = 0.0f, cu = 0.0f;
#pragma unroll
    for (int oy = -1; oy <= 1; oy++)
#pragma unroll
        for (int ox = -1; ox <= 1; ox++) {
            if (oy == 0 && ox == 0) continue;
            const float wgt = (oy * oy + ox * ox) == 1 ? 1.0f : r2;
            float dpsi, om;
            fair_masked(xj, T[ty + 1 + oy][tx + 1 + ox], inv_delta, dpsi, om);   // 0 off S
            gr += wgt * dpsi;
            cu += wgt * om;
        }
    const float sdir = rho * Gj + (1.0f - rho) * gj;
    const float den = ra * dlj + 2.0f * beta * cu;
    xn[j] = fmaxf(xj - __fdividef(sdir + beta * gr, den), 0.0f);
}

// One FISTA iteration of the inner denoising problem (NEXT-1):
//   x_i = max(0, v - (grad R(v) + rho D_L (v - x_k) + s) / (rho D_L + 2 beta sum w)),  s = rho G + (1-rho) g
//   v_i = x_i + mom (x_i - x_{i-1})            (skipped on the last iteration)
// x_prev may alias x_out (element-wise, read before write).
template <int NBR, bool LAST>
__global__ void __launch_bounds__(256) fista_step_kernel(DevGeom g, const float* __restrict__ v, const float* xprev,
                                                        const float* __restrict__ xk, float* xout, float* __restrict__ vout,
                                                        const float* __restrict__ G, const float* __restrict__ gs,
                                                        const float* __restrict__ dl, const uint8_t* __restrict__ m,
                                                        const double* __restrict__ rho_p, const double* __restrict__ alpha_p,
                                                        float beta, float inv_delta, float mom, size_t N) {
    size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= N) return;
    if (!m[j]) {
        xout[j] = 0.0f;
        if (!LAST) vout[j] = 0.0f;
        return;
    }
    const int nz = g.nz;
    const int iz = (int)(j % nz);
    const size_t c = j / nz;
    const int ix = (int)(c % g.nx), iy = (int)(c / g.nx);
    const float vj = v[j];
    float gr = 0.0f, sw = 0.0f;
#pragma unroll
    for (int oy = -1; oy <= 1; oy++)
#pragma unroll
        for (int ox = -1; ox <= 1; ox++)
#pragma unroll
            for (int oz = (NBR == 26 ? -1 : 0); oz <= (NBR == 26 ? 1 : 0); oz++) {
                if (oy == 0 && ox == 0 && oz == 0) continue;
                const int ky = iy + oy, kx = ix + ox, kz = iz + oz;
                if (ky < 0 || ky >= g.ny || kx < 0 || kx >= g.nx || kz < 0 || kz >= nz) continue;
                const size_t kk = ((size_t)ky * g.nx + kx) * nz + kz;
                if (!__ldg(&m[kk])) continue;
                constexpr float r2 = 0.70710678118654752f, r3 = 0.57735026918962576f;
                const int d2 = oy * oy + ox * ox + oz * oz;
                const float wgt = d2 == 1 ? 1.0f : (d2 == 2 ? r2 : r3);
                float dpsi, om;
                fair(vj - __ldg(&v[kk]), inv_delta, dpsi, om);
                gr += wgt * dpsi;
                sw += wgt;
            }
    const float rho = (float)*rho_p;
    const float rdl = rho * (float)*alpha_p * dl[j];   // rho H, H = alpha D_L (BB)
    const float s = rho * G[j] + (1.0f - rho) * gs[j];
    const float grad = beta * gr + rdl * (vj - xk[j]) + s;
    const float xp = xprev[j];
    const float xn = fmaxf(vj - __fdividef(grad, rdl + 2.0f * beta * sw), 0.0f);
    xout[j] = xn;
    if (!LAST) vout[j] = xn + mom * (xn - xp);
}

template <int NBR>
__global__ void __launch_bounds__(256) reg_grad_kernel(DevGeom g, const float* __restrict__ x, const uint8_t* __restrict__ m,
                                                      float* __restrict__ grad, float* __restrict__ curv, float beta,
                                                      float inv_delta, size_t N) {
    size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= N) return;
    float gr = 0.0f, cu = 0.0f;
    if (m[j]) {
        const int nz = g.nz;
        int iz = (int)(j % nz);
        size_t c = j / nz;
        int ix = (int)(c % g.nx), iy = (int)(c / g.nx);
        fair_stencil<NBR>(g, x, m, iy, ix, iz, x[j], inv_delta, gr, cu);
    }
    grad[j] = beta * gr;
    if (curv) curv[j] = 2.0f * beta * cu;
}

// ---------------------------------------------------------------------------
// Unfused g-update (multi-rank path, after the NCCL all-reduce of G+)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) gupd_kernel(const float* __restrict__ Gp, GupdArgs ga, size_t N) {
    size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    double xi = 0.0;
    if (j < N) {
        float rho = (float)*ga.rho;
        float P = Gp[j], G = ga.G_old[j], gg = ga.gs[j];
        ga.G_new[j] = P;
        ga.gs[j] = (rho * P + gg) / (1.0f + rho);
        if (ga.gbar) ga.gbar[j] += P * ga.inv_M;
        if (ga.mask[j]) xi = (double)(gg - P) * (double)(P - G);
    }
    block_sum_store<256>(xi, &ga.xi_part[blockIdx.x]);
    xi_arrive<256>(ga, gridDim.x);
}

// ---------------------------------------------------------------------------
// Band-limited exchange of the helical multi-rank path: a rank's partial
// back-projection is non-zero only in the z-band of slices its contiguous view block can see,
// and its next forward projection reads x only there.  Blocks of rows [ra, ra + rows) x
// slices [b0, b0 + bl) of an [*][nx][nz] image travel packed as [(iy - ra) nx + ix][z - b0].
// ---------------------------------------------------------------------------
constexpr int kMaxBandRanks = 16;

__global__ void __launch_bounds__(256) band_pack_kernel(const float* __restrict__ img, float* __restrict__ buf, int ra,
                                                       int rows, int nx, int nz, int b0, int bl) {
    const size_t n = (size_t)rows * nx * bl;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const size_t c = i / bl;
        buf[i] = img[((size_t)ra * nx + c) * nz + b0 + (int)(i - c * bl)];
    }
}

__global__ void __launch_bounds__(256) band_unpack_kernel(float* __restrict__ img, const float* __restrict__ buf, int ra,
                                                         int rows, int nx, int nz, int b0, int bl) {
    const size_t n = (size_t)rows * nx * bl;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const size_t c = i / bl;
        img[((size_t)ra * nx + c) * nz + b0 + (int)(i - c * bl)] = buf[i];
    }
}

struct BandSet {
    const float* buf[kMaxBandRanks];   // rank q's block for this rank's rows, slices [b0[q], b1[q])
    int b0[kMaxBandRanks], b1[kMaxBandRanks];
    int P;
};

// dst rows [ra, ra + rows), every slice: the sum over ranks q = 0 .. P-1 (fixed order) of
// rank q's block where the slice lies in its band (0 elsewhere).
__global__ void __launch_bounds__(256) band_sum_kernel(float* __restrict__ dst, int ra, int rows, int nx, int nz,
                                                      BandSet bs) {
    const size_t n = (size_t)rows * nx * nz;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const size_t c = i / nz;
        const int z = (int)(i - c * nz);
        float v = 0.0f;
        for (int q = 0; q < bs.P; q++)
            if (z >= bs.b0[q] && z < bs.b1[q]) v += bs.buf[q][c * (size_t)(bs.b1[q] - bs.b0[q]) + (z - bs.b0[q])];
        dst[(size_t)ra * nx * nz + i] = v;
    }
}

// Windowed exchange of the helical z-slab path: views k < count of this rank's
// view window (the views whose cone reaches its slab).  Each ray is summed over the ranks whose
// windows hold the view, in rank order (the same terms in the same order on every rank that
// holds the view, so those ranks hold identical sums; ranks outside contribute exactly 0 to
// the full sum), then s <- scale W (s - y) as resid_kernel does.
struct ZWinSet {
    const float* buf[kMaxBandRanks];   // rank q's partial for window views [o0[q], o1[q])
    int o0[kMaxBandRanks], o1[kMaxBandRanks];
    int P, self;                       // q = self reads s itself
};

__global__ void __launch_bounds__(256) zwin_sum_resid_kernel(float* __restrict__ s, const float* __restrict__ yobs,
                                                            const float* __restrict__ wts, int first, int stride,
                                                            int count, int cells_per_view, float scale, ZWinSet zs) {
    const size_t n = (size_t)count * cells_per_view;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const int k = (int)(i / cells_per_view);
        const size_t c = i - (size_t)k * cells_per_view;
        float v = 0.0f;
        for (int q = 0; q < zs.P; q++) {
            if (q == zs.self)
                v += s[i];
            else if (k >= zs.o0[q] && k < zs.o1[q])
                v += zs.buf[q][(size_t)(k - zs.o0[q]) * cells_per_view + c];
        }
        const size_t gi = (size_t)(first + k * stride) * cells_per_view + c;
        const float yo = yobs ? __ldg(&yobs[gi]) : 0.0f;
        s[i] = scale * __ldg(&wts[gi]) * (v - yo);
    }
}

// Multi-rank slab path: G+ (already reduce-scattered into G_new[j0, j1)) -> g-update and
// this rank's xi; the last block stores the rank's fixed-order xi sum in *xi_out (the
// ranks' sums are then all-reduced and xi_rule_kernel applies K4 on every rank).
__global__ void __launch_bounds__(256) gupd_slab_kernel(GupdArgs ga, size_t j0, size_t j1, double* xi_out) {
    const size_t j = j0 + (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    double xi = 0.0;
    if (j < j1) {
        const float rho = (float)*ga.rho;
        const float P = ga.G_new[j], G = ga.G_old[j], gg = ga.gs[j];
        ga.gs[j] = (rho * P + gg) / (1.0f + rho);
        if (ga.gbar) ga.gbar[j] += P * ga.inv_M;
        if (ga.mask[j]) xi = (double)(gg - P) * (double)(P - G);
    }
    block_sum_store<256>(xi, &ga.xi_part[blockIdx.x]);
    __shared__ int last;
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned prev = atomicAdd(&ga.sc->arrive, 1u);
        last = (prev == gridDim.x - 1u);
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        double sum = 0.0;
        for (unsigned b = 0; b < gridDim.x; b++) sum += __ldcg(&ga.xi_part[b]);
        *xi_out = sum;
        ga.sc->arrive = 0;
    }
}

// ---------------------------------------------------------------------------
// Barzilai-Borwein scale (NEXT-2, reading B-BB): at the end of outer
// iteration k, over S and voxels [j0, j1) (this rank's rows):
//   num = sum (gbar_k - gbar_{k-1})(xbar_k - xbar_{k-1}),  den = sum D_L (xbar_k - xbar_{k-1})^2  (xbar: the mean of
//   the iteration's inner iterates, the points its subset gradients were taken at),
// then x_prev <- xbar, gbar_prev <- gbar, gbar <- 0, xbar <- 0.  The last block (single rank) sets
// alpha = clip(num / den, alpha_min, 1) once two iterations are complete; with several
// ranks it stores (num, den) for an all-reduce and bb_rule_kernel applies the rule.
struct BBArgs {
    float* xbar;           // mean of the iteration's inner iterates (reset here)
    float* xprev;          // xbar of the previous iteration
    float* gbar;
    float* gprev;
    const float* dl;
    const uint8_t* mask;
    double* part;          // 2 per block
    double* out2;          // multi-rank: this rank's (num, den); nullptr: finalize here
    Scalars* sc;
    double alpha_min;
};

// xbar += x / M over [j0, j1): the mean of the points at which an iteration's subset
// gradients are evaluated (the secant pair of reading B-BB)
__global__ void __launch_bounds__(256) xbar_acc_kernel(float* __restrict__ xbar, const float* __restrict__ x,
                                                       float inv_M, size_t j0, size_t j1) {
    const size_t j = j0 + (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < j1) xbar[j] = fmaf(x[j], inv_M, xbar[j]);
}

__device__ __forceinline__ void bb_rule(Scalars* sc, double num, double den, double alpha_min) {
    sc->kiter += 1;
    if (sc->kiter >= 2) {
        double a = den > 0.0 ? num / den : 1.0;
        sc->alpha = a > 1.0 ? 1.0 : (a < alpha_min ? alpha_min : a);
    }
}

__global__ void __launch_bounds__(256) bb_alpha_kernel(BBArgs b, size_t j0, size_t j1) {
    const size_t j = j0 + (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    double num = 0.0, den = 0.0;
    if (j < j1) {
        const float xj = b.xbar[j], gj = b.gbar[j];
        if (b.mask[j]) {
            const double sq = (double)xj - (double)b.xprev[j];
            num = ((double)gj - (double)b.gprev[j]) * sq;
            den = (double)b.dl[j] * sq * sq;
        }
        b.xprev[j] = xj;
        b.gprev[j] = gj;
        b.gbar[j] = 0.0f;
        b.xbar[j] = 0.0f;
    }
    block_sum_store<256>(num, &b.part[2 * blockIdx.x]);
    __syncthreads();   // block_sum_store's shared scratch is reused
    block_sum_store<256>(den, &b.part[2 * blockIdx.x + 1]);
    __shared__ int last;
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned prev = atomicAdd(&b.sc->arrive_bb, 1u);
        last = (prev == gridDim.x - 1u);
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        double sn = 0.0, sd = 0.0;
        for (unsigned q = 0; q < gridDim.x; q++) {
            sn += __ldcg(&b.part[2 * q]);
            sd += __ldcg(&b.part[2 * q + 1]);
        }
        b.sc->arrive_bb = 0;
        if (b.out2) {
            b.out2[0] = sn;
            b.out2[1] = sd;
        } else {
            bb_rule(b.sc, sn, sd, b.alpha_min);
        }
    }
}

__global__ void bb_rule_kernel(Scalars* sc, const double* sums2, double alpha_min) {
    bb_rule(sc, sums2[0], sums2[1], alpha_min);
}

// K4 on the all-reduced xi (one block)
__global__ void __launch_bounds__(256) xi_rule_kernel(GupdArgs ga, const double* xi_glob) {
    xi_finalize_block<256>(xi_glob, 1, ga);
}

// ---------------------------------------------------------------------------
// K4: xi = fixed-order fp64 sum of block partials; restart rule; rho_l
// ---------------------------------------------------------------------------
__global__ void init_scalars_kernel(Scalars* sc, double rho0) {
    sc->rho = rho0;
    sc->l = 0;
    sc->step = 0;
    sc->arrive = 0;
    sc->alpha = 1.0;
    sc->kiter = 0;
    sc->arrive_bb = 0;
}

// ---------------------------------------------------------------------------
// Setup helpers
// ---------------------------------------------------------------------------
__global__ void mask_to_float_kernel(const uint8_t* __restrict__ m, float* __restrict__ f, size_t N) {
    size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < N) f[j] = m[j] ? 1.0f : 0.0f;
}

__global__ void mask_finalize_kernel(uint8_t* __restrict__ m, float* __restrict__ dl, size_t N) {
    size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < N) {
        bool in = m[j] && dl[j] > 0.0f;
        m[j] = in ? 1 : 0;
        if (!in) dl[j] = 0.0f;
    }
}

__global__ void zero_offmask_kernel(float* __restrict__ x, const uint8_t* __restrict__ m, size_t N) {
    size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < N && !m[j]) x[j] = 0.0f;
}

// U count (fp64 geometry): thread per (view, column), loop over z.
struct DevGeomD {
    int kind, nx, ny, nz, ns, nt;
    double dx, dy, dz, x0, y0, z0, dso, dsd, ds, dt, offs, offt;
    double s_lo, s_hi, t_lo, t_hi;
    const double2* vz;  // per view: (beta, z_s)
};

__global__ void __launch_bounds__(256) count_vv_kernel(DevGeomD g, int first, int stride, int count,
                                                      const uint8_t* __restrict__ m,
                                                      unsigned long long* __restrict__ total) {
    size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    size_t ncol = (size_t)g.nx * g.ny;
    unsigned long long cu = 0, cn = 0, cc = 0;
    if (idx < ncol * (size_t)count) {
        int k = (int)(idx / ncol);
        size_t col = idx % ncol;
        int ix = (int)(col % g.nx), iy = (int)(col / g.nx);
        double2 vz = g.vz[first + k * stride];
        double sb = sin(vz.x), cb = cos(vz.x);
        double xc = g.x0 + ix * g.dx, yc = g.y0 + iy * g.dy;
        double tmin = 1e300, tmax = -1e300;
        for (int q = 0; q < 4; q++) {
            double px = xc + ((q & 1) ? 0.5 : -0.5) * g.dx, py = yc + ((q & 2) ? 0.5 : -0.5) * g.dy;
            double along = g.dso + px * sb - py * cb, perp = px * cb + py * sb;
            double t = g.dsd * atan2(perp, along);
            tmin = fmin(tmin, t);
            tmax = fmax(tmax, t);
        }
        double a = fmax(tmin, g.s_lo), b = fmin(tmax, g.s_hi);
        if (b > a) {
            // channels whose bin overlaps (a, b) with positive length
            double cbase = -(g.ns - 1) / 2.0 - g.offs;
            long long c0 = (long long)floor(a / g.ds - cbase + 0.5), c1 = (long long)ceil(b / g.ds - cbase - 0.5);
            long long nch = c1 - c0 + 1;
            double along = g.dso + xc * sb - yc * cb, perp = xc * cb + yc * sb;
            double rho = sqrt(along * along + perp * perp), mag = g.dsd / rho;
            bool any = false;
            for (int iz = 0; iz < g.nz; iz++) {
                if (!m[col * g.nz + iz]) continue;
                long long nrow = 1;
                if (g.kind != 0) {
                    double zj = g.z0 + iz * g.dz;
                    double tm = (zj - 0.5 * g.dz - vz.y) * mag, tp = (zj + 0.5 * g.dz - vz.y) * mag;
                    double ta = fmax(tm, g.t_lo), tb = fmin(tp, g.t_hi);
                    if (!(tb > ta)) continue;
                    double rbase = -(g.nt - 1) / 2.0 - g.offt;
                    long long r0 = (long long)floor(ta / g.dt - rbase + 0.5), r1 = (long long)ceil(tb / g.dt - rbase - 0.5);
                    nrow = r1 - r0 + 1;
                }
                cu++;
                cn += (unsigned long long)(nch * nrow);
                any = true;
            }
            cc += any ? 1 : 0;
        }
    }
    // warp reduce then integer atomics (exact, order-independent)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        cu += __shfl_down_sync(0xffffffffu, cu, o);
        cn += __shfl_down_sync(0xffffffffu, cn, o);
        cc += __shfl_down_sync(0xffffffffu, cc, o);
    }
    if ((threadIdx.x & 31) == 0 && cu) {
        atomicAdd(&total[0], cu);
        atomicAdd(&total[1], cn);
        atomicAdd(&total[2], cc);
    }
}

}  // namespace ct
