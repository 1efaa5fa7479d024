// ct_common.cuh — device-side scan geometry and the ONE separable-footprint
// routine shared by the forward and back projectors (so a_ij is identical in
// A and A').  sm_100a, fp32.
//
// SF-TR footprint with A1 amplitude (reading O2 / G1 of DESIGN.md; "A is
// the system matrix of a CT scan"):
//   a_ij = l_phi * l_theta * F_s(c) * F_t(r)
//   F_s(c): bin average of the trapezoid whose breakpoints are the arc positions
//           of the voxel's four in-plane corners;
//   F_t(r): overlap of the magnified voxel z-extent with detector row r / dt;
//   l_phi = dx / max(|cos phi0|, |sin phi0|), l_theta = sqrt(1 + ((z - z_s)/rho_h)^2).
//
// Precision: the corner breakpoints are evaluated relative to
// the voxel-centre ray (one atan2f per (view, column) plus a small-angle series
// for the corner offsets), in channel units, so fp32 keeps ~1e-5 relative accuracy.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

// Debug build (-DCT_DEBUG_CHECKS=1, tools/debug_checks.sh): device asserts on the invariants the
// kernels rely on without checking them (shared-memory indices in range, the forward tile's
// one-writer-per-address rounds, zero contributions of the back-projector's unpredicated tail
// lanes).  compute-sanitizer is not available on the GPU pool; this is its stand-in.
#ifndef CT_DEBUG_CHECKS
#define CT_DEBUG_CHECKS 0
#endif
#if CT_DEBUG_CHECKS
#undef NDEBUG
#include <cassert>
#define CT_DCHECK(c) assert(c)
#else
#define CT_DCHECK(c) ((void)0)
#endif

namespace ct {

constexpr int kMaxFoot = 8;   // channel window of a voxel footprint (validated at create)

struct DevGeom {
    int kind;                 // 0 fan2d, 1 cone axial, 2 cone helical
    int nx, ny, nz, ns, nt, na;
    float dx, dy, dz;
    float x0, y0;             // centre of voxel (ix=0, iy=0)
    float zb0;                // lower boundary of voxel iz = 0
    float dso, dsd;
    float dsd_ds;             // dsd / ds  (radians -> channel units)
    float cbase;              // channel coordinate of fan angle 0: (ns-1)/2 + offs
    float cedge;              // cbase + 1/2 (rounded once): bin c's left edge is c - cedge (centred units)
    float rbase;              // row coordinate of t = 0: (nt-1)/2 + offt
    float dt;
    float zs0, dzs;           // helical source height z_s(v) = zs0 + v dzs (dzs = 0: axial)
    float zhalf;              // bound on |z - z_s| of any voxel a view can see (mm)
    int fpar, fspan;          // fan 2D forward: lane-parity buffers P and tile channel-span bound
    int vrel;                 // fan 2D: vertex positions relative to a per-block reference ray (1) or absolute (0)
    int lpoly;                // cone, nt <= 64: polynomial l_theta in fwd3d2 / back3d (ltheta_of)
    const float4* views;      // per view: (sin beta, cos beta, qi, qf) with
                              // (z_s - zb0)/dz = qi + qf, qi integer (exact in fp32)
};

// Transaxial footprint of one voxel column for one view (channel units).
struct Trans {
    float cc;       // channel coordinate of the voxel-centre ray
    float t0, t1, t2, t3;   // sorted breakpoints relative to cc (channel units)
    float lphi;     // A1 in-plane amplitude (mm)
    float rho;      // in-plane source-to-centre distance (mm)
};

__device__ __forceinline__ void sort2(float& a, float& b) {
    float lo = fminf(a, b), hi = fmaxf(a, b);
    a = lo;
    b = hi;
}

__device__ __forceinline__ float small_atan(float u) {
    // atan(u) = u - u^3/3 + u^5/5 - ...; |u| = corner half-diagonal / rho_h
    // (< 2e-2 for every validated geometry) -> truncation u^7/7 < 2e-13
    float u2 = u * u;
    return u * (1.0f - u2 * (1.0f / 3.0f - u2 * 0.2f));
}

// atan(u) for any u: odd minimax polynomial on [-1, 1] (max error 1.0e-7 in fp32,
// comparable to atan2f) with the reduction atan(u) = sign(u) pi/2 - atan(1/u).
__device__ __forceinline__ float fast_atan(float u) {
    const float au = fabsf(u);
    const bool big = au > 1.0f;
    const float t = big ? __fdividef(1.0f, au) : au;
    const float t2 = t * t;
    float p = 2.456723016e-03f;
    p = fmaf(p, t2, -1.440135344e-02f);
    p = fmaf(p, t2, 3.978122036e-02f);
    p = fmaf(p, t2, -7.234857604e-02f);
    p = fmaf(p, t2, 1.049894656e-01f);
    p = fmaf(p, t2, -1.416122948e-01f);
    p = fmaf(p, t2, 1.998590685e-01f);
    p = fmaf(p, t2, -3.333259704e-01f);
    p = fmaf(p, t2, 9.999998864e-01f);
    float r = p * t;
    r = big ? 1.57079632679489662f - r : r;
    return copysignf(r, u);
}

__device__ __forceinline__ void transaxial(const DevGeom& g, float sb, float cb, float xc, float yc, Trans& tr) {
    float along = g.dso + xc * sb - yc * cb;     // (p - S) . e_c  (> 0: the image is inside the orbit)
    float perp = xc * cb + yc * sb;              // (p - S) . e_perp
    float rho2 = along * along + perp * perp;
    float rho = sqrtf(rho2);
    tr.rho = rho;
    tr.cc = fast_atan(__fdividef(perp, along)) * g.dsd_ds + g.cbase;
    // corner offsets (+-hx, +-hy).  Opposite corners are negatives of each other,
    // so two "diagonals" (sx, sy) = (+,+) and (+,-) give all four breakpoints:
    //   corner = +-(d_along, d_perp); Delta gamma = atan(cross / dot) relative to the centre ray.
    float hx = 0.5f * g.dx, hy = 0.5f * g.dy;
    float ax = hx * sb, ay = -hy * cb, px = hx * cb, py = hy * sb;
    float t[4];
#pragma unroll
    for (int k = 0; k < 2; k++) {
        float sy = k ? -1.0f : 1.0f;
        float da = ax + sy * ay, dp = px + sy * py;
        float cross = along * dp - perp * da;      // odd in the corner offset
        float lin = along * da + perp * dp;        // odd in the corner offset
        t[2 * k] = small_atan(__fdividef(cross, rho2 + lin)) * g.dsd_ds;
        t[2 * k + 1] = small_atan(__fdividef(-cross, rho2 - lin)) * g.dsd_ds;
    }
    // 5-comparator sorting network
    sort2(t[0], t[1]);
    sort2(t[2], t[3]);
    sort2(t[0], t[2]);
    sort2(t[1], t[3]);
    sort2(t[1], t[2]);
    tr.t0 = t[0]; tr.t1 = t[1]; tr.t2 = t[2]; tr.t3 = t[3];
    float dirx = fabsf(xc + g.dso * sb), diry = fabsf(yc - g.dso * cb);
    tr.lphi = __fdividef(g.dx * rho, fmaxf(dirx, diry));
}

// Antiderivative of the unit trapezoid (branch-free, degenerate widths safe).
struct TrapCdf {
    float t0, t1, t2, h0, h3;
    __device__ __forceinline__ TrapCdf(const Trans& tr) {
        t0 = tr.t0; t1 = tr.t1; t2 = tr.t2;
        h0 = __fdividef(0.5f, fmaxf(tr.t1 - tr.t0, 1e-20f));
        h3 = __fdividef(0.5f, fmaxf(tr.t3 - tr.t2, 1e-20f));
        t3 = tr.t3;
    }
    float t3;
    __device__ __forceinline__ float operator()(float s) const {
        float a = fminf(fmaxf(s, t0), t1) - t0;
        float f = fminf(fmaxf(s, t1), t2) - t1;
        float b = fminf(fmaxf(s, t2), t3) - t2;
        return a * a * h0 + f + b - b * b * h3;
    }
};

// Footprint bins with end information: if the first (last) bin is not clamped by
// the detector edge, its left (right) edge lies outside (t0, t3), so F there is
// exactly 0 (total) and needs no evaluation.
__device__ __forceinline__ void foot_range_ends(const DevGeom& g, const Trans& tr, int& cA, int& n, bool& clampL,
                                                bool& clampR) {
    int a = __float2int_rd(tr.cc + tr.t0 + 0.5f);
    int b = __float2int_rd(tr.cc + tr.t3 + 0.5f);
    clampL = a < 0;
    clampR = b > g.ns - 1;
    a = max(a, 0);
    b = min(b, g.ns - 1);
    cA = a;
    n = b - a + 1;
}

// First channel of the footprint and number of channels (clamped to the detector).
__device__ __forceinline__ void foot_range(const DevGeom& g, const Trans& tr, int& cA, int& n) {
    int a = __float2int_rd(tr.cc + tr.t0 + 0.5f);
    int b = __float2int_rd(tr.cc + tr.t3 + 0.5f);
    a = max(a, 0);
    b = min(b, g.ns - 1);
    cA = a;
    n = b - a + 1;   // may be <= 0 (footprint off the detector)
}

// Weight of channel c: lphi * F_s(c) (bin edges c -+ 0.5 relative to cc).
__device__ __forceinline__ float chan_weight(const TrapCdf& F, float cc, float lphi, int c) {
    float e0 = (float)c - 0.5f - cc;
    return lphi * (F(e0 + 1.0f) - F(e0));
}

// Axial parameters of a column for one view, in voxel-index units q relative to
// the integer qi of the source height (keeps fp32 precision on long helices):
//   q(r) = qf + (r - rbase) * kz is the voxel coordinate (minus qi) of row r's
//   centre; row r spans [q(r) - kz/2, q(r) + kz/2]; F_t = overlap_q / kz.
struct Axial {
    int qi;        // integer part of (z_s - zb0)/dz
    float qf;      // fractional remainder
    float kz;      // dt / (mag * dz),  mag = dsd / rho
    float inv_kz;
    float dz_rho;  // dz / rho  (for l_theta)
};

__device__ __forceinline__ void axial(const DevGeom& g, float4 view, float rho, Axial& ax) {
    ax.qi = (int)view.z;
    ax.qf = view.w;
    ax.kz = g.dt * rho / (g.dsd * g.dz);
    ax.inv_kz = __fdividef(g.dsd * g.dz, g.dt * rho);   // MUFU reciprocal paths (~2 ulp)
    ax.dz_rho = __fdividef(g.dz, rho);
}

__device__ __forceinline__ float sqrt_approx(float v) {
    // MUFU square root (rel. error ~2^-22), ample for l_theta in [1, 1.01]
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
    return r;
}

#ifndef CT_LPOLY
#define CT_LPOLY 1   // 0: never use the polynomial l_theta (ct_geom_create leaves DevGeom::lpoly = 0)
#endif
// l_theta of the production projectors (fwd3d2 / back3d).  LP (DevGeom::lpoly, set at create when
// every tz a projector can meet satisfies |tz| <= kLpolyTzMax): the tables carry dz / rho
// pre-scaled by 1/sqrt(2), so h = tz / sqrt(2) and sqrt(1 + tz^2) ~= 1 + h^2 with relative error
// <= tz^4 / 8 <= 5.2e-6 -- one FFMA instead of FFMA + MUFU on the slice loads' dependency chain.
constexpr float kLpolyTzMax = 0.08f;
template <bool LP>
__host__ __device__ constexpr float lt_scale() { return LP ? 0.70710678118654752f : 1.0f; }
template <bool LP>
__device__ __forceinline__ float ltheta_of(float tz) {
    return LP ? fmaf(tz, tz, 1.0f) : sqrt_approx(fmaf(tz, tz, 1.0f));
}

__device__ __forceinline__ float ltheta(const Axial& ax, int iz) {
    float tz = ((float)(iz - ax.qi) + 0.5f - ax.qf) * ax.dz_rho;
    return sqrt_approx(fmaf(tz, tz, 1.0f));
}

__device__ __forceinline__ float row_center_q(const Axial& ax, const DevGeom& g, int r) {
    return ax.qf + ((float)r - g.rbase) * ax.kz;
}

// F_t(iz, r): overlap of voxel [iz, iz+1] with row r's q-interval, / kz.
__device__ __forceinline__ float axial_weight(const Axial& ax, float qr, int iz) {
    float lo = qr - 0.5f * ax.kz, hi = qr + 0.5f * ax.kz;
    float zi = (float)(iz - ax.qi);
    float ov = fminf(zi + 1.0f, hi) - fmaxf(zi, lo);
    return fmaxf(ov, 0.0f) * ax.inv_kz;
}

// Voxel range [iz0, iz1] overlapping row r (unclamped).
__device__ __forceinline__ void row_voxels(const Axial& ax, float qr, int& iz0, int& iz1) {
    iz0 = __float2int_rd(qr - 0.5f * ax.kz) + ax.qi;
    iz1 = __float2int_rd(qr + 0.5f * ax.kz) + ax.qi;
}

// Row range [r0, r1] overlapping voxel iz (unclamped).
__device__ __forceinline__ void voxel_rows(const Axial& ax, const DevGeom& g, int iz, int& r0, int& r1) {
    float zi = (float)(iz - ax.qi);
    r0 = __float2int_rd((zi - ax.qf) * ax.inv_kz + g.rbase - 0.5f);
    r1 = __float2int_rd((zi + 1.0f - ax.qf) * ax.inv_kz + g.rbase + 0.5f);
}

// Programmatic dependent launch (sm_90+): a kernel launched with the PDL attribute may start
// while its predecessor in the stream is still running; pdl_wait() blocks until that
// predecessor has completed and its writes are visible (so code before it may touch only
// static data: geometry tables, the support mask, shared memory).  pdl_trigger() lets the
// next kernel's blocks be scheduled once every block of this grid has issued it.
// Both are no-ops for a normal launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// The compiler treats read-only (ld.global.nc) loads as invariant and may hoist them above
// griddepcontrol.wait despite its memory clobber.  A pointer to data a predecessor kernel
// writes is passed through pdl_after() after the wait: the loads through the returned
// pointer depend on an opaque asm output that follows the wait (volatile asms keep order).
template <typename T>
__device__ __forceinline__ T* pdl_after(T* p) {
    asm volatile("" : "+l"(p));
    return p;
}
// Loads of data a PDL predecessor writes use coherent ld.global (L1-cached): ld.global.nc
// (__ldg, or what nvcc emits for const __restrict__ pointers) promises the data is read-only
// for the kernel's whole lifetime, which a predecessor still running before the wait breaks,
// and ptxas does hoist .nc loads above griddepcontrol.wait.
__device__ __forceinline__ float ld_dep(const float* p) {
    float v;
    asm("ld.global.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ double ld_dep(const double* p) {
    double v;
    asm("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }

// L2 eviction-priority hints (PTX createpolicy + .L2::cache_hint): a fractional policy with
// fraction 1.0 applies to every access made with it.
__device__ __forceinline__ unsigned long long l2_evict_last() {
    unsigned long long p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ unsigned long long l2_evict_first() {
    unsigned long long p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ float ldg_pol(const float* a, unsigned long long pol) {
    float v;
    asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(a), "l"(pol));
    return v;
}
__device__ __forceinline__ void stg_pol(float* a, float v, unsigned long long pol) {
    asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(a), "f"(v), "l"(pol) : "memory");
}

// Fair potential pieces (reading G3/G14)
#ifndef CT_FAIR_RCP_APPROX
#define CT_FAIR_RCP_APPROX 1
#endif
__device__ __forceinline__ void fair(float t, float inv_delta, float& dpsi, float& omega) {
    const float v = fmaf(fabsf(t), inv_delta, 1.0f);   // >= 1
#if CT_FAIR_RCP_APPROX
    // MUFU reciprocal (max error ~1 ulp on [1, inf)): one instruction instead of the
    // correctly rounded sequence; the 26-neighbour stencil evaluates it 26 times per voxel
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(omega) : "f"(v));
#else
    omega = __frcp_rn(v);
#endif
    dpsi = t * omega;
}

// Branch-free form for the shared-memory stencils: voxels outside S (or outside the grid)
// are stored as +inf, so t = xj - xk = -inf, v = inf, omega = rcp(inf) = +0 (PTX
// rcp.approx: +-inf -> +-0) and dpsi = max(t, -FLT_MAX) omega = -0: an excluded pair adds
// exactly zero, and for an included pair the values are those of fair() (same operations).
// (A/B, c5 K3: the NaN form's per-neighbour branch kept the ADU pipe 68 % busy.)
constexpr unsigned kOffS = 0x7f800000u;   // +inf: not in S
__device__ __forceinline__ void fair_masked(float xj, float xk, float inv_delta, float& dpsi, float& omega) {
    const float t = xj - xk;
    const float v = fmaf(fabsf(t), inv_delta, 1.0f);
#if CT_FAIR_RCP_APPROX
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(omega) : "f"(v));
#else
    omega = __frcp_rn(v);   // correctly rounded: rcp(inf) = +0 as well
#endif
    dpsi = fmaxf(t, -3.40282347e38f) * omega;
}
// Accumulating form: g += psi'(t) = max(t, -FLT_MAX) omega (one FFMA), c += omega.
__device__ __forceinline__ void fair_masked_acc(float xj, float xk, float inv_delta, float& g, float& c) {
    const float t = xj - xk;
    const float v = fmaf(fabsf(t), inv_delta, 1.0f);
    float omega;
#if CT_FAIR_RCP_APPROX
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(omega) : "f"(v));
#else
    omega = __frcp_rn(v);
#endif
    g = fmaf(fmaxf(t, -3.40282347e38f), omega, g);
    c += omega;
}

}  // namespace ct
