// ct_fbp.cuh — FBP / FDK initial image x^0 (NEXT-4; "initialized with a standard
// filtered back-projection (FBP) reconstruction"; reading B-FBP in DESIGN.md).  sm_100a, fp32.
//
// Full-scan equiangular fan-beam FBP with the FDK extension for a cylindrical detector on a
// circular orbit; for helical scans (reading B-FBP-H) the same filtering
// and a back-projection over the views that see the voxel, normalised by their number:
//   f(p) = 2 pi sum_{v seen} Q_v / L^2 / #{v seen}   (projected row inside [0, nt - 1]).
//   R'(gamma_k, t) = R(gamma_k, t) D cos(gamma_k) D / sqrt(D^2 + zeta^2),  zeta = t dso/dsd
//   Q(gamma_n, t)  = tau sum_k R'(gamma_k, t) g((n - k) tau),  g even, zero at even n != 0
//   f(p)           = dbeta sum_v Q_v(gamma(p), t(p)) / L(p)^2     (bilinear in gamma, t)
// One-time setup work (not on the OS-LALM hot path); plain SIMT kernels.
#pragma once
#include "ct_common.cuh"

namespace ct {

// ramp-filter tap g(n tau) for the equiangular fan (Kak & Slaney 3.4.1)
__device__ __forceinline__ float fbp_tap(int n, float tau) {
    if (n == 0) return 1.0f / (8.0f * tau * tau);
    if ((n & 1) == 0) return 0.0f;
    const float s = sinf((float)n * tau);
    return -1.0f / (2.0f * 9.8696044010893586f * s * s);
}

// CTA = (view, detector row): weight the row, convolve with the ramp taps (odd offsets only).
// y is the ABI sinogram [na][ns][nt]; q is [na][nt][ns] (channel fastest).
__global__ void __launch_bounds__(256) fbp_filter_kernel(DevGeom g, const float* __restrict__ y, float* __restrict__ q) {
    extern __shared__ float fsm[];
    const int ns = g.ns, nt = g.nt;
    float* rp = fsm;          // weighted row, ns
    float* gk = fsm + ns;     // taps at odd offsets d = 1, 3, ...: gk[(d - 1) / 2]
    const int v = blockIdx.x, r = blockIdx.y;
    const float tau = 1.0f / g.dsd_ds, D = g.dso;
    const float zeta = g.kind == 0 ? 0.0f : ((float)r - g.rbase) * g.dt * g.dso / g.dsd;
    const float wz = D / sqrtf(D * D + zeta * zeta);
    for (int k = threadIdx.x; k < ns; k += blockDim.x) {
        const float gam = ((float)k - g.cbase) * tau;
        rp[k] = __ldg(&y[((size_t)v * ns + k) * nt + r]) * D * cosf(gam) * wz;
    }
    for (int d = threadIdx.x; d < ns; d += blockDim.x) gk[d] = fbp_tap(2 * d + 1, tau);
    __syncthreads();
    const float g0 = fbp_tap(0, tau);
    for (int n = threadIdx.x; n < ns; n += blockDim.x) {
        float acc = g0 * rp[n];
        for (int i = 0;; i++) {
            const int d = 2 * i + 1;
            if (d > n && n + d >= ns) break;
            const float a = (n - d >= 0) ? rp[n - d] : 0.0f, b = (n + d < ns) ? rp[n + d] : 0.0f;
            acc = fmaf(a + b, gk[i], acc);
        }
        q[((size_t)v * nt + r) * ns + n] = tau * acc;
    }
}

// Thread = voxel (z fastest, as the image layout): dbeta sum_v Q_v(gamma, t) / L^2; helical:
// the views whose source height is within the cone's z reach of the voxel (dg.zhalf), those
// whose projected row lies on the detector counted and averaged.
__global__ void __launch_bounds__(256) fbp_back_kernel(DevGeom g, const float* __restrict__ q, float* __restrict__ x,
                                                      int count) {
    const size_t N = (size_t)g.nx * g.ny * g.nz;
    const size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= N) return;
    const int iz = (int)(j % g.nz);
    const size_t col = j / g.nz;
    const int ix = (int)(col % g.nx), iy = (int)(col / g.nx);
    const float xc = g.x0 + ix * g.dx, yc = g.y0 + iy * g.dy;
    const float zc = g.zb0 + ((float)iz + 0.5f) * g.dz;   // voxel centre (axial: z_s = 0)
    const int ns = g.ns, nt = g.nt;
    const bool helical = g.kind == 2 && g.dzs > 0.0f;
    int v0 = 0, v1 = count;
    if (helical) {   // views whose source height can be within the cone's reach of the voxel
        const float zr = zc - g.zs0;
        v0 = max(0, (int)floorf((zr - g.zhalf) / g.dzs) - 1);
        v1 = min(count, (int)ceilf((zr + g.zhalf) / g.dzs) + 2);
    }
    float acc = 0.0f;
    int seen = 0;
    for (int v = v0; v < v1; v++) {
        const float4 vw = __ldg(&g.views[v]);
        const float sb = vw.x, cb = vw.y;
        const float along = g.dso + xc * sb - yc * cb, perp = xc * cb + yc * sb;
        const float L2 = along * along + perp * perp;
        float ur = 0.0f;
        if (nt > 1) {
            // (z - z_s) / dz from the view table's exact split of the source height
            const float dzr = ((float)iz + 0.5f - vw.z) - vw.w;
            ur = dzr * g.dz * g.dsd / sqrtf(L2) / g.dt + g.rbase;
            if (helical) {
                if (!(ur >= 0.0f && ur <= (float)(nt - 1))) continue;
                seen++;
            }
        }
        const float uc = atan2f(perp, along) * g.dsd_ds + g.cbase;
        const int k0 = __float2int_rd(uc);
        const float fk = uc - (float)k0;
        const float* qv = q + (size_t)v * nt * ns;
        float val;
        if (nt == 1) {
            const float a = (k0 >= 0 && k0 < ns) ? __ldg(&qv[k0]) : 0.0f;
            const float b = (k0 + 1 >= 0 && k0 + 1 < ns) ? __ldg(&qv[k0 + 1]) : 0.0f;
            val = a + fk * (b - a);
        } else {
            const int r0 = __float2int_rd(ur);
            const float fr = ur - (float)r0;
            float s = 0.0f;
#pragma unroll
            for (int bq = 0; bq < 2; bq++) {
                const int r = r0 + bq;
                if (r < 0 || r >= nt) continue;
                const float* qr = qv + (size_t)r * ns;
                const float a = (k0 >= 0 && k0 < ns) ? __ldg(&qr[k0]) : 0.0f;
                const float b = (k0 + 1 >= 0 && k0 + 1 < ns) ? __ldg(&qr[k0 + 1]) : 0.0f;
                s += (bq ? fr : 1.0f - fr) * (a + fk * (b - a));
            }
            val = s;
        }
        acc += val / L2;
    }
    if (helical)
        x[j] = seen ? acc * (6.283185307179586f / (float)seen) : 0.0f;
    else
        x[j] = acc * (6.283185307179586f / (float)count);
}

}  // namespace ct
