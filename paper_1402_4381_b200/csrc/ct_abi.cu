// ct_abi.cu — C ABI of the OS-LALM CT hot path on B200 (sm_100a):
// geometry tables, kernel launches, the OS-LALM inner-step sequence with CUDA
// graph replay, and the NCCL (multi-GPU) exchange.  See include/ct_oslalm.h for
// the contract of every entry point and DESIGN.md for the design.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3 (ranges visible to ncu --nvtx / nsys)

#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "../../include/ct_oslalm.h"
#include "ct_kernels.cuh"
#include "ct_fan2d.cuh"
#include "ct_fbp.cuh"
#include "ct_comm.cuh"

using namespace ct;

#ifndef CT_VREL
#define CT_VREL 1   // fan 2D: vertex positions relative to per-block reference rays (A/B: 0 = absolute)
#endif
#ifndef CT_PDL
#define CT_PDL 1   // programmatic dependent launch of the 2D inner-step kernels (A/B: 0 disables)
#endif
// Launch with the programmatic-stream-serialization attribute (PDL): the kernel's blocks
// may start while the previous kernel in the stream finishes; the kernel synchronises with
// pdl_wait() before it reads the predecessor's output.
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = CT_PDL;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

#ifndef CT_FWD2D_PT
#define CT_FWD2D_PT 1     // compile-time lane-parity buffer count for P = 1, 2
#endif
#ifndef CT_FWD3D_PAIR
#define CT_FWD3D_PAIR 1   // nt <= 64: pair-row forward kernel (fwd3d2_kernel); 0: fwd3d_kernel
#endif
#ifndef CT_FWD3D2_TC
#define CT_FWD3D2_TC 22   // axial scans; A/B (c3): 22 beats 16, 18, 20, 24, 26, 32 by 2-10 %
#endif
#ifndef CT_FWD3D2_MINB
#define CT_FWD3D2_MINB 5
#endif
#ifndef CT_BAND_OVERLAP
#define CT_BAND_OVERLAP 1   // band exchange: send each destination slab's blocks while the next slab is back-projected
#endif
#ifndef CT_FWD3D2_YSPLIT
#define CT_FWD3D2_YSPLIT 0   // 1: OS-LALM projections in two launches over image-row halves (L2 working set; A/B: c5 11.44 -> 11.68, c4 3.34 -> 3.74 ms, off)
#endif
#ifndef CT_FWD3D2_TC_HEL
#define CT_FWD3D2_TC_HEL 26   // helical scans; A/B (c4, c5): 26 (24 warps/SM) beats 22, 32, 40, 48
#endif
#ifndef CT_FWD3D2_NW_HEL
#define CT_FWD3D2_NW_HEL 8    // 3 CTAs of 8 warps (A/B: c5 11.42 -> 11.29, c4 3.35 -> 3.18 ms vs 6 of 4; 12 of 2: slower)
#endif
#ifndef CT_FWD3D2_MINB_HEL
#define CT_FWD3D2_MINB_HEL 3
#endif
#ifndef CT_FWD3D2_NW
#define CT_FWD3D2_NW 4    // warps (row groups) per CTA (8: c3 -1 %, c5 +12 %)
#endif
#ifndef CT_FWD3D_TC
#define CT_FWD3D_TC 24   // channels per 3D forward CTA (A/B: 24 beats 16 and 32 by ~10 %)
#endif

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
static thread_local char g_err[512] = "";
static std::atomic<unsigned long long> g_launches{0};

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

#define CT_CUDA(call)                                                                          \
    do {                                                                                       \
        cudaError_t e_ = (call);                                                               \
        if (e_ != cudaSuccess) return fail(CT_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

#define CT_LAUNCHED(nk)                                                                        \
    do {                                                                                       \
        cudaError_t e_ = cudaGetLastError();                                                   \
        if (e_ != cudaSuccess) return fail(CT_ECUDA, "kernel launch: %s", cudaGetErrorString(e_)); \
        g_launches += (nk);                                                                    \
    } while (0)

// NVTX range over one ABI call (host side; a CUDA-graph replay shows as one range)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

extern "C" const char* ct_last_error(void) { return g_err; }
extern "C" unsigned long long ct_kernel_launches(void) { return g_launches.load(); }
#ifndef CT_SRC_HASH
#define CT_SRC_HASH "unknown"
#endif
extern "C" const char* ct_build_info(void) {
    return "ct_oslalm sm_100a: fwd2d fwd3d back2d back3d (fused g-update + xi/rho finalize) sqs_update reg_grad gupd "
           "count_vv; src=" CT_SRC_HASH;
}

// ---------------------------------------------------------------------------
// NCCL (loaded at run time; torch has already loaded libnccl.so.2)
// ---------------------------------------------------------------------------
struct NcclApi {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                  cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
static NcclApi g_nccl;
static std::mutex g_nccl_mu;

static bool load_nccl() {
    std::lock_guard<std::mutex> lk(g_nccl_mu);
    if (g_nccl.ok) return true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return false;
    g_nccl.GetUniqueId = (decltype(g_nccl.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    g_nccl.CommInitRank = (decltype(g_nccl.CommInitRank))dlsym(h, "ncclCommInitRank");
    g_nccl.AllReduce = (decltype(g_nccl.AllReduce))dlsym(h, "ncclAllReduce");
    g_nccl.ReduceScatter = (decltype(g_nccl.ReduceScatter))dlsym(h, "ncclReduceScatter");
    g_nccl.AllGather = (decltype(g_nccl.AllGather))dlsym(h, "ncclAllGather");
    g_nccl.Send = (decltype(g_nccl.Send))dlsym(h, "ncclSend");
    g_nccl.Recv = (decltype(g_nccl.Recv))dlsym(h, "ncclRecv");
    g_nccl.GroupStart = (decltype(g_nccl.GroupStart))dlsym(h, "ncclGroupStart");
    g_nccl.GroupEnd = (decltype(g_nccl.GroupEnd))dlsym(h, "ncclGroupEnd");
    g_nccl.CommDestroy = (decltype(g_nccl.CommDestroy))dlsym(h, "ncclCommDestroy");
    g_nccl.GetErrorString = (decltype(g_nccl.GetErrorString))dlsym(h, "ncclGetErrorString");
    g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.AllReduce && g_nccl.ReduceScatter &&
                g_nccl.AllGather && g_nccl.Send && g_nccl.Recv && g_nccl.GroupStart && g_nccl.GroupEnd &&
                g_nccl.CommDestroy;
    return g_nccl.ok;
}

static const char* nccl_err(ncclResult_t r) { return g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "error"; }

// One process per GPU: the exchange steps as NCCL calls on the caller's stream.
struct NcclComm : Comm {
    ncclComm_t comm = nullptr;
    char err[256] = "";
    const char* kind() const override { return "nccl"; }
    const char* last_err() const override { return err; }
    ~NcclComm() override {
        if (comm && g_nccl.ok) g_nccl.CommDestroy(comm);
    }
    int rc(ncclResult_t r, const char* what) {
        if (r == ncclSuccess) return 0;
        snprintf(err, sizeof(err), "%s: %s", what, nccl_err(r));
        return -1;
    }
    static ncclDataType_t nt(int dt) { return dt == COMM_F64 ? ncclFloat64 : dt == COMM_F32 ? ncclFloat32 : ncclUint8; }
    int allreduce_sum(const void* send, void* recv, size_t n, int dt, cudaStream_t st) override {
        return rc(g_nccl.AllReduce(send, recv, n, nt(dt), ncclSum, comm, st), "ncclAllReduce");
    }
    int reduce_scatter_sum(const float* send, float* recv, size_t n, cudaStream_t st) override {
        return rc(g_nccl.ReduceScatter(send, recv, n, ncclFloat32, ncclSum, comm, st), "ncclReduceScatter");
    }
    int all_gather(const float* send, float* recv, size_t n, cudaStream_t st) override {
        return rc(g_nccl.AllGather(send, recv, n, ncclFloat32, comm, st), "ncclAllGather");
    }
    int halo(const void* send_lo, const void* send_hi, void* recv_lo, void* recv_hi, size_t n, int dt,
             cudaStream_t st) override {
        ncclResult_t r = g_nccl.GroupStart();
        if (rank > 0) {
            if (r == ncclSuccess) r = g_nccl.Send(send_lo, n, nt(dt), rank - 1, comm, st);
            if (r == ncclSuccess) r = g_nccl.Recv(recv_lo, n, nt(dt), rank - 1, comm, st);
        }
        if (rank < nranks - 1) {
            if (r == ncclSuccess) r = g_nccl.Send(send_hi, n, nt(dt), rank + 1, comm, st);
            if (r == ncclSuccess) r = g_nccl.Recv(recv_hi, n, nt(dt), rank + 1, comm, st);
        }
        ncclResult_t r2 = g_nccl.GroupEnd();
        return rc(r != ncclSuccess ? r : r2, "z-slab halo exchange");
    }
    int alltoallv(const float* const* send, const size_t* scount, float* const* recv, const size_t* rcount,
                  cudaStream_t st) override {
        if (scount[rank] != rcount[rank]) {
            snprintf(err, sizeof(err), "alltoallv: self block %zu != %zu", scount[rank], rcount[rank]);
            return -1;
        }
        if (scount[rank] && cudaMemcpyAsync(recv[rank], send[rank], scount[rank] * 4, cudaMemcpyDeviceToDevice, st) !=
                                cudaSuccess) {
            snprintf(err, sizeof(err), "alltoallv: self copy failed");
            return -1;
        }
        ncclResult_t r = g_nccl.GroupStart();
        for (int q = 0; q < nranks && r == ncclSuccess; q++) {
            if (q == rank) continue;
            if (scount[q]) r = g_nccl.Send(send[q], scount[q], ncclFloat32, q, comm, st);
            if (r == ncclSuccess && rcount[q]) r = g_nccl.Recv(recv[q], rcount[q], ncclFloat32, q, comm, st);
        }
        ncclResult_t r2 = g_nccl.GroupEnd();
        return rc(r != ncclSuccess ? r : r2, "band exchange (grouped send/recv)");
    }
};


// ---------------------------------------------------------------------------
// geometry
// ---------------------------------------------------------------------------
struct ct_geom {
    ct_geom_desc d;
    DevGeom dg;
    DevGeomD dgd;
    float4* d_views = nullptr;
    double2* d_vz = nullptr;
    unsigned long long* acc2d = nullptr;   // fan 2D ct_fwd_proj: [na][ns] 64-bit fixed-point sums (kept zero)
    int rank = 0, nranks = 1;
    Comm* comm = nullptr;    // exchange backend (NcclComm / VirtualComm); owned
    int zslab = 0;   // NEXT-3: this geometry is rank `rank`'s z-slab of the volume (sinogram-domain sums)
    int exchange = CT_EXCHANGE_AUTO;   // row-slab path: full reduce-scatter / all-gather or z-band blocks
    // z-slab ranks: every rank's slab (lower boundary zb0, slices), gathered at ct_comm_init_zslab
    std::vector<float> slab_zb0;
    std::vector<int> slab_nz;
};

static int comm_rc(const ct_geom* g, int rc) {
    return rc ? fail(CT_ENCCL, "%s exchange: %s", g->comm->kind(), g->comm->last_err()) : CT_OK;
}

static int allreduce(const ct_geom* g, float* buf, size_t n, cudaStream_t st) {
    return comm_rc(g, g->comm->allreduce_sum(buf, buf, n, COMM_F32, st));
}

static inline int nz_of(const ct_geom* g) { return g->d.kind == CT_FAN2D ? 1 : g->d.nz; }
static inline int nt_of(const ct_geom* g) { return g->d.kind == CT_FAN2D ? 1 : g->d.nt; }
static inline size_t n_vox(const ct_geom* g) { return (size_t)g->d.nx * g->d.ny * nz_of(g); }
static inline size_t n_cells_view(const ct_geom* g) { return (size_t)g->d.ns * nt_of(g); }

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

extern "C" int ct_geom_create(const ct_geom_desc* d, ct_geom** out) {
    if (!d || !out) return fail(CT_EINVAL, "ct_geom_create: null argument");
    *out = nullptr;
    if (d->kind < CT_FAN2D || d->kind > CT_CONE_HELICAL) return fail(CT_EINVAL, "unknown geometry kind %d", d->kind);
    bool is2d = d->kind == CT_FAN2D;
    int nz = is2d ? 1 : d->nz, nt = is2d ? 1 : d->nt;
    if (d->nx < 1 || d->ny < 1 || nz < 1 || d->ns < 1 || nt < 1 || d->na < 1)
        return fail(CT_EINVAL, "sizes must be positive (nx=%d ny=%d nz=%d ns=%d nt=%d na=%d)", d->nx, d->ny, nz, d->ns,
                    nt, d->na);
    if (!(d->dx > 0 && d->dy > 0 && d->ds > 0 && d->dso > 0 && d->dsd > d->dso) || (!is2d && !(d->dz > 0 && d->dt > 0)))
        return fail(CT_EINVAL, "spacings must be positive and dsd > dso");
    if (fabs(d->dx - d->dy) > 1e-9 * d->dx) return fail(CT_EINVAL, "dx must equal dy (square voxels)");
    if (!is2d && nt > 128) return fail(CT_EUNSUPPORTED, "nt = %d > 128 detector rows", nt);
    if (!is2d && nz > 4096) return fail(CT_EUNSUPPORTED, "nz = %d > 4096 slices", nz);
    if (d->kind == CT_CONE_HELICAL && !(d->pitch > 0)) return fail(CT_EINVAL, "helical geometry needs pitch > 0");
    if ((double)d->nx * d->ny * nz >= 2147483647.0 || (double)d->na * d->ns * nt >= 2147483647.0)
        return fail(CT_EUNSUPPORTED, "image or sinogram has >= 2^31 elements (32-bit kernel indexing)");
    // footprint width bound: voxel half-diagonal magnified at the closest approach
    double hx = 0.5 * (d->nx - 1) * d->dx + fabs(d->offx) + d->dx, hy = 0.5 * (d->ny - 1) * d->dy + fabs(d->offy) + d->dy;
    double rmax = sqrt(hx * hx + hy * hy);
    if (rmax >= d->dso) return fail(CT_EINVAL, "image (radius %.1f mm) reaches the source orbit (dso %.1f)", rmax, d->dso);
    // a footprint of width w channels touches at most ceil(w) + 1 <= kMaxFoot bins
    double wmax = d->dx * sqrt(2.0) * d->dsd / ((d->dso - rmax) * d->ds);
    if (wmax > kMaxFoot - 1)
        return fail(CT_EUNSUPPORTED, "voxel footprint may be %.2f channels wide (> %d)", wmax, kMaxFoot - 1);

    int dg_fpar = 1, dg_fspan = 1, dg_vrel = 0;
    if (is2d) {
        // fwd2d_tile_kernel: (1) lanes l and l + P must hit different first channels: a pixel
        // step along the warp's line moves the footprint by >= dx sin(pi/4 - delta) mag_min / ds
        // channels (delta = ray-direction spread over a tile); (2) the tile's channel span.
        double tdiag = kF2T * sqrt(2.0) * d->dx;
        double delta = asin(std::min(0.999, 0.5 * tdiag / (d->dso - rmax)));
        double shift = d->dx * sin(M_PI / 4 - delta) * d->dsd / ((d->dso + rmax) * d->ds);
        int P = (int)ceil(1.02 / std::max(shift, 1e-9));
        // unclipped tile span + the kMaxFoot bins a lane may address past its footprint
        int span = (int)ceil(tdiag * d->dsd / ((d->dso - rmax) * d->ds)) + 3 + kMaxFoot;
        if (!(shift > 0) || P > 8 || (size_t)8 * P * span * 4 > 160 * 1024)
            return fail(CT_EUNSUPPORTED, "fan-beam forward tiles: pixel step %.3f channels (P = %d), span %d", shift, P,
                        span);
        dg_fpar = P;
        dg_fspan = span;
        // relative vertex positions: |cross/dot| <= tan(asin(|offset| / distance)) over the kVB-vertex
        // block grid (offsets up to kVB/2 sqrt(2) pixels from the block's reference vertex; the
        // tiles' reference tables reach one block past the image)
        const double bx = 0.5 * 32.0 * ceil(d->nx / 32.0) * d->dx + fabs(d->offx) + 2.0 * kVB * d->dx;
        const double by = 0.5 * 32.0 * ceil(d->ny / 32.0) * d->dy + fabs(d->offy) + 2.0 * kVB * d->dy;
        const double dist = d->dso - sqrt(bx * bx + by * by);
        const double off = 0.5 * kVB * sqrt(2.0) * d->dx;
        dg_vrel = (dist > off && tan(asin(off / dist)) <= 0.1) ? 1 : 0;
    }
    int dev = d->device;
    DeviceGuard guard(dev);
    ct_geom* g = new ct_geom();
    g->d = *d;
    g->d.nz = nz;
    g->d.nt = nt;
    DevGeom& dg = g->dg;
    dg.kind = d->kind;
    dg.nx = d->nx; dg.ny = d->ny; dg.nz = nz; dg.ns = d->ns; dg.nt = nt; dg.na = d->na;
    dg.dx = (float)d->dx; dg.dy = (float)d->dy; dg.dz = is2d ? 1.0f : (float)d->dz;
    dg.x0 = (float)(-(d->nx - 1) / 2.0 * d->dx + d->offx);
    dg.y0 = (float)(-(d->ny - 1) / 2.0 * d->dy + d->offy);
    double z0 = is2d ? 0.0 : (-(nz - 1) / 2.0 * d->dz + d->offz);
    double zb0 = is2d ? -0.5 : z0 - 0.5 * d->dz;
    dg.zb0 = (float)zb0;
    dg.dso = (float)d->dso; dg.dsd = (float)d->dsd;
    dg.dsd_ds = (float)(d->dsd / d->ds);
    dg.cbase = (float)((d->ns - 1) / 2.0 + d->offs);
    dg.cedge = (float)((d->ns - 1) / 2.0 + d->offs + 0.5);
    dg.rbase = (float)((nt - 1) / 2.0 + d->offt);
    dg.dt = is2d ? 1.0f : (float)d->dt;
    {
        // helical: z_s(v) = zs0 + v * dzs; the largest z half-coverage of the detector
        // (at the smallest magnification, rho_max = dso + rmax) bounds the views a z-chunk needs
        double turns_ = d->orbit_deg / 360.0;
        double h_ = d->kind == CT_CONE_HELICAL ? d->pitch * nt * d->dt * d->dso / d->dsd : 0.0;
        double dzs = d->kind == CT_CONE_HELICAL ? h_ / (d->na / turns_) : 0.0;
        dg.zs0 = (float)(-(d->na - 1) / 2.0 * dzs);
        dg.dzs = (float)dzs;
        dg.zhalf = (float)((0.5 * nt * (is2d ? 1.0 : d->dt) + 0.5 * fabs(d->offt) * (is2d ? 1.0 : d->dt)) *
                           (d->dso + rmax) / d->dsd + (is2d ? 0.0 : d->dz));
    }

    std::vector<float4> hv(d->na);
    std::vector<double2> hvz(d->na);
    double turns = d->orbit_deg / 360.0;
    double h = d->kind == CT_CONE_HELICAL ? d->pitch * nt * d->dt * d->dso / d->dsd : 0.0;
    for (int v = 0; v < d->na; v++) {
        double beta = d->orbit_start_deg * M_PI / 180.0 + 2.0 * M_PI * turns * v / d->na;
        double zs = d->kind == CT_CONE_HELICAL ? (v - (d->na - 1) / 2.0) * h / (d->na / turns) : 0.0;
        double q = is2d ? 0.0 : (zs - zb0) / d->dz;
        double qi = floor(q);
        hv[v] = make_float4((float)sin(beta), (float)cos(beta), (float)qi, (float)(q - qi));
        hvz[v] = make_double2(beta, zs);
    }
    DevGeomD& gd = g->dgd;
    gd.kind = d->kind; gd.nx = d->nx; gd.ny = d->ny; gd.nz = nz; gd.ns = d->ns; gd.nt = nt;
    gd.dx = d->dx; gd.dy = d->dy; gd.dz = is2d ? 1.0 : d->dz;
    gd.x0 = -(d->nx - 1) / 2.0 * d->dx + d->offx;
    gd.y0 = -(d->ny - 1) / 2.0 * d->dy + d->offy;
    gd.z0 = z0;
    gd.dso = d->dso; gd.dsd = d->dsd; gd.ds = d->ds; gd.dt = is2d ? 1.0 : d->dt; gd.offs = d->offs; gd.offt = d->offt;
    gd.s_lo = (0 - (d->ns - 1) / 2.0 - d->offs) * d->ds - 0.5 * d->ds;
    gd.s_hi = ((d->ns - 1) - (d->ns - 1) / 2.0 - d->offs) * d->ds + 0.5 * d->ds;
    gd.t_lo = (0 - (nt - 1) / 2.0 - d->offt) * gd.dt - 0.5 * gd.dt;
    gd.t_hi = ((nt - 1) - (nt - 1) / 2.0 - d->offt) * gd.dt + 0.5 * gd.dt;

    cudaError_t e = cudaMalloc(&g->d_views, sizeof(float4) * d->na);
    if (e == cudaSuccess) e = cudaMalloc(&g->d_vz, sizeof(double2) * d->na);
    if (e == cudaSuccess) e = cudaMemcpy(g->d_views, hv.data(), sizeof(float4) * d->na, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(g->d_vz, hvz.data(), sizeof(double2) * d->na, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && is2d) e = cudaMalloc(&g->acc2d, sizeof(unsigned long long) * d->na * d->ns);
    if (e == cudaSuccess && is2d) e = cudaMemset(g->acc2d, 0, sizeof(unsigned long long) * d->na * d->ns);
    if (e != cudaSuccess) {
        cudaFree(g->d_views);
        cudaFree(g->d_vz);
        cudaFree(g->acc2d);
        delete g;
        return fail(e == cudaErrorMemoryAllocation ? CT_ENOMEM : CT_ECUDA, "geometry tables: %s", cudaGetErrorString(e));
    }
    dg.views = g->d_views;
    dg.fpar = dg_fpar;
    dg.fspan = dg_fspan;
    dg.vrel = CT_VREL ? dg_vrel : 0;
    {
        // polynomial l_theta (ltheta_of) where every tz = (z - z_s) / rho a fwd3d2 / back3d pair can
        // weight is small: |z - z_s| <= (row extent) rho / dsd + one slice, rho >= dso - rmax
        const double rb = (nt - 1) / 2.0 + (is2d ? 0.0 : d->offt);
        const double rowmax = std::max(fabs(-0.5 - rb), fabs(nt - 0.5 - rb));
        const double tzmax = is2d ? 1.0 : rowmax * d->dt / d->dsd + d->dz / (d->dso - rmax);
        dg.lpoly = (CT_LPOLY && CT_FWD3D_PAIR && !is2d && nt <= 64 && tzmax <= (double)kLpolyTzMax) ? 1 : 0;
    }
    gd.vz = g->d_vz;
    *out = g;
    return CT_OK;
}

extern "C" void ct_geom_destroy(ct_geom* g) {
    if (!g) return;
    DeviceGuard guard(g->d.device);
    delete g->comm;
    cudaFree(g->d_views);
    cudaFree(g->d_vz);
    cudaFree(g->acc2d);
    delete g;
}

static int check_views(const ct_geom* g, ct_views v) {
    if (v.count < 0 || v.stride < 1 || v.first < 0) return fail(CT_EINVAL, "bad view list {%d,%d,%d}", v.first, v.stride, v.count);
    if (v.count > 0 && (long long)v.first + (long long)(v.count - 1) * v.stride >= g->d.na)
        return fail(CT_EINVAL, "view list {%d,%d,%d} exceeds na=%d", v.first, v.stride, v.count, g->d.na);
    return CT_OK;
}

// ---------------------------------------------------------------------------
// launch helpers
// ---------------------------------------------------------------------------
// Dynamic shared memory above 48 KB must be opted into per kernel and per device: remember
// the largest size set for each (kernel, device) pair (calls may come from several threads
// and devices of one process).
static cudaError_t ensure_dyn_smem(const void* func, size_t bytes) {
    if (bytes <= 48 * 1024) return cudaSuccess;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> done;
    std::lock_guard<std::mutex> lk(mu);
    size_t& have = done[{func, dev}];
    if (have >= bytes) return cudaSuccess;
    e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) have = bytes;
    return e;
}

template <int TC, int NTP, bool RESID>
static cudaError_t launch_fwd3d(const DevGeom& dg, dim3 grid, ct_views v, const float* x, float* out, const float* yobs,
                                const float* w, float scale, const int2* ext, cudaStream_t st) {
    constexpr size_t smem = fwd3d_smem<TC, NTP, 256>();
    cudaError_t e = ensure_dyn_smem((const void*)fwd3d_kernel<TC, NTP, 256, RESID>, smem);
    if (e != cudaSuccess) return e;
    fwd3d_kernel<TC, NTP, 256, RESID><<<grid, 256, smem, st>>>(dg, v.first, v.stride, x, out, yobs, w, scale, ext);
    return cudaSuccess;
}

template <int TC, int NW, int H, bool RESID, int MINB, bool LP>
static cudaError_t launch_fwd3d2(const DevGeom& dg, ct_views v, const float* x, float* out, const float* yobs,
                                 const float* w, float scale, const int2* ext, cudaStream_t st, float* part) {
    constexpr size_t smem = fwd3d2_smem<TC, NW>();
    cudaError_t e = ensure_dyn_smem((const void*)fwd3d2_kernel<TC, NW, H, false, MINB, LP>, smem);
    if (e == cudaSuccess) e = ensure_dyn_smem((const void*)fwd3d2_kernel<TC, NW, H, RESID, MINB, LP>, smem);
    if (e != cudaSuccess) return e;
    dim3 grid((dg.ns + TC - 1) / TC, v.count);
    if (part) {   // y-split: rows [0, ny/2) into `part`, then rows [ny/2, ny) + part through the epilogue
        const int yh = dg.ny / 2;
        fwd3d2_kernel<TC, NW, H, false, MINB, LP><<<grid, NW * 32, smem, st>>>(dg, v.first, v.stride, x, part, nullptr,
                                                                          nullptr, 1.0f, ext, 0, yh, nullptr);
        fwd3d2_kernel<TC, NW, H, RESID, MINB, LP><<<grid, NW * 32, smem, st>>>(dg, v.first, v.stride, x, out, yobs, w, scale,
                                                                          ext, yh, dg.ny, part);
        g_launches += 1;
    } else {
        fwd3d2_kernel<TC, NW, H, RESID, MINB, LP><<<grid, NW * 32, smem, st>>>(dg, v.first, v.stride, x, out, yobs, w, scale,
                                                                          ext, 0, dg.ny, nullptr);
    }
    return cudaSuccess;
}

// Pair-row forward (nt <= 64): tile width and resident CTAs per SM by scan kind (A/B, c3-c5)
template <int H, bool RESID, bool LP>
static cudaError_t launch_fwd3d2_kind(const DevGeom& dg, ct_views v, const float* x, float* out, const float* yobs,
                                      const float* w, float scale, const int2* ext, cudaStream_t st, float* part) {
    if (dg.kind == CT_CONE_HELICAL)
        return launch_fwd3d2<CT_FWD3D2_TC_HEL, CT_FWD3D2_NW_HEL, H, RESID, CT_FWD3D2_MINB_HEL, LP>(dg, v, x, out, yobs,
                                                                                                w, scale, ext, st, part);
    return launch_fwd3d2<CT_FWD3D2_TC, CT_FWD3D2_NW, H, RESID, CT_FWD3D2_MINB, LP>(dg, v, x, out, yobs, w, scale, ext,
                                                                                    st, part);
}
template <int H, bool RESID>
static cudaError_t launch_fwd3d2_sel(const DevGeom& dg, ct_views v, const float* x, float* out, const float* yobs,
                                     const float* w, float scale, const int2* ext, cudaStream_t st, float* part) {
    if (dg.lpoly) return launch_fwd3d2_kind<H, RESID, true>(dg, v, x, out, yobs, w, scale, ext, st, part);
    return launch_fwd3d2_kind<H, RESID, false>(dg, v, x, out, yobs, w, scale, ext, st, part);
}

// Per-call forward-projection scratch (owned by the caller of launch_fwd, so concurrent
// projections through one geometry on different streams never share it):
//   acc2d  fan beam: [count][ns] 64-bit fixed-point sums, zero on entry and on exit
//   ext    cone beam: per image line the range of columns with a nonzero voxel (nullptr: no trimming)
struct FwdScratch {
    unsigned long long* acc2d;
    int2* ext;
    float* part = nullptr;   // cone, nt <= 64: first half's sums of the y-split forward (nullptr: no split)
};

template <bool RESID>
static int launch_fwd(const ct_geom* g, ct_views v, const float* x, float* out, const float* yobs, const float* w,
                      float scale, cudaStream_t st, FwdScratch fs) {
    if (v.count == 0) return CT_OK;
    const DevGeom& dg = g->dg;
    if (dg.kind == CT_FAN2D) {
        const size_t smem = sizeof(float) * 8 * dg.fpar * dg.fspan;
        // P = 2 (c1, c2 and most fan geometries) and P = 1 get compile-time instances
        auto kern = dg.vrel ? (dg.fpar == 2 && CT_FWD2D_PT ? fwd2d_tile_kernel<true, 2>
                               : dg.fpar == 1 && CT_FWD2D_PT ? fwd2d_tile_kernel<true, 1> : fwd2d_tile_kernel<true, 0>)
                            : (dg.fpar == 2 && CT_FWD2D_PT ? fwd2d_tile_kernel<false, 2>
                               : dg.fpar == 1 && CT_FWD2D_PT ? fwd2d_tile_kernel<false, 1> : fwd2d_tile_kernel<false, 0>);
        CT_CUDA(ensure_dyn_smem((const void*)kern, smem));
        dim3 grid((dg.nx + kF2T - 1) / kF2T, (dg.ny + kF2T - 1) / kF2T, (v.count + kF2VC - 1) / kF2VC);
        CT_CUDA(launch_pdl(kern, grid, dim3(256), smem, st, dg, v.first, v.stride, v.count, x, fs.acc2d));
        const int cells = v.count * dg.ns;
        cudaError_t fe = launch_pdl(fwd2d_finalize_kernel<RESID>, dim3((cells + 255) / 256), dim3(256), 0, st, dg,
                                    v.first, v.stride, v.count, fs.acc2d, out, yobs, w, scale);
        if (fe != cudaSuccess) {   // the finalize re-zeroes the accumulator: do it here instead
            cudaMemsetAsync(fs.acc2d, 0, sizeof(unsigned long long) * (size_t)cells, st);
            return fail(CT_ECUDA, "fwd2d_finalize launch: %s", cudaGetErrorString(fe));
        }
        CT_LAUNCHED(1);
    } else {
        // per line, the columns holding a nonzero voxel of x (trims the wedge walk)
        const int next = dg.nx + dg.ny;
        if (fs.ext) {
            fwd3d_extent_init<<<(next + 255) / 256, 256, 0, st>>>(fs.ext, next);
            fwd3d_extent_kernel<<<(dg.nx * dg.ny + 7) / 8, 256, 0, st>>>(dg, x, fs.ext);
            CT_LAUNCHED(2);
        }
        constexpr int TC = CT_FWD3D_TC;
        if (v.count > 65535) {   // gridDim.y limit: launch the view list in chunks
            for (int c0 = 0; c0 < v.count; c0 += 65535) {
                const ct_views vc{v.first + c0 * v.stride, v.stride, std::min(65535, v.count - c0)};
                if (int e = launch_fwd<RESID>(g, vc, x, out + (size_t)c0 * dg.ns * dg.nt, yobs, w, scale, st, fs)) return e;
            }
            return CT_OK;
        }
        dim3 grid((dg.ns + TC - 1) / TC, v.count);
        if (dg.nt <= 32 && CT_FWD3D_PAIR)
            CT_CUDA((launch_fwd3d2_sel<2, RESID>(dg, v, x, out, yobs, w, scale, fs.ext, st, fs.part)));
        else if (dg.nt <= 32)
            CT_CUDA((launch_fwd3d<TC, 32, RESID>(dg, grid, v, x, out, yobs, w, scale, fs.ext, st)));
        else if (dg.nt <= 64 && CT_FWD3D_PAIR)
            CT_CUDA((launch_fwd3d2_sel<1, RESID>(dg, v, x, out, yobs, w, scale, fs.ext, st, fs.part)));
        else if (dg.nt <= 64)
            CT_CUDA((launch_fwd3d<TC, 64, RESID>(dg, grid, v, x, out, yobs, w, scale, fs.ext, st)));
        else
            CT_CUDA((launch_fwd3d<TC, 128, RESID>(dg, grid, v, x, out, yobs, w, scale, fs.ext, st)));
    }
    CT_LAUNCHED(1);
    return CT_OK;
}

// 3D back-projection: one warp per whole voxel column with shared-memory accumulators, so
// the work follows each view's active slices (axial and helical scans alike).
static void back_grid(const ct_geom* g, dim3& grid) {
    const DevGeom& dg = g->dg;
    if (dg.kind == CT_FAN2D)
        grid = dim3((dg.nx + 31) / 32, (dg.ny + 7) / 8, 1);
    else
        grid = dim3((dg.nx + 3) / 4, (dg.ny + 1) / 2, 1);
}

static size_t back_nblocks(const ct_geom* g) {
    dim3 gr;
    back_grid(g, gr);
    return (size_t)gr.x * gr.y * gr.z;
}

// rows [row0, row1) of the image (cone beam; row1 < 0: every row)
template <int EPI>
static int launch_back(const ct_geom* g, ct_views v, const float* y, float* x, const GupdArgs& ga, cudaStream_t st,
                       int row0 = 0, int row1 = -1) {
    const DevGeom& dg = g->dg;
    dim3 grid;
    back_grid(g, grid);
    if (row1 < 0) row1 = dg.ny;
    if (dg.kind != CT_FAN2D) grid.y = (unsigned)std::max(1, (row1 - row0 + 1) / 2);
    if (dg.kind == CT_FAN2D)
        if (dg.vrel)
            CT_CUDA(launch_pdl(back2d_kernel<EPI, true>, grid, dim3(256), 0, st, dg, v.first, v.stride, v.count, y, x, ga));
        else
            CT_CUDA(launch_pdl(back2d_kernel<EPI, false>, grid, dim3(256), 0, st, dg, v.first, v.stride, v.count, y, x, ga));
    else {
        const size_t smem = back3d_smem_fixed() + sizeof(float) * 8 * ((size_t)dg.nz + kBackPad);
#define CT_B3_LAUNCH(NTM_, LP_)                                                                               \
    {                                                                                                        \
        CT_CUDA(ensure_dyn_smem((const void*)back3d_kernel<EPI, NTM_, LP_>, smem));                          \
        back3d_kernel<EPI, NTM_, LP_><<<grid, 256, smem, st>>>(dg, v.first, v.stride, v.count, y, x, ga, row0, row1); \
    }
        if (dg.nt == 64 && dg.lpoly) CT_B3_LAUNCH(64, true)
        else if (dg.nt == 64) CT_B3_LAUNCH(64, false)
        else if (dg.nt == 32 && dg.lpoly) CT_B3_LAUNCH(32, true)
        else if (dg.nt == 32) CT_B3_LAUNCH(32, false)
        else if (dg.lpoly) CT_B3_LAUNCH(0, true)
        else CT_B3_LAUNCH(0, false)
#undef CT_B3_LAUNCH
    }
    CT_LAUNCHED(1);
    return CT_OK;
}

static inline unsigned nblk(size_t n) { return (unsigned)((n + 255) / 256); }


// ---------------------------------------------------------------------------
// projections, D_L, regulariser, U
// ---------------------------------------------------------------------------
extern "C" int ct_fwd_proj(const ct_geom* g, ct_views v, const float* x, float* y, void* stream) {
    NvtxRange nvtx_("ct_fwd_proj");
    if (!g || !x || !y) return fail(CT_EINVAL, "ct_fwd_proj: null argument");
    if (int e = check_views(g, v)) return e;
    DeviceGuard guard(g->d.device);
    // cone beam: no column trimming (it needs per-call scratch); fan beam: the geometry's
    // accumulator (FAN2D handles: one stream at a time for ct_fwd_proj, include/ct_oslalm.h)
    return launch_fwd<false>(g, v, x, y, nullptr, nullptr, 1.0f, (cudaStream_t)stream, FwdScratch{g->acc2d, nullptr});
}

extern "C" int ct_back_proj(const ct_geom* g, ct_views v, const float* y, float* x, int accumulate, void* stream) {
    NvtxRange nvtx_("ct_back_proj");
    if (!g || !x || (!y && v.count > 0)) return fail(CT_EINVAL, "ct_back_proj: null argument");
    if (int e = check_views(g, v)) return e;
    DeviceGuard guard(g->d.device);
    GupdArgs ga{};
    if (accumulate) return launch_back<EPI_ACCUM>(g, v, y, x, ga, (cudaStream_t)stream);
    return launch_back<EPI_STORE>(g, v, y, x, ga, (cudaStream_t)stream);
}

// ---------------------------------------------------------------------------
// Diagnostic: L2-resident read bandwidth (the "HBM/L2 gather roofline" denominator of
// SURVEY §8(d); no vendor L2 number is available).  Every thread streams the buffer
// `reps` times with float4 loads (grid-stride), so after the first pass it is L2-resident.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) l2_read_kernel(const float4* __restrict__ a, size_t n4, int reps, float* out) {
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int r = 0; r < reps; r++)
        for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
            const float4 v = __ldcg(&a[i]);
            s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
        }
    if (s.x + s.y + s.z + s.w == 123.456f) out[0] = s.x;   // keeps the loads alive
}

extern "C" int ct_peak_l2_read(int device, size_t bytes, int reps, double* gbs) {
    if (!gbs || bytes < 1024 || reps < 1) return fail(CT_EINVAL, "ct_peak_l2_read: bad arguments");
    DeviceGuard guard(device);
    float4* a = nullptr;
    float* out = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaError_t e = cudaMalloc(&a, bytes);
    if (e == cudaSuccess) e = cudaMalloc(&out, sizeof(float));
    if (e == cudaSuccess) e = cudaMemset(a, 0, bytes);
    if (e == cudaSuccess) e = cudaEventCreate(&e0);
    if (e == cudaSuccess) e = cudaEventCreate(&e1);
    float ms = 0.0f;
    if (e == cudaSuccess) {
        const size_t n4 = bytes / 16;
        const unsigned grid = (unsigned)(sms * 8);
        l2_read_kernel<<<grid, 256>>>(a, n4, 2, out);   // warm: pulls the buffer into L2
        cudaEventRecord(e0);
        l2_read_kernel<<<grid, 256>>>(a, n4, reps, out);
        cudaEventRecord(e1);
        e = cudaEventSynchronize(e1);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
    }
    cudaFree(a);
    cudaFree(out);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (e != cudaSuccess) return fail(CT_ECUDA, "ct_peak_l2_read: %s", cudaGetErrorString(e));
    *gbs = (double)bytes * reps / (ms / 1e3) / 1e9;
    return CT_OK;
}

// FBP / FDK initial image (NEXT-4; reading B-FBP)
static int check_fbp(const ct_geom* g) {
    if (g->d.kind != CT_CONE_HELICAL && fabs(g->d.orbit_deg - 360.0) > 1e-9)
        return fail(CT_EUNSUPPORTED, "ct_fbp of a circular orbit needs one full turn (orbit 360 deg)");
    return CT_OK;
}

extern "C" int ct_fbp_scratch_bytes(const ct_geom* g, size_t* out) {
    if (!g || !out) return fail(CT_EINVAL, "ct_fbp_scratch_bytes: null argument");
    if (int e = check_fbp(g)) return e;
    *out = (size_t)g->d.na * n_cells_view(g) * sizeof(float);
    return CT_OK;
}

extern "C" int ct_fbp(const ct_geom* g, const float* y, float* x, void* scratch, void* stream) {
    NvtxRange nvtx_("ct_fbp");
    if (!g || !y || !x || !scratch) return fail(CT_EINVAL, "ct_fbp: null argument");
    if (int e = check_fbp(g)) return e;
    DeviceGuard guard(g->d.device);
    cudaStream_t st = (cudaStream_t)stream;
    const DevGeom& dg = g->dg;
    float* q = (float*)scratch;
    const size_t smem = sizeof(float) * 2 * dg.ns;
    CT_CUDA(ensure_dyn_smem((const void*)fbp_filter_kernel, smem));
    fbp_filter_kernel<<<dim3(dg.na, dg.nt), 256, smem, st>>>(dg, y, q);
    fbp_back_kernel<<<nblk(n_vox(g)), 256, 0, st>>>(dg, q, x, dg.na);
    CT_LAUNCHED(2);
    return CT_OK;
}

static size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

// Forward-projection scratch for `count` views: fan accumulator [count][ns] (8 B) or cone
// column extents [nx + ny] (8 B).
static size_t fwd_scratch_bytes(const ct_geom* g, int count) {
    return g->d.kind == CT_FAN2D ? align256((size_t)count * g->d.ns * 8) : align256((size_t)(g->d.nx + g->d.ny) * 8);
}

static FwdScratch fwd_scratch_at(const ct_geom* g, void* p) {
    return g->d.kind == CT_FAN2D ? FwdScratch{(unsigned long long*)p, nullptr} : FwdScratch{nullptr, (int2*)p};
}

// ct_sqs_denom scratch: 1_S image | all-view sinogram | forward scratch (all views)
static void sqs_scratch_layout(const ct_geom* g, size_t off[3], size_t* total) {
    off[0] = 0;
    off[1] = align256(n_vox(g) * sizeof(float));
    off[2] = off[1] + align256((size_t)g->d.na * n_cells_view(g) * sizeof(float));
    *total = off[2] + fwd_scratch_bytes(g, g->d.na) + 256;   // + 256: the caller's pointer may be unaligned
}

extern "C" int ct_sqs_denom_scratch_bytes(const ct_geom* g, size_t* out) {
    if (!g || !out) return fail(CT_EINVAL, "ct_sqs_denom_scratch_bytes: null argument");
    size_t off[3];
    sqs_scratch_layout(g, off, out);
    return CT_OK;
}

static void zslab_window(const ct_geom* g, ct_views v, int* k0, int* k1);
static bool use_zwin(const ct_geom* g, int M);
static size_t zwin_floats(const ct_geom* g, int M, int r);
static int zslab_fwd_resid(const ct_geom* g, ct_views v, const float* x, float* out, const float* y, const float* w,
                           float scale, cudaStream_t st, FwdScratch fs, float* zbuf = nullptr);

extern "C" int ct_sqs_denom(const ct_geom* g, const float* w, uint8_t* mask, float* dl, void* scratch, void* stream) {
    NvtxRange nvtx_("ct_sqs_denom");
    if (!g || !w || !mask || !dl || !scratch) return fail(CT_EINVAL, "ct_sqs_denom: null argument");
    DeviceGuard guard(g->d.device);
    cudaStream_t st = (cudaStream_t)stream;
    size_t N = n_vox(g);
    size_t soff[3], stotal;
    sqs_scratch_layout(g, soff, &stotal);
    char* sbase = (char*)(((uintptr_t)scratch + 255) & ~(uintptr_t)255);
    float* one = (float*)(sbase + soff[0]);
    float* sino = (float*)(sbase + soff[1]);
    const FwdScratch fs = fwd_scratch_at(g, sbase + soff[2]);
    if (fs.acc2d) CT_CUDA(cudaMemsetAsync(fs.acc2d, 0, (size_t)g->d.na * g->d.ns * 8, st));
    // multi-rank: this rank's contiguous block of all views, partial D_L summed with NCCL
    int base = g->d.na / g->nranks, extra = g->d.na % g->nranks;
    ct_views all{g->rank * base + std::min(g->rank, extra), 1, base + (g->rank < extra ? 1 : 0)};
    mask_to_float_kernel<<<nblk(N), 256, 0, st>>>(mask, one, N);
    CT_LAUNCHED(1);
    GupdArgs ga{};
    ga.mask = mask;   // D_L is only needed on S (set to 0 elsewhere below)
    if (g->zslab) {
        // z-slab ranks: A 1_S summed over the slabs (every ray), weighted, back onto the slab
        const ct_views va{0, 1, g->d.na};
        if (int e = zslab_fwd_resid(g, va, one, sino, nullptr, w, 1.0f, st, fs)) return e;
        int k0, k1;
        zslab_window(g, va, &k0, &k1);
        if (int e = launch_back<EPI_STORE>(g, ct_views{k0, 1, k1 - k0}, sino + (size_t)k0 * n_cells_view(g), dl, ga, st))
            return e;
    } else {
        if (int e = launch_fwd<true>(g, all, one, sino, nullptr, w, 1.0f, st, fs)) return e;
        if (int e = launch_back<EPI_STORE>(g, all, sino, dl, ga, st)) return e;
        if (g->comm)
            if (int e = allreduce(g, dl, N, st)) return e;
    }
    mask_finalize_kernel<<<nblk(N), 256, 0, st>>>(mask, dl, N);
    CT_LAUNCHED(1);
    return CT_OK;
}

static int reg_launch(const ct_geom* g, const ct_reg* r, const uint8_t* mask, const float* x, float* grad, float* curv,
                      cudaStream_t st) {
    size_t N = n_vox(g);
    float inv_d = (float)(1.0 / r->delta);
    if (r->nbr == 8)
        reg_grad_kernel<8><<<nblk(N), 256, 0, st>>>(g->dg, x, mask, grad, curv, (float)r->beta, inv_d, N);
    else
        reg_grad_kernel<26><<<nblk(N), 256, 0, st>>>(g->dg, x, mask, grad, curv, (float)r->beta, inv_d, N);
    CT_LAUNCHED(1);
    return CT_OK;
}

static int check_reg(const ct_geom* g, const ct_reg* r) {
    if (!r) return fail(CT_EINVAL, "null regulariser");
    if (!(r->nbr == 8 || r->nbr == 26)) return fail(CT_EINVAL, "nbr must be 8 or 26 (got %d)", r->nbr);
    if (r->nbr == 26 && g->d.kind == CT_FAN2D) return fail(CT_EINVAL, "nbr = 26 needs a 3D geometry");
    if (!(r->delta > 0) || !(r->beta >= 0)) return fail(CT_EINVAL, "need delta > 0 and beta >= 0");
    return CT_OK;
}

extern "C" int ct_reg_grad(const ct_geom* g, const ct_reg* r, const uint8_t* mask, const float* x, float* grad,
                           float* curv, void* stream) {
    NvtxRange nvtx_("ct_reg_grad");
    if (!g || !mask || !x || !grad) return fail(CT_EINVAL, "ct_reg_grad: null argument");
    if (int e = check_reg(g, r)) return e;
    DeviceGuard guard(g->d.device);
    return reg_launch(g, r, mask, x, grad, curv, (cudaStream_t)stream);
}

extern "C" int ct_count_vv(const ct_geom* g, ct_views v, const uint8_t* mask, void* scratch, long long* out, void* stream) {
    if (!g || !mask || !scratch || !out) return fail(CT_EINVAL, "ct_count_vv: null argument");
    if (int e = check_views(g, v)) return e;
    DeviceGuard guard(g->d.device);
    cudaStream_t st = (cudaStream_t)stream;
    CT_CUDA(cudaMemsetAsync(scratch, 0, 3 * sizeof(unsigned long long), st));
    size_t n = (size_t)g->d.nx * g->d.ny * v.count;
    if (n) {
        count_vv_kernel<<<nblk(n), 256, 0, st>>>(g->dgd, v.first, v.stride, v.count, mask, (unsigned long long*)scratch);
        CT_LAUNCHED(1);
    }
    unsigned long long h[3] = {0, 0, 0};
    CT_CUDA(cudaMemcpyAsync(h, scratch, sizeof(h), cudaMemcpyDeviceToHost, st));
    CT_CUDA(cudaStreamSynchronize(st));
    for (int i = 0; i < 3; i++) out[i] = (long long)h[i];
    return CT_OK;
}

// ---------------------------------------------------------------------------
// OS-LALM state
// ---------------------------------------------------------------------------
struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    const void* key[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    int curG = -1;
    size_t nodes = 0;
    unsigned long long used = 0;   // replay counter value of the last use (LRU replacement)
};
constexpr int kGraphCache = 4;   // (buffers, G parity) combinations kept instantiated

struct ct_oslalm_state {
    const ct_geom* g;
    ct_oslalm_cfg cfg;
    std::vector<int> order;
    size_t N, sino_elems, nparts;
    float* gs;
    float* Gbuf[2];
    float* xalt;
    float* Gtmp;
    float* sino;
    float* vbuf[2] = {nullptr, nullptr};
    // multi-rank slab path: rank prank of P owns image rows [iy0, iy1), i.e.
    // elements [off0, off0 + S) of every padded image buffer (P * S >= N elements)
    int P = 1, prank = 0, slab = 0, iy0 = 0, iy1 = 0;
    bool has_comm = false;
    size_t S = 0, off0 = 0, Npad = 0;
    float* xp[2] = {nullptr, nullptr};   // full images (all-gathered), ping-pong
    int band = 0;                        // band-limited exchange (helical row slabs)
    cudaStream_t cs = nullptr;           // band exchange: communication stream (overlaps the back-projection)
    cudaEvent_t ev_slab[kMaxBandRanks] = {};
    cudaEvent_t ev_cs = nullptr;
    float* bbuf[4] = {nullptr, nullptr, nullptr, nullptr};   // reduce send / recv, gather send / recv
    double* xi_ex = nullptr;             // [0] this rank's xi, [1] all-reduced xi, [2..3] BB sums
    float* xprev = nullptr;              // BB: xbar of the previous outer iteration
    float* xbar = nullptr;               // BB: mean of the current iteration's inner iterates
    float* gbar = nullptr;               // BB: mean subset gradient of the current iteration
    float* gprev = nullptr;              // BB: ... of the previous iteration
    double* bb_part = nullptr;
    // z-slab ranks (NEXT-3): packed boundary slices sent to / received from the neighbours
    float* zsend[2] = {nullptr, nullptr};
    float* zrecv[2] = {nullptr, nullptr};
    uint8_t* zmask[2] = {nullptr, nullptr};
    int zmask_ready = 0;
    float* zwin = nullptr;               // helical z-slab ranks: the neighbours' window-overlap partials
    double* xi_part;
    FwdScratch fs{nullptr, nullptr};     // this state's forward-projection scratch (own, per state)
    Scalars* sc;
    double* dlog;        // M x 3 doubles (per iteration)
    int curG = 0;
    int initialised = 0;
    int log_slot = -1;
    cudaStream_t cap = nullptr;
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    GraphEntry graphs[kGraphCache];
    unsigned long long replays = 0;
    // diagnostic per-kernel timing
    int timing = 0;
    std::vector<cudaEvent_t> evpool;
    std::vector<std::pair<int, int>> evmarks;   // (class, index of start event)
    double tms[5] = {0, 0, 0, 0, 0};
    long long tcnt[5] = {0, 0, 0, 0, 0};
};

static int tmark(ct_oslalm_state* s, cudaStream_t st) {
    if (!s->timing) return -1;
    size_t i = 0;
    for (auto& m : s->evmarks) i = std::max(i, (size_t)m.second + 2);
    if (s->evpool.size() < i + 2) {
        while (s->evpool.size() < i + 2) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            s->evpool.push_back(e);
        }
    }
    cudaEventRecord(s->evpool[i], st);
    return (int)i;
}

static void tmark_end(ct_oslalm_state* s, cudaStream_t st, int cls, int i0) {
    if (!s->timing || i0 < 0) return;
    cudaEventRecord(s->evpool[i0 + 1], st);
    s->evmarks.push_back({cls, i0});
}

static int tcollect(ct_oslalm_state* s) {
    if (!s->timing || s->evmarks.empty()) return CT_OK;
    CT_CUDA(cudaEventSynchronize(s->evpool[s->evmarks.back().second + 1]));
    for (auto& m : s->evmarks) {
        float ms = 0;
        CT_CUDA(cudaEventElapsedTime(&ms, s->evpool[m.second], s->evpool[m.second + 1]));
        s->tms[m.first] += ms;
        s->tcnt[m.first] += 1;
    }
    s->evmarks.clear();
    return CT_OK;
}

static void bit_reversal(int M, std::vector<int>& order) {
    int bits = 0;
    while ((1 << bits) < M) bits++;
    order.clear();
    for (int i = 0; i < (1 << bits); i++) {
        int r = 0;
        for (int b = 0; b < bits; b++)
            if (i & (1 << b)) r |= 1 << (bits - 1 - b);
        if (r < M) order.push_back(r);
    }
}

static int check_cfg(const ct_geom* g, const ct_oslalm_cfg* c) {
    if (!c) return fail(CT_EINVAL, "null cfg");
    if (c->M < 1 || c->M > g->d.na) return fail(CT_EINVAL, "M = %d must be in [1, na = %d]", c->M, g->d.na);
    if (c->mode != CT_RHO_FIXED && c->mode != CT_RHO_CONTINUATION) return fail(CT_EINVAL, "bad rho mode %d", c->mode);
    if (c->mode == CT_RHO_FIXED && !(c->rho_fixed > 0 && c->rho_fixed <= 1))
        return fail(CT_EINVAL, "rho_fixed must be in (0, 1]");
    if (c->mode == CT_RHO_CONTINUATION && !(c->rho_min > 0 && c->rho_min <= 1))
        return fail(CT_EINVAL, "rho_min must be in (0, 1]");
    if (c->inner != CT_INNER_SQS && c->inner != CT_INNER_FISTA) return fail(CT_EINVAL, "bad inner mode %d", c->inner);
    if (c->inner == CT_INNER_SQS && c->n_inner != 1)
        return fail(CT_EINVAL, "CT_INNER_SQS takes exactly one step (n_inner = %d); use CT_INNER_FISTA", c->n_inner);
    if (c->inner == CT_INNER_FISTA && (c->n_inner < 1 || c->n_inner > 64))
        return fail(CT_EINVAL, "n_inner = %d outside [1, 64]", c->n_inner);
    if (g->zslab && c->inner == CT_INNER_FISTA)
        return fail(CT_EUNSUPPORTED, "z-slab ranks support the SQS inner step only (FISTA passes need halos)");
    if (c->bb != 0 && c->bb != 1) return fail(CT_EINVAL, "bb must be 0 or 1");
    if (c->bb && !(c->alpha_min > 0 && c->alpha_min <= 1)) return fail(CT_EINVAL, "alpha_min must be in (0, 1]");
    return check_reg(g, &c->reg);
}

// Rows per slab for P ranks (the last slab may be short; buffers are padded to P * S).
static void slab_geometry(const ct_geom* g, int P, int rank, int* iy0, int* iy1, size_t* S) {
    int R = (g->d.ny + P - 1) / P;
    *iy0 = std::min(g->d.ny, rank * R);
    *iy1 = std::min(g->d.ny, (rank + 1) * R);
    *S = (size_t)R * g->d.nx * nz_of(g);
}

static bool use_slabs(const ct_geom* g, const ct_oslalm_cfg* c) {
    // FISTA's n stencil passes would need a halo exchange per pass: it keeps the all-reduce path
    return g->comm != nullptr && !g->zslab && c->inner == CT_INNER_SQS;
}

// Band-limited exchange for the row-slab path: helical scans, 2..16 ranks,
// every rank owning at least one image row, unless ct_comm_set_exchange chose FULL.
static bool use_band(const ct_geom* g, const ct_oslalm_cfg* c) {
    if (!use_slabs(g, c) || g->nranks < 2 || g->nranks > kMaxBandRanks) return false;
    if (g->exchange == CT_EXCHANGE_FULL) return false;
    if (g->exchange == CT_EXCHANGE_AUTO && g->d.kind != CT_CONE_HELICAL) return false;
    if (g->d.kind == CT_FAN2D) return false;
    int iy0, iy1;
    size_t S;
    slab_geometry(g, g->nranks, g->nranks - 1, &iy0, &iy1, &S);
    return iy1 > iy0;
}

// y-split forward (two launches over image-row halves) for the OS-LALM state's
// projections of cone scans with nt <= 64 (the pair-row kernel)
static bool use_ysplit(const ct_geom* g) {
    return CT_FWD3D2_YSPLIT && g->d.kind != CT_FAN2D && g->d.nt <= 64 && CT_FWD3D_PAIR && g->d.ny >= 2;
}

static void state_layout(const ct_geom* g, const ct_oslalm_cfg* c, size_t off[20], size_t* total) {
    int iy0, iy1;
    size_t S;
    slab_geometry(g, g->nranks, g->rank, &iy0, &iy1, &S);
    const size_t N = std::max(n_vox(g), (size_t)g->nranks * S);   // padded image length
    int maxcount = (g->d.na + c->M - 1) / c->M;
    size_t sino = (size_t)maxcount * n_cells_view(g);
    size_t nparts = std::max(back_nblocks(g), (size_t)nblk(N));
    size_t o = 0;
    off[0] = o; o += align256(N * 4);       // g
    off[1] = o; o += align256(N * 4);       // G0
    off[2] = o; o += align256(N * 4);       // G1
    off[3] = o; o += align256(N * 4);       // xalt
    off[4] = o; o += align256(N * 4);       // Gtmp (multi-rank)
    off[5] = o; o += align256(sino * 4);    // residual sinogram
    off[6] = o; o += align256(nparts * 8);  // xi partials
    off[7] = o; o += align256(sizeof(Scalars));
    off[8] = o; o += align256((size_t)c->M * 3 * 8);  // device log
    const bool two_v = c->inner == CT_INNER_FISTA && c->n_inner > 1;
    off[9] = o; o += two_v ? 2 * align256(N * 4) : 0;  // FISTA extrapolation points v (ping-pong)
    const bool slab = use_slabs(g, c);
    off[10] = o; o += slab ? 2 * align256(N * 4) : 0;  // slab path: all-gathered full images (ping-pong)
    off[11] = o; o += align256(4 * 8);                 // xi / BB sums exchange
    off[12] = o; o += c->bb ? 4 * align256(N * 4) + align256(2 * 8 * nblk(N)) : 0;   // BB: xbar_prev, gbar, gbar_prev, xbar, partials
    const size_t ncols = (size_t)g->d.nx * g->d.ny;
    off[13] = o; o += g->zslab ? 4 * align256(ncols * 4) + 2 * align256(ncols) : 0;   // z-slab halos
    // forward-projection scratch (fan accumulator for one subset's views; z-slab ranks project
    // whole subsets too; cone column extents)
    off[14] = o; o += fwd_scratch_bytes(g, maxcount);
    off[15] = o; o += use_band(g, c) ? 4 * align256(N * 4) : 0;   // band exchange buffers
    off[16] = o; o += use_ysplit(g) ? align256(sino * 4) : 0;         // y-split forward partial sums
    off[17] = o; o += use_zwin(g, c->M) ? align256(std::max<size_t>(1, zwin_floats(g, c->M, g->rank)) * 4) : 0;   // z-slab windowed exchange
    *total = o;
}

extern "C" int ct_oslalm_state_bytes(const ct_geom* g, const ct_oslalm_cfg* c, size_t* out) {
    if (!g || !out) return fail(CT_EINVAL, "ct_oslalm_state_bytes: null argument");
    if (int e = check_cfg(g, c)) return e;
    size_t off[20];
    state_layout(g, c, off, out);
    return CT_OK;
}

extern "C" int ct_oslalm_state_create(const ct_geom* g, const ct_oslalm_cfg* c, void* ws, size_t bytes,
                                      ct_oslalm_state** out) {
    if (!g || !ws || !out) return fail(CT_EINVAL, "ct_oslalm_state_create: null argument");
    if (int e = check_cfg(g, c)) return e;
    size_t off[20], total;
    state_layout(g, c, off, &total);
    if (bytes < total) return fail(CT_ENOMEM, "workspace of %zu bytes < required %zu", bytes, total);
    if ((uintptr_t)ws & 255) return fail(CT_EINVAL, "workspace must be 256-byte aligned");
    DeviceGuard guard(g->d.device);
    ct_oslalm_state* s = new ct_oslalm_state();
    s->g = g;
    s->cfg = *c;
    bit_reversal(c->M, s->order);
    s->N = n_vox(g);
    s->nparts = std::max(back_nblocks(g), (size_t)nblk(s->N));
    char* b = (char*)ws;
    s->gs = (float*)(b + off[0]);
    s->Gbuf[0] = (float*)(b + off[1]);
    s->Gbuf[1] = (float*)(b + off[2]);
    s->xalt = (float*)(b + off[3]);
    s->Gtmp = (float*)(b + off[4]);
    s->sino = (float*)(b + off[5]);
    s->xi_part = (double*)(b + off[6]);
    s->sc = (Scalars*)(b + off[7]);
    s->dlog = (double*)(b + off[8]);
    s->P = g->nranks;
    s->prank = g->rank;
    slab_geometry(g, s->P, s->prank, &s->iy0, &s->iy1, &s->S);
    s->Npad = std::max(s->N, (size_t)s->P * s->S);
    s->off0 = (size_t)s->prank * s->S;
    s->slab = use_slabs(g, c) ? 1 : 0;
    s->has_comm = g->comm != nullptr;
    if (c->inner == CT_INNER_FISTA && c->n_inner > 1) {
        s->vbuf[0] = (float*)(b + off[9]);
        s->vbuf[1] = (float*)(b + off[9] + align256(s->Npad * 4));
    }
    if (s->slab) {
        s->xp[0] = (float*)(b + off[10]);
        s->xp[1] = (float*)(b + off[10] + align256(s->Npad * 4));
    }
    s->xi_ex = (double*)(b + off[11]);
    s->fs = fwd_scratch_at(g, b + off[14]);
    if (use_ysplit(g)) s->fs.part = (float*)(b + off[16]);
    s->band = use_band(g, c) ? 1 : 0;
    if (s->band)
        for (int i = 0; i < 4; i++) s->bbuf[i] = (float*)(b + off[15] + i * align256(s->Npad * 4));
    if (use_zwin(g, c->M)) s->zwin = (float*)(b + off[17]);
    if (g->zslab) {
        const size_t ncols = (size_t)g->d.nx * g->d.ny, fb = align256(ncols * 4);
        s->zsend[0] = (float*)(b + off[13]);
        s->zsend[1] = (float*)(b + off[13] + fb);
        s->zrecv[0] = (float*)(b + off[13] + 2 * fb);
        s->zrecv[1] = (float*)(b + off[13] + 3 * fb);
        s->zmask[0] = (uint8_t*)(b + off[13] + 4 * fb);
        s->zmask[1] = (uint8_t*)(b + off[13] + 4 * fb + align256(ncols));
    }
    if (c->bb) {
        s->xprev = (float*)(b + off[12]);
        s->gbar = (float*)(b + off[12] + align256(s->Npad * 4));
        s->gprev = (float*)(b + off[12] + 2 * align256(s->Npad * 4));
        s->xbar = (float*)(b + off[12] + 3 * align256(s->Npad * 4));
        s->bb_part = (double*)(b + off[12] + 4 * align256(s->Npad * 4));
    }
    cudaError_t e = cudaStreamCreateWithFlags(&s->cap, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->ev_in, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->ev_out, cudaEventDisableTiming);
    if (e == cudaSuccess && s->band) {
        e = cudaStreamCreateWithFlags(&s->cs, cudaStreamNonBlocking);
        for (int q = 0; q < s->P && e == cudaSuccess; q++) e = cudaEventCreateWithFlags(&s->ev_slab[q], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->ev_cs, cudaEventDisableTiming);
    }
    if (e != cudaSuccess) {
        delete s;
        return fail(CT_ECUDA, "state streams: %s", cudaGetErrorString(e));
    }
    *out = s;
    return CT_OK;
}

extern "C" void ct_oslalm_state_destroy(ct_oslalm_state* s) {
    if (!s) return;
    DeviceGuard guard(s->g->d.device);
    for (auto& ge : s->graphs)
        if (ge.exec) cudaGraphExecDestroy(ge.exec);
    for (auto e : s->evpool) cudaEventDestroy(e);
    if (s->cap) cudaStreamDestroy(s->cap);
    if (s->cs) cudaStreamDestroy(s->cs);
    for (auto e : s->ev_slab)
        if (e) cudaEventDestroy(e);
    if (s->ev_cs) cudaEventDestroy(s->ev_cs);
    if (s->ev_in) cudaEventDestroy(s->ev_in);
    if (s->ev_out) cudaEventDestroy(s->ev_out);
    delete s;
}

extern "C" int ct_oslalm_state_reset(ct_oslalm_state* s) {
    if (!s) return fail(CT_EINVAL, "ct_oslalm_state_reset: null argument");
    s->initialised = 0;
    return CT_OK;
}

extern "C" int ct_oslalm_set_timing(ct_oslalm_state* s, int enable) {
    if (!s) return fail(CT_EINVAL, "ct_oslalm_set_timing: null argument");
    s->timing = enable ? 1 : 0;
    for (int i = 0; i < 5; i++) { s->tms[i] = 0; s->tcnt[i] = 0; }
    s->evmarks.clear();
    return CT_OK;
}

extern "C" int ct_oslalm_get_timing(const ct_oslalm_state* s, double* ms5, long long* cnt5) {
    if (!s || !ms5 || !cnt5) return fail(CT_EINVAL, "ct_oslalm_get_timing: null argument");
    for (int i = 0; i < 5; i++) { ms5[i] = s->tms[i]; cnt5[i] = s->tcnt[i]; }
    return CT_OK;
}

extern "C" int ct_oslalm_state_get(const ct_oslalm_state* s, ct_oslalm_state_view* out) {
    if (!s || !out) return fail(CT_EINVAL, "ct_oslalm_state_get: null argument");
    out->g = s->gs;
    out->G = s->Gbuf[s->curG];
    out->rho = &s->sc->rho;
    out->l = &s->sc->l;
    out->step = &s->sc->step;
    out->initialised = s->initialised;
    out->alpha = &s->sc->alpha;
    return CT_OK;
}

// views of subset m owned by this rank (contiguous block)
static ct_views rank_views(const ct_geom* g, int M, int m) {
    int count = (g->d.na - m + M - 1) / M;
    if (g->zslab) return ct_views{m, M, count};   // z-slab ranks project every view onto their slab
    int base = count / g->nranks, extra = count % g->nranks;
    int k0 = g->rank * base + std::min(g->rank, extra);
    int n = base + (g->rank < extra ? 1 : 0);
    return ct_views{m + k0 * M, M, n};
}

// z-slab ranks (NEXT-3): of views {first + k stride, k < count}, the contiguous range [k0, k1)
// whose cone can reach this rank's slab (helical: |z - z_s| <= zhalf; axial: all views).
// zslab_window_of: the same for rank q's slab (extents gathered at ct_comm_init_zslab).
static void zslab_window_of(const ct_geom* g, ct_views v, double zb0, int nz, int* k0, int* k1) {
    *k0 = 0;
    *k1 = v.count;
    const DevGeom& dg = g->dg;
    if (g->d.kind != CT_CONE_HELICAL || !(dg.dzs > 0.0f) || v.count == 0) return;
    const double zlo = zb0, zhi = zb0 + (double)nz * dg.dz, zh = (double)dg.zhalf + dg.dz;
    const double vlo = (zlo - zh - dg.zs0) / dg.dzs, vhi = (zhi + zh - dg.zs0) / dg.dzs;
    *k0 = std::max(0, (int)floor((vlo - v.first) / v.stride) - 1);
    *k1 = std::min(v.count, (int)ceil((vhi - v.first) / v.stride) + 2);
    if (*k1 < *k0) *k1 = *k0;
}

static void zslab_window(const ct_geom* g, ct_views v, int* k0, int* k1) {
    zslab_window_of(g, v, g->dg.zb0, g->dg.nz, k0, k1);
}

// overlap [o0, o1) of ranks r's and q's windows of views v (v's indices)
static void zwin_overlap_rq(const ct_geom* g, ct_views v, int r, int q, int* o0, int* o1) {
    int a0, a1, b0, b1;
    zslab_window_of(g, v, g->slab_zb0[r], g->slab_nz[r], &a0, &a1);
    zslab_window_of(g, v, g->slab_zb0[q], g->slab_nz[q], &b0, &b1);
    *o0 = std::max(a0, b0);
    *o1 = std::max(*o0, std::min(a1, b1));
}

static void zwin_overlap(const ct_geom* g, ct_views v, int q, int* o0, int* o1) {
    zwin_overlap_rq(g, v, g->rank, q, o0, o1);
}

// floats rank r receives in the windowed exchange for the largest subset of an M-subset state
static size_t zwin_floats(const ct_geom* g, int M, int r) {
    size_t best = 0;
    for (int m = 0; m < M; m++) {
        const ct_views v{m, M, (g->d.na - m + M - 1) / M};
        size_t n = 0;
        for (int q = 0; q < g->nranks; q++) {
            if (q == r) continue;
            int o0, o1;
            zwin_overlap_rq(g, v, r, q, &o0, &o1);
            n += (size_t)(o1 - o0);
        }
        best = std::max(best, n);
    }
    return best * n_cells_view(g);
}

// Windowed sinogram exchange of the helical z-slab path (2..16 ranks): only the views two
// ranks' windows share travel, instead of an all-reduce of the whole subset sinogram.  BAND
// forces it, FULL the all-reduce; AUTO takes it when the busiest rank receives fewer bytes than
// a ring all-reduce moves per rank (2 (P-1)/P of the subset sinogram; c5: P = 2, 4 yes, P = 8
// no — the cone's z reach makes neighbouring windows overlap by most of a subset).  Every rank
// evaluates the same rule on the same slab table, so all ranks agree.
static bool use_zwin(const ct_geom* g, int M) {
    if (!(g->zslab && g->comm && g->d.kind == CT_CONE_HELICAL && g->dg.dzs > 0.0f && g->nranks >= 2 &&
          g->nranks <= kMaxBandRanks && (int)g->slab_nz.size() == g->nranks))
        return false;
    if (g->exchange == CT_EXCHANGE_FULL) return false;
    if (g->exchange == CT_EXCHANGE_BAND) return true;
    size_t busiest = 0;
    for (int r = 0; r < g->nranks; r++) busiest = std::max(busiest, zwin_floats(g, M, r));
    const size_t sub = (size_t)((g->d.na + M - 1) / M) * n_cells_view(g);
    return (double)busiest < 2.0 * (g->nranks - 1) / g->nranks * (double)sub;
}

// Forward projection summed over the z-slab ranks: out[k] = sum_slabs A_slab x_slab for
// views k < v.count (only the rank's view window is projected; other views contribute 0),
// then s <- scale W (s - y) on every ray (y nullable).  With `zbuf` (the state's windowed-exchange
// buffer, use_zwin) only the rank's window is summed (over the ranks sharing each view) and
// finalised; the rays outside it are left unspecified (nothing back-projects them here).
static int zslab_fwd_resid(const ct_geom* g, ct_views v, const float* x, float* out, const float* y, const float* w,
                           float scale, cudaStream_t st, FwdScratch fs, float* zbuf) {
    const size_t cells = n_cells_view(g);
    int k0, k1;
    zslab_window(g, v, &k0, &k1);
    if (k0 > 0) CT_CUDA(cudaMemsetAsync(out, 0, (size_t)k0 * cells * 4, st));
    if (k1 < v.count) CT_CUDA(cudaMemsetAsync(out + (size_t)k1 * cells, 0, (size_t)(v.count - k1) * cells * 4, st));
    if (k1 > k0)
        if (int e = launch_fwd<false>(g, ct_views{v.first + k0 * v.stride, v.stride, k1 - k0}, x, out + (size_t)k0 * cells,
                                      nullptr, nullptr, 1.0f, st, fs))
            return e;
    if (zbuf) {
        // neighbours' partials of the shared views in, rank-order sum + residual on the window
        const int P = g->nranks, p = g->rank;
        const float* sptr[kMaxBandRanks];
        float* rptr[kMaxBandRanks];
        size_t sc[kMaxBandRanks], rc[kMaxBandRanks], ro = 0;
        ZWinSet zs{};
        zs.P = P;
        zs.self = p;
        for (int q = 0; q < P; q++) {
            int o0, o1;
            zwin_overlap(g, v, q, &o0, &o1);
            const size_t n = q == p ? 0 : (size_t)(o1 - o0) * cells;
            sc[q] = rc[q] = n;
            sptr[q] = out + (size_t)o0 * cells;
            rptr[q] = zbuf + ro;
            zs.buf[q] = zbuf + ro;
            zs.o0[q] = o0 - k0;   // window-relative
            zs.o1[q] = o1 - k0;
            ro += n;
        }
        if (int e = comm_rc(g, g->comm->alltoallv(sptr, sc, rptr, rc, st))) return e;
        if (k1 > k0) {
            const size_t n = (size_t)(k1 - k0) * cells;
            zwin_sum_resid_kernel<<<(unsigned)std::min<size_t>((n + 255) / 256, 148 * 16), 256, 0, st>>>(out + (size_t)k0 * cells, y, w, v.first + k0 * v.stride,
                                                               v.stride, k1 - k0, (int)cells, scale, zs);
            CT_LAUNCHED(1);
        }
        return CT_OK;   // views outside the window: not back-projected onto this slab (zero footprint)
    }
    if (int e = allreduce(g, out, (size_t)v.count * cells, st)) return e;
    const size_t n = (size_t)v.count * cells;
    resid_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(out, y, w, v.first, v.stride, v.count, (int)cells, scale);
    CT_LAUNCHED(1);
    return CT_OK;
}

// Boundary slices to / from the neighbouring z-slab ranks (rank - 1 below, rank + 1 above).
template <class T>
static int zslab_halo(const ct_geom* g, const T* x, T* send_lo, T* send_hi, T* recv_lo, T* recv_hi, cudaStream_t st) {
    const int ncols = g->d.nx * g->d.ny, nz = g->d.nz;
    zslice_pack_kernel<T><<<(ncols + 255) / 256, 256, 0, st>>>(x, nz, 0, send_lo, ncols);
    zslice_pack_kernel<T><<<(ncols + 255) / 256, 256, 0, st>>>(x, nz, nz - 1, send_hi, ncols);
    CT_LAUNCHED(2);
    return comm_rc(g, g->comm->halo(send_lo, send_hi, recv_lo, recv_hi, (size_t)ncols,
                                    sizeof(T) == 1 ? COMM_U8 : COMM_F32, st));
}


// Slices [b0, b1) in which rank q's partial back-projection of subset m can be non-zero, and
// which its forward projection of subset m reads: the source heights of its contiguous view
// block widened by the cone's z reach (dg.zhalf, a bound over every voxel) and one slice.
static void rank_band(const ct_geom* g, int M, int m, int q, int* b0, int* b1) {
    const DevGeom& dg = g->dg;
    const int count = (g->d.na - m + M - 1) / M;
    const int base = count / g->nranks, extra = count % g->nranks;
    const int k0 = q * base + std::min(q, extra), n = base + (q < extra ? 1 : 0);
    if (n <= 0) {
        *b0 = *b1 = 0;
        return;
    }
    const double za = (double)dg.zs0 + (double)(m + k0 * M) * dg.dzs, zb = (double)dg.zs0 + (double)(m + (k0 + n - 1) * M) * dg.dzs;
    const double zh = (double)dg.zhalf + dg.dz;
    *b0 = std::max(0, (int)floor((std::min(za, zb) - zh - dg.zb0) / dg.dz) - 1);
    *b1 = std::min(g->d.nz, (int)ceil((std::max(za, zb) + zh - dg.zb0) / dg.dz) + 1);
    if (*b1 < *b0) *b1 = *b0;
}

static void rank_rows(const ct_geom* g, int q, int* iy0, int* rows) {
    int a, b;
    size_t S;
    slab_geometry(g, g->nranks, q, &a, &b, &S);
    *iy0 = a;
    *rows = b - a;
}

static unsigned band_grid(size_t n) { return (unsigned)std::min<size_t>((n + 255) / 256, 148 * 16); }

// G+ slab of this rank (rows [iy0, iy1), all slices) = sum over ranks of their partial
// back-projections Gpart, exchanging only the z-band blocks (replaces the reduce-scatter).
static int band_reduce(ct_oslalm_state* s, int m, const float* Gpart, float* Gnew, cudaStream_t st) {
    const ct_geom* g = s->g;
    const int P = s->P, p = s->prank, nx = g->d.nx, nz = g->d.nz;
    int b0[kMaxBandRanks], b1[kMaxBandRanks], ry[kMaxBandRanks], rn[kMaxBandRanks];
    for (int q = 0; q < P; q++) {
        rank_band(g, s->cfg.M, m, q, &b0[q], &b1[q]);
        rank_rows(g, q, &ry[q], &rn[q]);
    }
    const float* sptr[kMaxBandRanks];
    float* rptr[kMaxBandRanks];
    size_t sc[kMaxBandRanks], rc[kMaxBandRanks];
    size_t so = 0, ro = 0;
    BandSet bs{};
    bs.P = P;
    const int bl = b1[p] - b0[p];
    for (int q = 0; q < P; q++) {
        // to q: q's rows of my partial, my band
        sc[q] = q == p ? 0 : (size_t)rn[q] * nx * bl;
        sptr[q] = s->bbuf[0] + so;
        if (sc[q]) {
            band_pack_kernel<<<band_grid(sc[q]), 256, 0, st>>>(Gpart, s->bbuf[0] + so, ry[q], rn[q], nx, nz, b0[p], bl);
            CT_LAUNCHED(1);
        }
        so += sc[q];
        // from q: my rows of q's partial, q's band (my own block packed locally)
        const size_t n = (size_t)rn[p] * nx * (b1[q] - b0[q]);
        rc[q] = q == p ? 0 : n;
        rptr[q] = s->bbuf[1] + ro;
        if (q == p && n) {
            band_pack_kernel<<<band_grid(n), 256, 0, st>>>(Gpart, s->bbuf[1] + ro, ry[p], rn[p], nx, nz, b0[p], bl);
            CT_LAUNCHED(1);
        }
        bs.buf[q] = s->bbuf[1] + ro;
        bs.b0[q] = b0[q];
        bs.b1[q] = b1[q];
        ro += n;
    }
    if (int e = comm_rc(g, g->comm->alltoallv(sptr, sc, rptr, rc, st))) return e;
    band_sum_kernel<<<band_grid((size_t)rn[p] * nx * nz), 256, 0, st>>>(Gnew, ry[p], rn[p], nx, nz, bs);
    CT_LAUNCHED(1);
    return CT_OK;
}

// Overlapped form of launch_back + band_reduce: the partial back-projection runs one destination
// row slab at a time (slab order 0..P-1 on every rank); after slab t is done, this rank's band
// block of it is packed and sent to rank t on the communication stream while slab t + 1 is
// back-projected (each step t is a grouped exchange in which rank t receives from every other
// rank).  The sum in rank order then follows on the compute stream.
static int band_back_reduce(ct_oslalm_state* s, int m, ct_views v, const float* sino, const GupdArgs& ga, float* Gpart,
                            float* Gnew, cudaStream_t st) {
    const ct_geom* g = s->g;
    const int P = s->P, p = s->prank, nx = g->d.nx, nz = g->d.nz;
    int b0[kMaxBandRanks], b1[kMaxBandRanks], ry[kMaxBandRanks], rn[kMaxBandRanks];
    for (int q = 0; q < P; q++) {
        rank_band(g, s->cfg.M, m, q, &b0[q], &b1[q]);
        rank_rows(g, q, &ry[q], &rn[q]);
    }
    const int bl = b1[p] - b0[p];
    float* rslot[kMaxBandRanks];
    BandSet bs{};
    bs.P = P;
    size_t ro = 0, so = 0;
    for (int q = 0; q < P; q++) {
        rslot[q] = s->bbuf[1] + ro;
        bs.buf[q] = rslot[q];
        bs.b0[q] = b0[q];
        bs.b1[q] = b1[q];
        ro += (size_t)rn[p] * nx * (b1[q] - b0[q]);
    }
    CT_CUDA(cudaEventRecord(s->ev_cs, st));
    CT_CUDA(cudaStreamWaitEvent(s->cs, s->ev_cs, 0));   // the communication stream follows st's prior work
    for (int t = 0; t < P; t++) {
        if (int e = launch_back<EPI_STORE>(g, v, sino, Gpart, ga, st, ry[t], ry[t] + rn[t])) return e;
        CT_CUDA(cudaEventRecord(s->ev_slab[t], st));
        CT_CUDA(cudaStreamWaitEvent(s->cs, s->ev_slab[t], 0));
        const size_t n = (size_t)rn[t] * nx * bl;
        float* dst = t == p ? rslot[p] : s->bbuf[0] + so;
        if (n) {
            band_pack_kernel<<<band_grid(n), 256, 0, s->cs>>>(Gpart, dst, ry[t], rn[t], nx, nz, b0[p], bl);
            CT_LAUNCHED(1);
        }
        const float* sptr[kMaxBandRanks];
        float* rptr[kMaxBandRanks];
        size_t sc[kMaxBandRanks], rc[kMaxBandRanks];
        for (int q = 0; q < P; q++) {
            sptr[q] = dst;
            sc[q] = (q == t && p != t) ? n : 0;            // my block of slab t -> rank t
            rptr[q] = rslot[q];
            rc[q] = (p == t && q != t) ? (size_t)rn[p] * nx * (b1[q] - b0[q]) : 0;   // rank t: every block of its slab
        }
        if (int e = comm_rc(g, g->comm->alltoallv(sptr, sc, rptr, rc, s->cs))) return e;
        if (t != p) so += n;
    }
    CT_CUDA(cudaEventRecord(s->ev_cs, s->cs));
    CT_CUDA(cudaStreamWaitEvent(st, s->ev_cs, 0));
    band_sum_kernel<<<band_grid((size_t)rn[p] * nx * nz), 256, 0, st>>>(Gnew, ry[p], rn[p], nx, nz, bs);
    CT_LAUNCHED(1);
    return CT_OK;
}

// After the K3 update of this rank's rows of xb: the neighbours' boundary rows (every slice;
// the next update's stencil) and every other rank's rows inside this rank's band of subset m
// (its next forward projection) -- replaces the all-gather.
static int band_gather(ct_oslalm_state* s, int m, float* xb, cudaStream_t st) {
    const ct_geom* g = s->g;
    const int P = s->P, p = s->prank, nx = g->d.nx, nz = g->d.nz;
    const size_t row = (size_t)nx * nz;
    int b0[kMaxBandRanks], b1[kMaxBandRanks], ry[kMaxBandRanks], rn[kMaxBandRanks];
    for (int q = 0; q < P; q++) {
        rank_band(g, s->cfg.M, m, q, &b0[q], &b1[q]);
        rank_rows(g, q, &ry[q], &rn[q]);
    }
    const int y0 = ry[p], y1 = ry[p] + rn[p];
    if (int e = comm_rc(g, g->comm->halo(xb + (size_t)y0 * row, xb + (size_t)(y1 - 1) * row,
                                         y0 > 0 ? xb + (size_t)(y0 - 1) * row : nullptr,
                                         y1 < g->d.ny ? xb + (size_t)y1 * row : nullptr, row, COMM_F32, st)))
        return e;
    const float* sptr[kMaxBandRanks];
    float* rptr[kMaxBandRanks];
    size_t sc[kMaxBandRanks], rc[kMaxBandRanks];
    size_t so = 0, ro = 0;
    for (int q = 0; q < P; q++) {
        // to q: my rows, q's band
        sc[q] = q == p ? 0 : (size_t)rn[p] * nx * (b1[q] - b0[q]);
        sptr[q] = s->bbuf[2] + so;
        if (sc[q]) {
            band_pack_kernel<<<band_grid(sc[q]), 256, 0, st>>>(xb, s->bbuf[2] + so, ry[p], rn[p], nx, nz, b0[q], b1[q] - b0[q]);
            CT_LAUNCHED(1);
        }
        so += sc[q];
        // from q: q's rows, my band
        rc[q] = q == p ? 0 : (size_t)rn[q] * nx * (b1[p] - b0[p]);
        rptr[q] = s->bbuf[3] + ro;
        ro += rc[q];
    }
    if (int e = comm_rc(g, g->comm->alltoallv(sptr, sc, rptr, rc, st))) return e;
    for (int q = 0; q < P; q++)
        if (rc[q]) {
            band_unpack_kernel<<<band_grid(rc[q]), 256, 0, st>>>(xb, rptr[q], ry[q], rn[q], nx, nz, b0[p], b1[p] - b0[p]);
            CT_LAUNCHED(1);
        }
    return CT_OK;
}

// G+ = M A_m'(W (A_m x - y)) for subset m with the requested epilogue.
static int subset_gradient(ct_oslalm_state* s, const ct_oslalm_data* d, const float* x, int m, int epi, cudaStream_t st) {
    // the fused K4 logs into slot s->log_slot (set by the caller)
    const ct_geom* g = s->g;
    int M = s->cfg.M;
    ct_views v = rank_views(g, M, m);
    int t0 = tmark(s, st);
    if (g->zslab) {
        if (int e = zslab_fwd_resid(g, v, x, s->sino, d->y, d->w, (float)M, st, s->fs, s->zwin)) return e;
    } else {
        if (int e = launch_fwd<true>(g, v, x, s->sino, d->y, d->w, (float)M, st, s->fs)) return e;
    }
    tmark_end(s, st, 1, t0);
    GupdArgs ga{};
    ga.mask = d->mask;
    ga.rho = &s->sc->rho;
    ga.xi_part = s->xi_part;
    ga.gs = s->gs;
    ga.sc = s->sc;
    ga.mode = s->cfg.mode;
    ga.rho_fixed = s->cfg.rho_fixed;
    ga.rho_min = s->cfg.rho_min;
    ga.log3 = s->dlog;
    ga.log_slot = s->log_slot;
    ga.gbar = epi == EPI_GUPD ? s->gbar : nullptr;   // BB: accumulate the iteration's mean subset gradient
    ga.inv_M = 1.0f / (float)M;
    if (g->zslab) {
        // z-slab rank: the back-projection onto the slab is complete (the residual holds every
        // ray), so the fused epilogue runs; only xi is a sum over ranks
        int k0, k1;
        zslab_window(g, v, &k0, &k1);
        const ct_views vw{v.first + k0 * v.stride, v.stride, k1 - k0};
        const float* rsino = s->sino + (size_t)k0 * n_cells_view(g);
        if (epi == EPI_INIT) {
            ga.G_new = s->Gbuf[s->curG];
            return launch_back<EPI_INIT>(g, vw, rsino, nullptr, ga, st);
        }
        ga.G_old = s->Gbuf[s->curG];
        ga.G_new = s->Gbuf[s->curG ^ 1];
        ga.xi_out = s->xi_ex;
        int t1 = tmark(s, st);
        if (int e = launch_back<EPI_GUPD>(g, vw, rsino, nullptr, ga, st)) return e;
        tmark_end(s, st, 2, t1);
        int t2 = tmark(s, st);
        if (int e = comm_rc(g, g->comm->allreduce_sum(s->xi_ex, s->xi_ex + 1, 1, COMM_F64, st))) return e;
        ga.xi_out = nullptr;
        xi_rule_kernel<<<1, 256, 0, st>>>(ga, s->xi_ex + 1);
        CT_LAUNCHED(1);
        tmark_end(s, st, 4, t2);
        return CT_OK;
    }
    if (g->comm == nullptr) {   // single GPU: fused epilogue
        if (epi == EPI_INIT) {
            ga.G_new = s->Gbuf[s->curG];
            return launch_back<EPI_INIT>(g, v, s->sino, nullptr, ga, st);
        }
        ga.G_old = s->Gbuf[s->curG];
        ga.G_new = s->Gbuf[s->curG ^ 1];
        int t1 = tmark(s, st);
        int e = launch_back<EPI_GUPD>(g, v, s->sino, nullptr, ga, st);
        tmark_end(s, st, 2, t1);
        return e;
    }
    if (s->slab) {
        // multi-rank slab path: partial back-projection (this rank's views), reduce-scatter of
        // the padded image into this rank's row slab of G+, slab g-update + xi, all-reduce of
        // the ranks' xi (8 bytes), K4 on every rank
        float* Gnew = s->Gbuf[epi == EPI_INIT ? s->curG : s->curG ^ 1];
        int t1 = tmark(s, st);
        if (s->band && CT_BAND_OVERLAP) {   // per-slab back-projection, blocks sent as each slab completes
            if (int e = band_back_reduce(s, m, v, s->sino, ga, s->Gtmp, Gnew, st)) return e;
        } else if (int e = launch_back<EPI_STORE>(g, v, s->sino, s->Gtmp, ga, st)) {
            return e;
        }
        tmark_end(s, st, 2, t1);
        int t2 = tmark(s, st);
        if (s->band && !CT_BAND_OVERLAP) {   // helical: z-band blocks instead of the full reduce-scatter
            if (int e = band_reduce(s, m, s->Gtmp, Gnew, st)) return e;
        } else if (!s->band) {
            if (int e = comm_rc(g, g->comm->reduce_scatter_sum(s->Gtmp, Gnew + s->off0, s->S, st))) return e;
        }
        const size_t j0 = s->off0, j1 = std::min(s->N, s->off0 + s->S);
        if (epi == EPI_INIT) {
            if (j1 > j0) CT_CUDA(cudaMemcpyAsync(s->gs + j0, Gnew + j0, (j1 - j0) * 4, cudaMemcpyDeviceToDevice, st));
            tmark_end(s, st, 4, t2);
            return CT_OK;
        }
        ga.G_old = s->Gbuf[s->curG];
        ga.G_new = Gnew;
        gupd_slab_kernel<<<nblk(std::max(j1, j0 + 1) - j0), 256, 0, st>>>(ga, j0, j1, s->xi_ex);
        CT_LAUNCHED(1);
        if (int e = comm_rc(g, g->comm->allreduce_sum(s->xi_ex, s->xi_ex + 1, 1, COMM_F64, st))) return e;
        xi_rule_kernel<<<1, 256, 0, st>>>(ga, s->xi_ex + 1);
        CT_LAUNCHED(1);
        tmark_end(s, st, 4, t2);
        return CT_OK;
    }
    // multi-rank (FISTA inner solver): partial back-projection, NCCL sum, unfused epilogue
    int t1 = tmark(s, st);
    if (int e = launch_back<EPI_STORE>(g, v, s->sino, s->Gtmp, ga, st)) return e;
    tmark_end(s, st, 2, t1);
    int t2 = tmark(s, st);
    if (int e = allreduce(g, s->Gtmp, s->N, st)) return e;
    if (epi == EPI_INIT) {
        CT_CUDA(cudaMemcpyAsync(s->Gbuf[s->curG], s->Gtmp, s->N * 4, cudaMemcpyDeviceToDevice, st));
        CT_CUDA(cudaMemcpyAsync(s->gs, s->Gtmp, s->N * 4, cudaMemcpyDeviceToDevice, st));
        return CT_OK;
    }
    ga.G_old = s->Gbuf[s->curG];
    ga.G_new = s->Gbuf[s->curG ^ 1];
    gupd_kernel<<<nblk(s->N), 256, 0, st>>>(s->Gtmp, ga, s->N);
    CT_LAUNCHED(1);
    tmark_end(s, st, 4, t2);
    return CT_OK;
}

// Enqueue one outer iteration (M inner steps) on stream st.  x is updated in place.
static int enqueue_iteration(ct_oslalm_state* s, const ct_oslalm_data* d, float* x, cudaStream_t st, int* nk) {
    const ct_geom* g = s->g;
    const ct_oslalm_cfg& c = s->cfg;
    int M = c.M;
    // slab path: iterate on the state's full-image buffers (all-gathered after each update)
    float* xa = s->slab ? s->xp[0] : x;
    float* xb = s->slab ? s->xp[1] : s->xalt;
    if (s->slab) CT_CUDA(cudaMemcpyAsync(xa, x, s->N * 4, cudaMemcpyDeviceToDevice, st));
    // rows this rank updates (all rows on one rank)
    const int ry0 = s->slab ? s->iy0 : 0, ry1 = s->slab ? s->iy1 : g->d.ny;
    const size_t rj0 = (size_t)ry0 * g->d.nx * nz_of(g), rj1 = (size_t)ry1 * g->d.nx * nz_of(g);
    float inv_d = (float)(1.0 / c.reg.delta);
    int kernels = 0;
    for (int j = 0; j < M; j++) {
        int t0 = tmark(s, st);
        if (c.inner == CT_INNER_SQS) {
            if (ry1 > ry0) {
                if (c.reg.nbr == 8 && nz_of(g) == 1)
                    CT_CUDA(launch_pdl(sqs_update2d_kernel, dim3((g->dg.nx + 31) / 32, (ry1 - ry0 + 7) / 8), dim3(256), 0,
                                       st, g->dg, (const float*)xa, xb, (const float*)s->Gbuf[s->curG],
                                       (const float*)s->gs, d->dl, d->mask, (const double*)&s->sc->rho,
                                       (const double*)&s->sc->alpha, (float)c.reg.beta, inv_d, ry0, ry1));
                else if (c.reg.nbr == 8)
                    sqs_update_kernel<8><<<nblk(rj1 - rj0), 256, 0, st>>>(g->dg, xa, xb, s->Gbuf[s->curG], s->gs, d->dl,
                                                                          d->mask, &s->sc->rho, &s->sc->alpha, (float)c.reg.beta,
                                                                          inv_d, rj0, rj1);
                else {
                    ZHalo hz{nullptr, nullptr, nullptr, nullptr};
                    if (g->zslab && g->nranks > 1) {   // neighbours' boundary slices of x (and of S, once)
                        if (int e = zslab_halo<float>(g, xa, s->zsend[0], s->zsend[1], s->zrecv[0], s->zrecv[1], st))
                            return e;
                        if (g->rank > 0) { hz.lo = s->zrecv[0]; hz.mlo = s->zmask[0]; }
                        if (g->rank < g->nranks - 1) { hz.hi = s->zrecv[1]; hz.mhi = s->zmask[1]; }
                    }
                    const dim3 grid((g->dg.nx + 7) / 8, (g->dg.nz + 31) / 32, (ry1 - ry0 + kK3Y - 1) / kK3Y);
                    if (hz.lo || hz.hi)
                        sqs_update3d_kernel<true><<<grid, 256, 0, st>>>(g->dg, xa, xb, s->Gbuf[s->curG], s->gs, d->dl,
                                                                        d->mask, &s->sc->rho, &s->sc->alpha,
                                                                        (float)c.reg.beta, inv_d, ry0, ry1, hz);
                    else
                        sqs_update3d_kernel<false><<<grid, 256, 0, st>>>(g->dg, xa, xb, s->Gbuf[s->curG], s->gs, d->dl,
                                                                         d->mask, &s->sc->rho, &s->sc->alpha,
                                                                         (float)c.reg.beta, inv_d, ry0, ry1, hz);
                }
                CT_LAUNCHED(1);
            }
            if (s->band) {   // x+ inside the next subset's band (+ the stencil's halo rows)
                if (int e = band_gather(s, s->order[(j + 1) % M], xb, st)) return e;
            } else if (s->slab) {   // every rank needs the full x+ for its next forward projection
                if (int e = comm_rc(g, g->comm->all_gather(xb + s->off0, xb, s->S, st))) return e;
            }
        } else {
            // n warm-started FISTA iterations: v_0 = x_0 = x_k (= xa), result in xb
            double t = 1.0;
            const float* v = xa;
            const float* xprev = xa;
            for (int i = 1; i <= c.n_inner; i++) {
                double tn = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t));
                float mom = (float)((t - 1.0) / tn);
                bool last = i == c.n_inner;
                float* vout = last ? nullptr : s->vbuf[i & 1];
#define CT_FISTA(NB, LAST)                                                                                         \
    fista_step_kernel<NB, LAST><<<nblk(s->N), 256, 0, st>>>(g->dg, v, xprev, xa, xb, vout, s->Gbuf[s->curG], s->gs, \
                                                            d->dl, d->mask, &s->sc->rho, &s->sc->alpha, (float)c.reg.beta, \
                                                            inv_d, mom, s->N)
                if (c.reg.nbr == 8) {
                    if (last) CT_FISTA(8, true); else CT_FISTA(8, false);
                } else {
                    if (last) CT_FISTA(26, true); else CT_FISTA(26, false);
                }
#undef CT_FISTA
                CT_LAUNCHED(1);
                v = vout;
                xprev = xb;
                t = tn;
            }
        }
        tmark_end(s, st, 0, t0);
        std::swap(xa, xb);
        if (c.bb) {   // BB (reading B-BB): mean of the points where this iteration's gradients are taken
            const size_t bj0 = s->slab ? s->off0 : 0, bj1 = s->slab ? std::min(s->N, s->off0 + s->S) : s->N;
            xbar_acc_kernel<<<nblk(std::max(bj1, bj0 + 1) - bj0), 256, 0, st>>>(s->xbar, xa, 1.0f / (float)M, bj0, bj1);
            kernels += 1;
        }
        s->log_slot = j;
        if (int e = subset_gradient(s, d, xa, s->order[(j + 1) % M], EPI_GUPD, st)) return e;
        s->log_slot = -1;
        s->curG ^= 1;
        kernels += 2 + (c.inner == CT_INNER_FISTA ? c.n_inner : 1) + (g->comm ? 1 : 0);
    }
    if (c.bb) {
        // Barzilai-Borwein scale for the next outer iteration (reading B-BB), over this rank's
        // rows (all rows on one rank; gbar is valid on the rank's slab in the slab path)
        const size_t bj0 = s->slab ? s->off0 : 0, bj1 = s->slab ? std::min(s->N, s->off0 + s->S) : s->N;
        BBArgs bbA{s->xbar, s->xprev, s->gbar, s->gprev, d->dl, d->mask, s->bb_part, g->comm ? s->xi_ex + 2 : nullptr,
                   s->sc, c.alpha_min};
        bb_alpha_kernel<<<nblk(std::max(bj1, bj0 + 1) - bj0), 256, 0, st>>>(bbA, bj0, bj1);
        kernels += 1;
        if (g->comm) {
            if (int e = comm_rc(g, g->comm->allreduce_sum(s->xi_ex + 2, s->xi_ex + 2, 2, COMM_F64, st))) return e;
            bb_rule_kernel<<<1, 1, 0, st>>>(s->sc, s->xi_ex + 2, c.alpha_min);
            kernels += 1;
        }
    }
    if (s->band)   // the iterate in full on every rank once per outer iteration
        if (int e = comm_rc(g, g->comm->all_gather(xa + s->off0, xa, s->S, st))) return e;
    if (xa != x) {
        CT_CUDA(cudaMemcpyAsync(x, xa, s->N * 4, cudaMemcpyDeviceToDevice, st));
    }
    if (s->slab) kernels += M;   // xi_rule per step
    if (nk) *nk = kernels;
    return CT_OK;
}

static int ensure_initialised(ct_oslalm_state* s, const ct_oslalm_data* d, float* x, cudaStream_t st) {
    if (s->initialised) return CT_OK;
    const ct_oslalm_cfg& c = s->cfg;
    init_scalars_kernel<<<1, 1, 0, st>>>(s->sc, c.mode == CT_RHO_FIXED ? c.rho_fixed : 1.0);
    CT_LAUNCHED(1);
    if (s->fs.acc2d) {   // the fan accumulator is kept zero by the projections from here on
        const int maxcount = (s->g->d.na + c.M - 1) / c.M;
        CT_CUDA(cudaMemsetAsync(s->fs.acc2d, 0, (size_t)maxcount * s->g->d.ns * 8, st));
    }
    zero_offmask_kernel<<<nblk(s->N), 256, 0, st>>>(x, d->mask, s->N);
    CT_LAUNCHED(1);
    if (c.bb) CT_CUDA(cudaMemsetAsync(s->gbar, 0, s->Npad * 4, st));
    if (c.bb) CT_CUDA(cudaMemsetAsync(s->xbar, 0, s->Npad * 4, st));
    if (s->g->zslab && s->g->nranks > 1) {   // the neighbours' boundary slices of S (static)
        uint8_t* sb = reinterpret_cast<uint8_t*>(s->zsend[0]);
        if (int e = zslab_halo<uint8_t>(s->g, d->mask, sb, sb + s->g->d.nx * s->g->d.ny, s->zmask[0], s->zmask[1], st))
            return e;
    }
    if (int e = subset_gradient(s, d, x, s->order[0], EPI_INIT, st)) return e;
    s->initialised = 1;
    return CT_OK;
}

static int check_data(const ct_oslalm_data* d, const float* x) {
    if (!d || !d->y || !d->w || !d->dl || !d->mask || !x) return fail(CT_EINVAL, "ct_oslalm: null data pointer");
    return CT_OK;
}

static bool cfg_equal(const ct_oslalm_cfg& a, const ct_oslalm_cfg& b) {
    return a.M == b.M && a.mode == b.mode && a.rho_fixed == b.rho_fixed && a.rho_min == b.rho_min &&
           a.n_inner == b.n_inner && a.inner == b.inner && a.reg.beta == b.reg.beta && a.reg.delta == b.reg.delta &&
           a.reg.nbr == b.reg.nbr && a.bb == b.bb && a.alpha_min == b.alpha_min;
}

extern "C" int ct_oslalm_iter(const ct_geom* g, const ct_oslalm_cfg* cfg, const ct_oslalm_data* d, ct_oslalm_state* s,
                              float* x, void* stream) {
    NvtxRange nvtx_("ct_oslalm_iter");
    if (!g || !s) return fail(CT_EINVAL, "ct_oslalm_iter: null argument");
    if (s->g != g) return fail(CT_ESTATE, "state was created for another geometry");
    if (cfg && !cfg_equal(*cfg, s->cfg)) {
        if (int e = check_cfg(g, cfg)) return e;
        if (cfg->M != s->cfg.M) return fail(CT_ESTATE, "M changed after state creation");
        if (cfg->inner != s->cfg.inner || cfg->n_inner != s->cfg.n_inner || cfg->bb != s->cfg.bb)
            return fail(CT_ESTATE, "inner solver changed after state creation (workspace layout)");
        s->cfg = *cfg;
        for (auto& ge : s->graphs)
            if (ge.exec) { cudaGraphExecDestroy(ge.exec); ge.exec = nullptr; }
    }
    if (int e = check_data(d, x)) return e;
    if (g->nranks != s->P || g->rank != s->prank || (g->comm != nullptr) != s->has_comm)
        return fail(CT_ESTATE, "communicator changed after state creation (create the state after ct_comm_init)");
    DeviceGuard guard(g->d.device);
    cudaStream_t st = (cudaStream_t)stream;
    if (int e = ensure_initialised(s, d, x, st)) return e;
    if (g->comm || s->timing) {
        if (int e = enqueue_iteration(s, d, x, st, nullptr)) return e;
        return tcollect(s);
    }

    // single rank: capture the iteration once per (buffers, G parity) and replay it
    const void* key[6] = {x, d->y, d->w, d->dl, d->mask, s->gs};
    GraphEntry* ge = nullptr;
    for (auto& e : s->graphs)
        if (e.exec && e.curG == s->curG && memcmp(e.key, key, sizeof(key)) == 0) ge = &e;
    int startG = s->curG;
    if (!ge) {
        // an empty slot, else the least recently used one (a caller alternating data buffers,
        // e.g. double-buffered inputs, keeps one instantiated graph per buffer set)
        ge = &s->graphs[0];
        for (auto& e : s->graphs) {
            if (!e.exec) { ge = &e; break; }
            if (e.used < ge->used) ge = &e;
        }
        if (ge->exec) { cudaGraphExecDestroy(ge->exec); ge->exec = nullptr; }
        cudaGraph_t graph;
        CT_CUDA(cudaStreamBeginCapture(s->cap, cudaStreamCaptureModeThreadLocal));
        unsigned long long before = g_launches.load();
        int nk = 0;
        int err = enqueue_iteration(s, d, x, s->cap, &nk);
        g_launches = before;  // capture does not execute kernels
        cudaError_t ce = cudaStreamEndCapture(s->cap, &graph);
        s->curG = startG;     // capture did not run; restore the parity
        if (err) return err;
        if (ce != cudaSuccess) return fail(CT_ECUDA, "graph capture: %s", cudaGetErrorString(ce));
        ce = cudaGraphInstantiate(&ge->exec, graph, 0);
        // kernel launches per replay = the graph's kernel nodes (exact, for ct_kernel_launches)
        size_t nn = 0, nkern = 0;
        cudaGraphGetNodes(graph, nullptr, &nn);
        std::vector<cudaGraphNode_t> nodes(nn);
        if (nn) cudaGraphGetNodes(graph, nodes.data(), &nn);
        for (size_t i = 0; i < nn; i++) {
            cudaGraphNodeType t;
            if (cudaGraphNodeGetType(nodes[i], &t) == cudaSuccess && t == cudaGraphNodeTypeKernel) nkern++;
        }
        cudaGraphDestroy(graph);
        if (ce != cudaSuccess) return fail(CT_ECUDA, "graph instantiate: %s", cudaGetErrorString(ce));
        memcpy(ge->key, key, sizeof(key));
        ge->curG = startG;
        ge->nodes = nkern ? nkern : (size_t)nk;
    }
    CT_CUDA(cudaEventRecord(s->ev_in, st));
    CT_CUDA(cudaStreamWaitEvent(s->cap, s->ev_in, 0));
    ge->used = ++s->replays;
    CT_CUDA(cudaGraphLaunch(ge->exec, s->cap));
    CT_CUDA(cudaEventRecord(s->ev_out, s->cap));
    CT_CUDA(cudaStreamWaitEvent(st, s->ev_out, 0));
    g_launches += ge->nodes;
    if (s->cfg.M & 1) s->curG ^= 1;
    return CT_OK;
}

extern "C" int ct_oslalm_run(const ct_geom* g, const ct_oslalm_cfg* cfg, const ct_oslalm_data* d, ct_oslalm_state* s,
                             float* x, int n_iter, ct_oslalm_log* log, void* stream) {
    NvtxRange nvtx_("ct_oslalm_run");
    if (n_iter < 0) return fail(CT_EINVAL, "n_iter < 0");
    if (log) log->count = 0;
    DeviceGuard guard(g ? g->d.device : 0);
    cudaStream_t st = (cudaStream_t)stream;
    std::vector<double> h;
    for (int it = 0; it < n_iter; it++) {
        if (int e = ct_oslalm_iter(g, cfg, d, s, x, stream)) return e;
        if (log) {
            int M = s->cfg.M;
            h.resize((size_t)M * 3);
            CT_CUDA(cudaMemcpyAsync(h.data(), s->dlog, sizeof(double) * M * 3, cudaMemcpyDeviceToHost, st));
            CT_CUDA(cudaStreamSynchronize(st));
            for (int j = 0; j < M && log->count < log->capacity; j++, log->count++) {
                if (log->rho) log->rho[log->count] = h[3 * j];
                if (log->xi) log->xi[log->count] = h[3 * j + 1];
                if (log->restart) log->restart[log->count] = (int)h[3 * j + 2];
            }
        }
    }
    CT_CUDA(cudaStreamSynchronize(st));
    CT_CUDA(cudaGetLastError());
    return CT_OK;
}

// ---------------------------------------------------------------------------
// multi-GPU
// ---------------------------------------------------------------------------
extern "C" int ct_comm_get_unique_id(void* uid) {
    if (!uid) return fail(CT_EINVAL, "null uid");
    if (!load_nccl()) return fail(CT_ENCCL, "libnccl.so.2 not loadable: %s", dlerror());
    ncclUniqueId id;
    ncclResult_t r = g_nccl.GetUniqueId(&id);
    if (r != ncclSuccess) return fail(CT_ENCCL, "ncclGetUniqueId failed (%d)", (int)r);
    memcpy(uid, &id, sizeof(id));
    return CT_OK;
}

extern "C" int ct_comm_init(ct_geom* g, int rank, int nranks, const void* uid) {
    if (!g || !uid) return fail(CT_EINVAL, "ct_comm_init: null argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(CT_EINVAL, "bad rank %d of %d", rank, nranks);
    // nranks == 1 still creates a (trivial) communicator: the exchange path (partial
    // back-projection, reduce-scatter, slab g-update, all-gather) then runs on one GPU.
    if (!load_nccl()) return fail(CT_ENCCL, "libnccl.so.2 not loadable");
    delete g->comm;
    g->comm = nullptr;
    DeviceGuard guard(g->d.device);
    ncclUniqueId id;
    memcpy(&id, uid, sizeof(id));
    NcclComm* c = new NcclComm();
    ncclResult_t r = g_nccl.CommInitRank(&c->comm, nranks, id, rank);
    if (r != ncclSuccess) {
        c->comm = nullptr;
        delete c;
        return fail(CT_ENCCL, "ncclCommInitRank: %s", nccl_err(r));
    }
    c->rank = rank;
    c->nranks = nranks;
    g->comm = c;
    g->rank = rank;
    g->nranks = nranks;
    g->zslab = 0;
    g->slab_zb0.clear();
    g->slab_nz.clear();
    return CT_OK;
}

extern "C" int ct_comm_set_exchange(ct_geom* g, int mode) {
    if (!g) return fail(CT_EINVAL, "ct_comm_set_exchange: null geometry");
    if (mode != CT_EXCHANGE_AUTO && mode != CT_EXCHANGE_FULL && mode != CT_EXCHANGE_BAND)
        return fail(CT_EINVAL, "ct_comm_set_exchange: bad mode %d", mode);
    if (mode == CT_EXCHANGE_BAND && g->d.kind == CT_FAN2D)
        return fail(CT_EUNSUPPORTED, "band-limited exchange needs a cone-beam geometry");
    g->exchange = mode;
    return CT_OK;
}

extern "C" int ct_comm_init_virtual(ct_geom** gs, int nranks, int zslab) {
    if (!gs || nranks < 1) return fail(CT_EINVAL, "ct_comm_init_virtual: bad arguments");
    for (int r = 0; r < nranks; r++) {
        if (!gs[r]) return fail(CT_EINVAL, "ct_comm_init_virtual: null geometry %d", r);
        if (gs[r]->d.device != gs[0]->d.device) return fail(CT_EINVAL, "virtual ranks must share one device");
        if (zslab && gs[r]->d.kind == CT_FAN2D) return fail(CT_EUNSUPPORTED, "z-slab decomposition needs a cone-beam geometry");
        for (int q = 0; q < r; q++)
            if (gs[q] == gs[r]) return fail(CT_EINVAL, "virtual ranks need distinct geometry handles");
    }
    DeviceGuard guard(gs[0]->d.device);
    auto grp = std::make_shared<VirtualGroup>();
    if (grp->init(nranks, gs[0]->d.device)) return fail(CT_ECUDA, "virtual ranks: stream / event creation failed");
    for (int r = 0; r < nranks; r++) {
        delete gs[r]->comm;
        VirtualComm* c = new VirtualComm();
        c->grp = grp;
        c->rank = r;
        c->nranks = nranks;
        gs[r]->comm = c;
        gs[r]->rank = r;
        gs[r]->nranks = nranks;
        gs[r]->zslab = zslab ? 1 : 0;
        gs[r]->slab_zb0.clear();
        gs[r]->slab_nz.clear();
        for (int q = 0; zslab && q < nranks; q++) {
            gs[r]->slab_zb0.push_back(gs[q]->dg.zb0);
            gs[r]->slab_nz.push_back(gs[q]->dg.nz);
        }
    }
    return CT_OK;
}

extern "C" int ct_comm_init_zslab(ct_geom* g, int rank, int nranks, const void* uid) {
    if (!g) return fail(CT_EINVAL, "ct_comm_init_zslab: null argument");
    if (g->d.kind == CT_FAN2D) return fail(CT_EUNSUPPORTED, "z-slab decomposition needs a cone-beam geometry");
    if (int e = ct_comm_init(g, rank, nranks, uid)) return e;
    g->zslab = 1;
    // every rank's slab extent (zb0, nz): the windowed exchange needs the other ranks' view windows
    DeviceGuard guard(g->d.device);
    float* dz = nullptr;
    cudaStream_t st = nullptr;
    std::vector<float> h(2 * (size_t)nranks);
    const float mine[2] = {g->dg.zb0, (float)g->dg.nz};
    cudaError_t ce = cudaMalloc(&dz, h.size() * 4);
    if (ce == cudaSuccess) ce = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    if (ce == cudaSuccess) ce = cudaMemcpy(dz + 2 * rank, mine, 8, cudaMemcpyHostToDevice);
    int rc = ce == cudaSuccess ? g->comm->all_gather(dz + 2 * rank, dz, 2, st) : 0;
    if (ce == cudaSuccess && !rc) ce = cudaStreamSynchronize(st);
    if (ce == cudaSuccess && !rc) ce = cudaMemcpy(h.data(), dz, h.size() * 4, cudaMemcpyDeviceToHost);
    if (st) cudaStreamDestroy(st);
    if (dz) cudaFree(dz);
    if (ce != cudaSuccess) return fail(CT_ECUDA, "ct_comm_init_zslab: %s", cudaGetErrorString(ce));
    if (rc) return comm_rc(g, rc);
    g->slab_zb0.resize(nranks);
    g->slab_nz.resize(nranks);
    for (int q = 0; q < nranks; q++) {
        g->slab_zb0[q] = h[2 * q];
        g->slab_nz[q] = (int)h[2 * q + 1];
    }
    return CT_OK;
}
