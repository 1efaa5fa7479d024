/*
 * ct_oslalm.h — C ABI of the B200 (sm_100a) OS-LALM CT hot path.
 *
 * Method: Nien & Fessler, "Fast X-ray CT image reconstruction using a linearized
 * augmented Lagrangian method with ordered subsets" (arXiv 1402.4381).
 * Citations "P:n" are lines of that paper's text; "O1..O7", "G1..G21"
 * are the readings of silent/ambiguous passages listed in DESIGN.md §Readings.
 *
 * Problem solved (eq. ct_recon):
 *     x_hat in argmin_{x in Omega} 1/2 ||y - A x||_W^2 + R(x),   Omega = {x >= 0}
 * with OS-LALM (eq. os_lalm_iterates), the SQS majoriser
 * L_diag = diag{A' W A 1} and bit-reversal subset order, one warm-started
 * FISTA step for the inner denoising problem (n = 1) and the
 * deterministic downward rho-continuation with adaptive restart.
 *
 * ---------------------------------------------------------------------------
 * Conventions for every call
 * ---------------------------------------------------------------------------
 * Pointers: every array argument is a DEVICE pointer on the geometry's device,
 *   allocated and owned by the caller (the Python binding uses torch).  The
 *   library owns only the opaque handles it returns (ct_geom, ct_oslalm_state)
 *   and frees them on destroy.  No allocations happen after create.
 * Layouts (z / detector-row fastest, chosen so that the separable footprint's
 *   axial loops are unit-stride):
 *     image     x[iy][ix][iz]        (nz = 1 for FAN2D)         fp32
 *     sinogram  y[k][c][r]           (k = index into a view list, c = channel,
 *                                     r = detector row; nt = 1 for FAN2D) fp32
 *     mask      m[iy][ix][iz]        uint8, nonzero = voxel in the support S
 * Streams: `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *   stream).  Work is enqueued asynchronously; only the calls documented as
 *   synchronising block the host.
 * Errors: return CT_OK (0) or a ct_status code; ct_last_error() returns a
 *   thread-local one-line message.  Arguments are validated before any launch
 *   (no partial writes on CT_EINVAL).  No C++ exception crosses the boundary.
 *   Asynchronous device faults surface at the next synchronising call.
 */
#ifndef CT_OSLALM_H
#define CT_OSLALM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    CT_OK = 0,
    CT_EINVAL = 1,       /* bad argument, shape or geometry                     */
    CT_EUNSUPPORTED = 2, /* valid but not implemented (e.g. n_inner != 1)       */
    CT_ENOMEM = 3,       /* workspace too small / device allocation failed     */
    CT_ECUDA = 4,        /* CUDA runtime error                                 */
    CT_ENCCL = 5,        /* NCCL error                                         */
    CT_ESTATE = 6        /* state/handle used inconsistently                   */
} ct_status;

typedef enum { CT_FAN2D = 0, CT_CONE_AXIAL = 1, CT_CONE_HELICAL = 2 } ct_geom_kind;

/*
 * Scan geometry (reading O1).  Arc (equi-angular) detector of radius dsd centred
 * on the source.  Voxel centres x_i = (i - (nx-1)/2) dx + offx (same for y, z).
 * View v: beta_v = orbit_start + 2 pi turns v / na, turns = orbit_deg / 360;
 * source at (-dso sin beta, dso cos beta, z_s(v)) with
 * z_s(v) = (v - (na-1)/2) * pitch * nt * dt * (dso/dsd) / (na/turns) (helical; 0 otherwise).
 * Channel c sits at fan angle gamma_c = (c - (ns-1)/2 - offs) ds / dsd; row r at
 * height t_r = (r - (nt-1)/2 - offt) dt on the cylindrical detector.
 * Lengths in mm, angles in degrees.  dx must equal dy.
 */
typedef struct {
    int kind;                 /* ct_geom_kind */
    int nx, ny, nz;
    double dx, dy, dz;
    double offx, offy, offz;
    int ns, nt;
    double ds, dt;
    double offs, offt;
    double dso, dsd;
    int na;
    double orbit_deg, orbit_start_deg;
    double pitch;
    int device;               /* CUDA device ordinal for all calls on this geometry */
} ct_geom_desc;

typedef struct ct_geom ct_geom;

/* A view list {first + k*stride : 0 <= k < count}.  Subset m of M (reading G12):
 * {m, M, ceil((na-m)/M)}; the full scan: {0, 1, na}. */
typedef struct {
    int first, stride, count;
} ct_views;

/* Validate the description and build per-view tables on the device.
 * The geometry tables are immutable afterwards, and every call that needs scratch takes
 * it from a caller-owned buffer (ct_sqs_denom's scratch, the OS-LALM state's workspace),
 * so cone-beam geometries may be used from several streams at once.  The one exception:
 * ct_fwd_proj on a FAN2D geometry accumulates into a geometry-owned 64-bit fixed-point
 * buffer (kept zero between calls), so standalone fan-beam ct_fwd_proj calls with one
 * geometry must be ordered on one stream (or by events).
 * Returns CT_EINVAL for inconsistent sizes, CT_EUNSUPPORTED if some voxel's
 * transaxial footprint could span more than 7 channels (kernel window limit), or,
 * for fan beams, if consecutive pixels can be less than 1/8 channel apart on the
 * detector (forward tile kernel's lane-parity buffers) or a 32x32 pixel tile's
 * channel span does not fit its shared-memory buffers. */
int ct_geom_create(const ct_geom_desc* desc, ct_geom** out);
void ct_geom_destroy(ct_geom* g);
const char* ct_last_error(void);

/*
 * Forward projection y = A_v x over the view list v ("one multiplication
 * by A"; system matrix A = separable-footprint SF-TR with A1 amplitude, reading
 * O2 / G1):  a_ij = l_phi * l_theta * F_s(c) * F_t(r).
 * x: [ny][nx][nz]; y: [count][ns][nt], overwritten.  Deterministic: no floating-point
 * atomics (the 2D tile sums meet in exact 64-bit integer adds, order-independent).
 * Fan beam (FAN2D): the 32x32-pixel tile partial sums are added in 64-bit fixed point
 * with unit 2^-40 (absolute quantum 9.1e-13 per tile partial); valid while every tile
 * partial and every |y| stays below 2^23 = 8.4e6 (with attenuation-scale images, ~0.02
 * mm^-1 and line integrals <= ~20, x may be scaled from ~1e-7 to ~1e5 and keep 1e-6
 * relative accuracy).  Outside that range the result is undefined (the fixed-point sum
 * overflows); nothing checks it.  Cone beam: plain fp32 sums in a fixed order, no range
 * limit.  Cone-beam ct_fwd_proj does not trim all-zero image columns (the OS-LALM path
 * and ct_sqs_denom do, with per-call scratch).
 */
int ct_fwd_proj(const ct_geom* g, ct_views v, const float* x, float* y, void* stream);

/*
 * Back projection x (+)= A_v' y, the exact adjoint of ct_fwd_proj (same a_ij; "one
 * multiplication by A'"; the gradient M A_m'(W(A_m x - y)) of P:380-397).
 * y: [count][ns][nt]; x: [ny][nx][nz]; accumulate != 0 adds to x, else overwrites.
 */
int ct_back_proj(const ct_geom* g, ct_views v, const float* y, float* x, int accumulate, void* stream);

/*
 * SQS denominator (L_diag = diag{A' W A 1}; reading O4/G13):
 *   D_L = A'(W .* (A 1_S)) over all na views, then S <- S and {D_L > 0},
 *   D_L := 0 off S.
 * w: [na][ns][nt] statistical weights; mask_inout: [ny][nx][nz] (updated in place);
 * dl: [ny][nx][nz] output.  `scratch` is a device buffer of at least
 * ct_sqs_denom_scratch_bytes() bytes (caller-owned).
 */
int ct_sqs_denom_scratch_bytes(const ct_geom* g, size_t* out);
int ct_sqs_denom(const ct_geom* g, const float* w, uint8_t* mask_inout, float* dl, void* scratch,
                 void* stream);

/*
 * Edge-preserving regulariser ("R is an edge-preserving regularizer";
 * reading G3/G14):  R(x) = beta sum_{unordered pairs {j,k} in S, k in N(j)} w_jk psi(x_j - x_k)
 * with the Fair potential psi(t) = delta^2 (|t|/delta - ln(1 + |t|/delta)),
 * N = 8 in-plane neighbours (nbr = 8) or the 26-neighbourhood (nbr = 26, 3D),
 * w_jk = 1/||offset||.  Writes grad_j = beta sum_k w_jk psi'(x_j - x_k) and,
 * if curv != NULL, the Huber curvature D_R,j = 2 beta sum_k w_jk / (1 + |x_j - x_k|/delta).
 * Both are 0 off S.
 */
typedef struct {
    double beta, delta;
    int nbr; /* 8 or 26 */
} ct_reg;

int ct_reg_grad(const ct_geom* g, const ct_reg* r, const uint8_t* mask, const float* x, float* grad,
                float* curv, void* stream);

/*
 * Work counts of a view list (the throughput metric's units):
 *   out_host[0] = U   = #(view, voxel in mask) pairs with a non-empty footprint,
 *   out_host[1] = nnz = #non-zero a_ij of those pairs (channels x rows overlapped),
 *   out_host[2] = C   = #(view, voxel column) pairs with >= 1 voxel counted in U.
 * Evaluated with fp64 geometry.  SYNCHRONISING.  `scratch`: device buffer >= 32 bytes.
 */
int ct_count_vv(const ct_geom* g, ct_views v, const uint8_t* mask, void* scratch, long long* out_host,
                void* stream);

/* ------------------------------------------------------------------------ */
/* OS-LALM                                                                  */
/*
 * FBP / FDK initial image x^0 (NEXT-4; "initialized with a standard filtered
 * back-projection (FBP) reconstruction"; reading B-FBP): full-scan equiangular
 * fan-beam FBP (Ram-Lak taps, cos gamma pre-weight, 1/L^2 back-projection weight,
 * linear interpolation), with the FDK extension (cone weight D / sqrt(D^2 + zeta^2),
 * bilinear interpolation) for axial cone beam.  Helical scans (the paper's helical cases
 * start from an FBP image too; reading B-FBP-H): the same filtering and
 * a back-projection over the views whose cone sees the voxel (projected row inside
 * [0, nt - 1]), normalised by their number (2 pi / #seen instead of 2 pi / na).
 *   y        : [na][ns][nt] post-log sinogram (device, read-only)
 *   x        : [ny][nx][nz] output image in mm^-1 (device, overwritten)
 *   scratch  : ct_fbp_scratch_bytes() bytes of device memory (filtered sinogram)
 * Errors: CT_EINVAL (null pointers), CT_EUNSUPPORTED (a circular orbit that is not one full
 * turn).  The image is not clipped to x >= 0 (OS-LALM's first update does).
 */
int ct_fbp_scratch_bytes(const ct_geom* g, size_t* out);
/* Diagnostic (no ct_geom): L2-resident read bandwidth of `device` in GB/s, measured by
 * streaming a `bytes`-sized buffer `reps` times (allocates and frees its own buffer).
 * The denominator of the gather roofline that bench.py reports. */
int ct_peak_l2_read(int device, size_t bytes, int reps, double* gbs);
int ct_fbp(const ct_geom* g, const float* y, float* x, void* scratch, void* stream);

/* ------------------------------------------------------------------------ */

typedef enum { CT_RHO_FIXED = 0, CT_RHO_CONTINUATION = 1 } ct_rho_mode;

typedef enum {
    CT_INNER_SQS = 0,   /* one SQS step with the Huber curvature of R at x (n_inner = 1; reading G14) */
    CT_INNER_FISTA = 1  /* n_inner warm-started FISTA iterations with the fixed Lipschitz metric
                           rho D_L + 2 beta sum_k w_jk ("n iterations of FISTA"; NEXT-1)   */
} ct_inner_mode;

typedef struct {
    int M;            /* number of ordered subsets, 1 <= M <= na                 */
    int mode;         /* ct_rho_mode                                             */
    double rho_fixed; /* FIXED mode: AL penalty rho in (0, 1]                    */
    double rho_min;   /* CONTINUATION floor, P:516 uses 1e-3                     */
    int n_inner;      /* inner iterations: 1 for CT_INNER_SQS, 1..64 for FISTA   */
    int inner;        /* ct_inner_mode                                           */
    ct_reg reg;
    /* EXPERIMENTAL.  Barzilai-Borwein scaling (NEXT-2, supplement P:1472-1492): with
     * bb = 1 the SQS Hessian D_L is replaced by H_k = alpha_k D_L, alpha_k fitted to the
     * secant equation y_k ~ H_k s_k in the D_L^{-1}-weighted least-squares sense, alpha <= 1:
     *   alpha_k = min(1, max(alpha_min, y_k's_k / s_k'D_L s_k)),
     * s_k = xbar_k - xbar_{k-1} (xbar_k: mean of outer iteration k's inner iterates, the points
     * its subset gradients were taken at), y_k = the difference of the mean subset gradients
     * of outer iterations k and k-1 (reading B-BB; for M = 1, xbar_k = x^k and this
     * is the paper's pair); alpha = 1 for the first two outer iterations.  With ordered subsets
     * (M = 4 .. 24 from x = 0) alpha cycles and the scaled steps can collapse the image towards
     * 0 (DESIGN.md B-BB): an option, not a default.                                        */
    int bb;           /* 0 or 1                                                  */
    double alpha_min; /* lower clip of alpha, in (0, 1] (1e-6)                   */
} ct_oslalm_cfg;

/* Caller-owned device arrays describing the problem. */
typedef struct {
    const float* y;      /* [na][ns][nt] post-log sinogram                     */
    const float* w;      /* [na][ns][nt] statistical weights W                 */
    const float* dl;     /* [ny][nx][nz] D_L from ct_sqs_denom (0 off S)       */
    const uint8_t* mask; /* [ny][nx][nz] support S from ct_sqs_denom           */
} ct_oslalm_data;

typedef struct ct_oslalm_state ct_oslalm_state;

/* Per inner step diagnostics (host memory, caller-owned). */
typedef struct {
    double* rho;   /* rho used in the step                              */
    double* xi;    /* restart indicator xi, fp64            */
    int* restart;  /* 1 if xi > 0 (counter l reset), else 0             */
    int capacity;  /* entries available                                 */
    int count;     /* entries written (output)                          */
} ct_oslalm_log;

/* Device pointers into a state's workspace (for tests and checkpointing). */
typedef struct {
    float* g;        /* split gradient g                          */
    float* G;        /* current scaled subset gradient M grad l_m(x)      */
    double* rho;     /* rho for the next inner step                       */
    long long* l;    /* continuation counter                              */
    long long* step; /* inner steps taken                                 */
    int initialised; /* 0 until the first ct_oslalm_iter/run              */
    double* alpha;   /* BB scale used by the next outer iteration (1 without BB) */
} ct_oslalm_state_view;

/*
 * Workspace bytes for a state (g, two G buffers, the alternate image, one
 * subset's residual sinogram, fp64 reduction partials, scalars and a device log).
 */
int ct_oslalm_state_bytes(const ct_geom* g, const ct_oslalm_cfg* cfg, size_t* out);

/* Create a state over a caller-owned device workspace of `bytes` bytes.
 * The handle keeps the cfg, an internal capture stream and CUDA-graph caches. */
int ct_oslalm_state_create(const ct_geom* g, const ct_oslalm_cfg* cfg, void* workspace, size_t bytes,
                           ct_oslalm_state** out);
void ct_oslalm_state_destroy(ct_oslalm_state* s);
int ct_oslalm_state_get(const ct_oslalm_state* s, ct_oslalm_state_view* out);

/* Forget the iterate history (next iter re-initialises G, g, l, rho); keeps graphs. */
int ct_oslalm_state_reset(ct_oslalm_state* s);

/*
 * Diagnostic per-kernel timing (CUDA events on the launching stream around every
 * kernel of the inner step; disables graph replay while enabled).  Classes:
 * 0 sqs_update (K3), 1 forward+residual (K1), 2 back-projection+epilogue (K2),
 * 3 xi/rho finalize (K4), 4 multi-rank exchange (all-reduce + g-update).
 * get_timing returns accumulated milliseconds and launch counts per class.
 */
int ct_oslalm_set_timing(ct_oslalm_state* s, int enable);
int ct_oslalm_get_timing(const ct_oslalm_state* s, double* ms5, long long* count5);

/*
 * One outer iteration = M inner steps in bit-reversal order (reading O7):
 *   rho <- FIXED ? rho_fixed : rho_l(l)
 *   x   <- max(0, x - (rho G + (1-rho) g + grad R(x)) / (rho D_L + D_R(x)))   on S, 0 off S
 *          (CT_INNER_SQS; with CT_INNER_FISTA: n_inner FISTA iterations on
 *           min_{x>=0} R(x) + rho/2 ||x - (x_k - s/(rho D_L))||^2_{D_L}, s = rho G + (1-rho) g)
 *   G+  <- M A_m'(W (A_m x - y)),  m = next subset    (fused residual in the projection)
 *   xi  <- sum_S (g - G+)(G+ - G);  g <- (rho G+ + g)/(1 + rho);  G <- G+   
 *   CONTINUATION: l <- (xi > 0) ? 0 : l + 1
 * The first call also initialises G = g = M A_{m0}'(W(A_{m0} x - y)), l = 0
 * (reading G10).  x [ny][nx][nz] is read and updated in place.  With one rank
 * the whole iteration is captured once as a CUDA graph and replayed.
 */
int ct_oslalm_iter(const ct_geom* g, const ct_oslalm_cfg* cfg, const ct_oslalm_data* data, ct_oslalm_state* s,
                   float* x, void* stream);

/*
 * n_iter iterations (n_iter forward/back-projection pairs).
 * SYNCHRONISING at the end (returns the status of the whole run).  If log is
 * non-NULL the per-inner-step rho, xi and restart flags are copied into it.
 */
int ct_oslalm_run(const ct_geom* g, const ct_oslalm_cfg* cfg, const ct_oslalm_data* data, ct_oslalm_state* s,
                  float* x, int n_iter, ct_oslalm_log* log, void* stream);

/*
 * Multi-GPU (BASELINE.json north_star "each subset's views are
 * sharded over GPUs ... the partial back-projections are combined"): attach an NCCL
 * communicator to the geometry.  `nccl_uid` points to the 128-byte ncclUniqueId created by
 * rank 0 (ct_comm_get_unique_id) and broadcast by the caller (torch.distributed).
 * Afterwards ct_oslalm_iter/run on this geometry process only this rank's contiguous block
 * of each subset's views; with the SQS inner step the ranks own padded row slabs of the
 * image: the partial back-projections are combined by ncclReduceScatter (fp32) into the row
 * slabs, the g-update, xi partial and K3 update run on the rank's slab, xi is all-reduced
 * (fp64, 8 bytes) and the updated slabs are all-gathered (ncclAllGather) for the next forward
 * projection (helical scans by default exchange only z-band blocks instead, overlapped with
 * the back-projection: ct_comm_set_exchange).  The FISTA inner solver all-reduces full images
 * instead.  D_L sums the ranks' partial back-projections with ncclAllReduce.  NCCL is loaded
 * at run time (libnccl.so.2);
 * CT_ENCCL if unavailable.  Call before creating OS-LALM states (CT_ESTATE otherwise).
 */
int ct_comm_init(ct_geom* g, int rank, int nranks, const void* nccl_uid);
/*
 * z-slab decomposition (NEXT-3; SURVEY §8(e) alternative, "sinogram-domain z-slabs"):
 * each rank's geometry `g` is its z-slab of the volume (same scan, nz = the slab's slices,
 * offz placing them; slabs in rank order along z).  A x is separable over voxels, so
 * the ranks forward-project their slab for every view whose cone meets it and the partial
 * sinograms are summed (ncclAllReduce of one subset's sinogram instead of an image); each
 * rank back-projects the full residual onto its own slab (no image exchange), xi and the
 * BB sums are all-reduced, and the 26-neighbour update takes the neighbours' boundary slices
 * (ncclSend/ncclRecv of one slice each way).  Cone beam only; SQS inner step only
 * (CT_EUNSUPPORTED otherwise).  Call before creating OS-LALM states; D_L likewise sums the
 * slabs' A 1_S.  Same arguments and errors as ct_comm_init.
 */
int ct_comm_init_zslab(ct_geom* g, int rank, int nranks, const void* nccl_uid128);
int ct_comm_get_unique_id(void* nccl_uid_out128);

/*
 * Exchange of the row-slab multi-rank path (SURVEY §8(e) "Helical (c4, c5):
 * band-limited exchange"):
 *   CT_EXCHANGE_FULL  reduce-scatter of the full partial image into row slabs, all-gather of x+;
 *   CT_EXCHANGE_BAND  a rank's partial back-projection of a subset is non-zero only in the
 *                     z-band of slices its contiguous view block can see (source heights of the
 *                     block +- the cone's z reach), and its next forward projection reads x only
 *                     there: only those z-band blocks are exchanged (grouped send / receive, a
 *                     fixed rank-order sum), plus one boundary row each way for the stencil and
 *                     one full all-gather per outer iteration.  The partial back-projection runs
 *                     one destination row slab at a time and each slab's blocks are sent on an
 *                     internal communication stream while the next slab is computed;
 *   CT_EXCHANGE_AUTO  BAND for helical scans with 2..16 ranks each owning >= 1 image row, else FULL
 *                     (the default).
 * z-slab geometries (ct_comm_init_zslab, helical, 2..16 ranks): FULL all-reduces each subset's
 * summed sinogram; BAND exchanges the windowed form instead — rank p's partial projection is
 * non-zero only for the views whose cone reaches its slab (its view window), so it sends every
 * other rank q only the views both windows hold and sums what it receives in rank order
 * (ranks sharing a view hold identical sums; views outside the window are not back-projected
 * onto the slab and are left unspecified in the state's sinogram); AUTO takes BAND when the
 * busiest rank receives fewer bytes than a ring all-reduce moves per rank, else FULL (every
 * rank evaluates the same rule from the slab extents gathered at ct_comm_init_zslab).  The
 * D_L setup (ct_sqs_denom) always all-reduces.
 * Call before creating OS-LALM states.  CT_EINVAL for an unknown mode, CT_EUNSUPPORTED for BAND
 * on a fan-beam geometry (an axial scan's bands cover the whole volume: it runs, exchanging
 * the same bytes as FULL).
 */
#define CT_EXCHANGE_AUTO 0
#define CT_EXCHANGE_FULL 1
#define CT_EXCHANGE_BAND 2
int ct_comm_set_exchange(ct_geom* g, int mode);

/*
 * Virtual ranks (validation of the multi-rank path on ONE device):
 * attach `nranks` distinct geometry handles gs[0..nranks-1] of one device to one group of
 * virtual ranks (rank r = gs[r]; zslab != 0: gs[r] is rank r's z-slab geometry, as for
 * ct_comm_init_zslab).  Every exchange step of the multi-rank path then runs as a
 * rendezvous of the ranks' host threads: each rank must be driven by its own thread on its
 * own stream (ct_oslalm_iter / ct_sqs_denom of all ranks concurrently, in the same order);
 * the collective's copies and fixed-order (rank 0..P-1) sum kernels run on a group stream
 * ordered by CUDA events after every rank's stream, and every rank's stream waits for them.
 * No kernel waits on another kernel.  Replaces any communicator attached before.  (The one
 * exception to "no allocation after create": the group allocates a device staging buffer
 * for its sums at the first collective that needs a larger one.)
 * Errors: CT_EINVAL (null / duplicate handles, different devices), CT_EUNSUPPORTED (zslab on
 * a fan geometry), CT_ECUDA.  A failed exchange returns CT_ENCCL on every rank.
 */
int ct_comm_init_virtual(ct_geom** gs, int nranks, int zslab);

/* Library identification string (kernel names, target). */
const char* ct_build_info(void);

/* Number of CUDA kernels this library has launched in the process so far (a graph
 * replay counts its kernel nodes).  Used by the benchmark's gpu_launches report. */
unsigned long long ct_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* CT_OSLALM_H */
