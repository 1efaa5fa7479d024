/*
 * oracle.c — plain, slow, fp64 CPU ORACLE for the OS-LALM CT hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_1402_4381_b200/) never links, imports or calls it,
 * and it shares no code, headers or tables with the CUDA path.
 *
 * What it computes (citations: P:n = /root/reference/PAPER.md line n;
 * O1..O7 / G1..G21 = the readings in SURVEY.md §8(c), restated in DESIGN.md):
 *   O1  scan geometry (fan / cone axial / cone helical, arc detector)
 *   O2  separable-footprint SF-TR system matrix with A1 amplitude
 *       ("A is the system matrix of a CT scan"; reading G1)
 *   O4  SQS denominator D_L = A'(W (A 1_S))        (L_diag = diag{A'WA1})
 *   O5  Fair-potential regulariser R, grad R, Huber curvature D_R  (G3, G14)
 *   O6  cost Psi(x) = 1/2 ||y - Ax||_W^2 + R(x)      (eq. ct_recon)
 *   O7  OS-LALM with deterministic downward continuation and restart
 *       (P:380-397 eq. os_lalm_iterates; P:495-516 eqs. period_indicator_qp,
 *        rho_l_formula_qp; P:529-537 substitution + SQS; n = 1 FISTA step)
 *
 * Layouts (the oracle's own textbook layout; tests permute to/from the ABI):
 *   image     x[iz][iy][ix]          (nz = 1 for 2D fan)
 *   sinogram  p[v][r][c]             (view, detector row, channel; nt = 1 in 2D)
 *
 * Arithmetic: fp64 throughout.  Parallelism: OpenMP over independent outputs
 * only (views for forward, image rows for back), so results are deterministic.
 * No blocking, fusion or reordering beyond the definitions.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_FAN2D 0
#define OR_CONE_AXIAL 1
#define OR_CONE_HELICAL 2

typedef struct {
    int kind;
    int nx, ny, nz;
    double dx, dy, dz, offx, offy, offz;
    int ns, nt;
    double ds, dt, offs, offt;
    double dso, dsd;
    int na;
    double orbit_deg, orbit_start_deg, pitch;
} or_geom;

/* ---------------- O1: geometry ---------------- */

static double vox_x(const or_geom* g, int ix) { return (ix - (g->nx - 1) / 2.0) * g->dx + g->offx; }
static double vox_y(const or_geom* g, int iy) { return (iy - (g->ny - 1) / 2.0) * g->dy + g->offy; }
static double vox_z(const or_geom* g, int iz) {
    if (g->kind == OR_FAN2D) return 0.0;
    return (iz - (g->nz - 1) / 2.0) * g->dz + g->offz;
}

/* beta_v = beta_0 + 2 pi turns v / na  (O1) */
double or_view_angle(const or_geom* g, int v) {
    double turns = g->orbit_deg / 360.0;
    return g->orbit_start_deg * M_PI / 180.0 + 2.0 * M_PI * turns * v / g->na;
}

/* z_s(v) = (v - (na-1)/2) * h / (na/turns), h = pitch nt dt dso/dsd  (O1, G17) */
double or_source_z(const or_geom* g, int v) {
    if (g->kind != OR_CONE_HELICAL) return 0.0;
    double turns = g->orbit_deg / 360.0;
    double h = g->pitch * g->nt * g->dt * g->dso / g->dsd;
    return (v - (g->na - 1) / 2.0) * h / (g->na / turns);
}

/* channel centre arc position s_c = dsd * gamma_c */
static double chan_s(const or_geom* g, int c) { return (c - (g->ns - 1) / 2.0 - g->offs) * g->ds; }
static double row_t(const or_geom* g, int r) { return (r - (g->nt - 1) / 2.0 - g->offt) * g->dt; }

/* ---------------- O2: SF-TR footprint ---------------- */

/* Antiderivative of the unit-height trapezoid rising on [t0,t1], flat on
 * [t1,t2], falling on [t2,t3], evaluated at s. */
static double trap_cdf(const double t[4], double s) {
    double total = 0.5 * (t[3] + t[2] - t[1] - t[0]);
    if (s <= t[0]) return 0.0;
    if (s >= t[3]) return total;
    if (s <= t[1]) return (s - t[0]) * (s - t[0]) / (2.0 * (t[1] - t[0]));
    if (s <= t[2]) return 0.5 * (t[1] - t[0]) + (s - t[1]);
    return total - (t[3] - s) * (t[3] - s) / (2.0 * (t[3] - t[2]));
}

typedef struct {
    double tau[4];     /* sorted transaxial breakpoints (arc length on detector) */
    double lphi;       /* dx / max(|cos phi0|, |sin phi0|) */
    double rho_h;      /* in-plane source-to-voxel-centre distance */
} or_trans;

static void sort4(double a[4]) {
    for (int i = 1; i < 4; i++) {
        double k = a[i];
        int j = i - 1;
        while (j >= 0 && a[j] > k) { a[j + 1] = a[j]; j--; }
        a[j + 1] = k;
    }
}

static void transaxial(const or_geom* g, double beta, double xc, double yc, or_trans* out) {
    double sb = sin(beta), cb = cos(beta);
    /* e_c = (sin b, -cos b) points from the source through the isocentre;
     * e_perp = (cos b, sin b); source at -dso e_c. */
    double cx[4] = {xc - g->dx / 2, xc + g->dx / 2, xc - g->dx / 2, xc + g->dx / 2};
    double cy[4] = {yc - g->dy / 2, yc - g->dy / 2, yc + g->dy / 2, yc + g->dy / 2};
    for (int k = 0; k < 4; k++) {
        double along = g->dso + cx[k] * sb - cy[k] * cb;
        double perp = cx[k] * cb + cy[k] * sb;
        out->tau[k] = g->dsd * atan2(perp, along);
    }
    sort4(out->tau);
    double along = g->dso + xc * sb - yc * cb;
    double perp = xc * cb + yc * sb;
    out->rho_h = sqrt(along * along + perp * perp);
    double sx = -g->dso * sb, sy = g->dso * cb;
    double rx = xc - sx, ry = yc - sy, rn = sqrt(rx * rx + ry * ry);
    double cphi = fabs(rx / rn), sphi = fabs(ry / rn);
    out->lphi = g->dx / (cphi > sphi ? cphi : sphi);
}

/* F_s(c) = (1/ds) * integral over channel c of the trapezoid */
static double Fs(const or_geom* g, const or_trans* tr, int c) {
    double s = chan_s(g, c);
    return (trap_cdf(tr->tau, s + g->ds / 2) - trap_cdf(tr->tau, s - g->ds / 2)) / g->ds;
}

/* Axial rect footprint [t-, t+] of voxel iz for source height zs */
static void axial_rect(const or_geom* g, const or_trans* tr, double zj, double zs,
                       double* tm, double* tp, double* lth) {
    double mag = g->dsd / tr->rho_h;
    *tm = (zj - g->dz / 2 - zs) * mag;
    *tp = (zj + g->dz / 2 - zs) * mag;
    double tz = (zj - zs) / tr->rho_h;
    *lth = sqrt(1.0 + tz * tz);
}

static double Ft(const or_geom* g, double tm, double tp, int r) {
    double lo = row_t(g, r) - g->dt / 2, hi = lo + g->dt;
    double a = tm > lo ? tm : lo, b = tp < hi ? tp : hi;
    return b > a ? (b - a) / g->dt : 0.0;
}

/* a_ij for one (voxel, cell); exported for brute-force tests */
double or_weight(const or_geom* g, int v, int ix, int iy, int iz, int r, int c) {
    or_trans tr;
    double beta = or_view_angle(g, v);
    transaxial(g, beta, vox_x(g, ix), vox_y(g, iy), &tr);
    double fs = Fs(g, &tr, c);
    if (g->kind == OR_FAN2D) return tr.lphi * fs;
    double tm, tp, lth;
    axial_rect(g, &tr, vox_z(g, iz), or_source_z(g, v), &tm, &tp, &lth);
    return tr.lphi * lth * fs * Ft(g, tm, tp, r);
}

/* transaxial footprint data for tests: tau[4], lphi, rho_h */
void or_transaxial(const or_geom* g, int v, int ix, int iy, double* out6) {
    or_trans tr;
    transaxial(g, or_view_angle(g, v), vox_x(g, ix), vox_y(g, iy), &tr);
    for (int k = 0; k < 4; k++) out6[k] = tr.tau[k];
    out6[4] = tr.lphi;
    out6[5] = tr.rho_h;
}

/* Channel range [c0,c1] whose bins intersect [t0,t3] (possibly empty). */
static void chan_range(const or_geom* g, const or_trans* tr, int* c0, int* c1) {
    double base = -(g->ns - 1) / 2.0 - g->offs;
    int a = (int)floor(tr->tau[0] / g->ds - base - 0.5) - 1;
    int b = (int)floor(tr->tau[3] / g->ds - base + 0.5) + 1;
    if (a < 0) a = 0;
    if (b > g->ns - 1) b = g->ns - 1;
    *c0 = a;
    *c1 = b;
}

static int nzv(const or_geom* g) { return g->kind == OR_FAN2D ? 1 : g->nz; }
static int ntv(const or_geom* g) { return g->kind == OR_FAN2D ? 1 : g->nt; }

/* Loop bounds only (no arithmetic): the detector rows [r0, r1] whose bins can intersect
 * the axial rect [tm, tp], widened by one row on each side; every row outside has
 * Ft = 0 exactly, and the loops still test Ft != 0, so the sums are term-for-term (and
 * bit-for-bit) those of a loop over all rows. */
static void row_range(const or_geom* g, double tm, double tp, int* r0, int* r1) {
    double base = -(g->nt - 1) / 2.0 - g->offt;
    int a = (int)floor(tm / g->dt - base - 0.5) - 1;
    int b = (int)floor(tp / g->dt - base + 0.5) + 1;
    *r0 = a < 0 ? 0 : a;
    *r1 = b > g->nt - 1 ? g->nt - 1 : b;
}

/* Loop bounds only: the slices whose axial rect (at the column's magnification) can meet
 * the detector rows, widened by one slice on each side; for every slice outside, all Ft
 * are 0 (same remark as row_range). */
static void slice_range(const or_geom* g, const or_trans* tr, double zs, int* z0, int* z1) {
    if (g->kind == OR_FAN2D) { *z0 = 0; *z1 = 0; return; }
    double mag = g->dsd / tr->rho_h;
    double t_lo = row_t(g, 0) - g->dt / 2, t_hi = row_t(g, g->nt - 1) + g->dt / 2;
    double za = zs + t_lo / mag - g->dz / 2, zb = zs + t_hi / mag + g->dz / 2;
    double ia = (za - g->offz) / g->dz + (g->nz - 1) / 2.0, ib = (zb - g->offz) / g->dz + (g->nz - 1) / 2.0;
    int a = (int)floor(ia) - 1, b = (int)ceil(ib) + 1;
    *z0 = a < 0 ? 0 : a;
    *z1 = b > g->nz - 1 ? g->nz - 1 : b;
}

/* Loop bound only: 0 if no voxel of the volume can meet the detector rows from a source at
 * height zs (helical scans; every a_ij of the view is then exactly 0 and the view's terms
 * are skipped), 1 otherwise.  Any voxel's magnification lies in [dsd/(dso + rmax),
 * dsd/(dso - rmax)] (rmax >= in-plane distance of any voxel centre from the axis), so its
 * axial rect can only meet [t_lo, t_hi] if its z-extent meets zs + [t_lo, t_hi] / mag; the
 * test is widened by one slice on each side. */
static int view_sees_volume(const or_geom* g, double zs) {
    if (g->kind != OR_CONE_HELICAL) return 1;
    double hx = 0.5 * (g->nx - 1) * g->dx + fabs(g->offx) + g->dx;
    double hy = 0.5 * (g->ny - 1) * g->dy + fabs(g->offy) + g->dy;
    double rmax = sqrt(hx * hx + hy * hy);
    if (rmax >= g->dso) return 1;
    double mlo = g->dsd / (g->dso + rmax), mhi = g->dsd / (g->dso - rmax);
    double t_lo = row_t(g, 0) - g->dt / 2, t_hi = row_t(g, g->nt - 1) + g->dt / 2;
    double a = fmin(t_lo / mlo, t_lo / mhi), b = fmax(t_hi / mlo, t_hi / mhi);
    double zlo = vox_z(g, 0) - g->dz / 2, zhi = vox_z(g, g->nz - 1) + g->dz / 2;
    return (zlo - g->dz < zs + b) && (zhi + g->dz > zs + a);
}

/* Forward projection  p[k][r][c] = sum_j a_{(v_k,r,c), j} x_j  over views
 * v_k = first + k*stride, k < count.  x may be masked by mask (NULL = all). */
void or_fwd(const or_geom* g, int first, int stride, int count, const double* x, double* p) {
    int NZ = nzv(g), NT = ntv(g);
    size_t cells = (size_t)NT * g->ns;
#pragma omp parallel for schedule(dynamic, 1)
    for (int k = 0; k < count; k++) {
        int v = first + k * stride;
        double* pv = p + (size_t)k * cells;
        memset(pv, 0, cells * sizeof(double));
        double beta = or_view_angle(g, v), zs = or_source_z(g, v);
        if (!view_sees_volume(g, zs)) continue;
        for (int iy = 0; iy < g->ny; iy++)
            for (int ix = 0; ix < g->nx; ix++) {
                or_trans tr;
                transaxial(g, beta, vox_x(g, ix), vox_y(g, iy), &tr);
                int c0, c1;
                chan_range(g, &tr, &c0, &c1);
                int z0, z1;
                slice_range(g, &tr, zs, &z0, &z1);
                if (c1 < c0) continue;
                /* F_s of the column's channels; slices outer, channels inner: every cell
                 * (r, c) still receives its terms in increasing iz (column by column), the
                 * same order as with channels outer, so the sums are bit-identical */
                double fsv[c1 - c0 + 1];
                for (int c = c0; c <= c1; c++) fsv[c - c0] = Fs(g, &tr, c);
                for (int iz = z0; iz <= z1; iz++) {
                    double xv = x[((size_t)iz * g->ny + iy) * g->nx + ix];
                    if (xv == 0.0) continue;
                    if (g->kind == OR_FAN2D) {
                        for (int c = c0; c <= c1; c++) {
                            double fs = fsv[c - c0];
                            if (fs == 0.0) continue;
                            pv[c] += tr.lphi * fs * xv;
                        }
                        continue;
                    }
                    double tm, tp, lth;
                    int r0, r1;
                    axial_rect(g, &tr, vox_z(g, iz), zs, &tm, &tp, &lth);
                    row_range(g, tm, tp, &r0, &r1);
                    for (int c = c0; c <= c1; c++) {
                        double fs = fsv[c - c0];
                        if (fs == 0.0) continue;
                        for (int r = r0; r <= r1; r++) {
                            double ft = Ft(g, tm, tp, r);
                            if (ft != 0.0) pv[(size_t)r * g->ns + c] += tr.lphi * lth * fs * ft * xv;
                        }
                    }
                }
            }
    }
}

/* Back projection  x_j = sum_i a_ij p_i  (exact adjoint of or_fwd). */
void or_back(const or_geom* g, int first, int stride, int count, const double* p, double* x) {
    int NZ = nzv(g), NT = ntv(g);
    size_t cells = (size_t)NT * g->ns;
#pragma omp parallel for schedule(dynamic, 1)
    for (int iy = 0; iy < g->ny; iy++)
        for (int ix = 0; ix < g->nx; ix++) {
            for (int iz = 0; iz < NZ; iz++) x[((size_t)iz * g->ny + iy) * g->nx + ix] = 0.0;
            for (int k = 0; k < count; k++) {
                int v = first + k * stride;
                const double* pv = p + (size_t)k * cells;
                double beta = or_view_angle(g, v), zs = or_source_z(g, v);
                if (!view_sees_volume(g, zs)) continue;
                or_trans tr;
                transaxial(g, beta, vox_x(g, ix), vox_y(g, iy), &tr);
                int c0, c1;
                chan_range(g, &tr, &c0, &c1);
                int z0, z1;
                slice_range(g, &tr, zs, &z0, &z1);
                if (c1 < c0) continue;
                /* slices outer, channels inner: every x[iz] still receives its terms in
                 * increasing c (view by view), as with channels outer: bit-identical sums */
                double fsv[c1 - c0 + 1];
                for (int c = c0; c <= c1; c++) fsv[c - c0] = Fs(g, &tr, c);
                for (int iz = z0; iz <= z1; iz++) {
                    double tm = 0.0, tp = 0.0, lth = 1.0;
                    int r0 = 0, r1 = -1;
                    if (g->kind != OR_FAN2D) {
                        axial_rect(g, &tr, vox_z(g, iz), zs, &tm, &tp, &lth);
                        row_range(g, tm, tp, &r0, &r1);
                    }
                    for (int c = c0; c <= c1; c++) {
                        double fs = fsv[c - c0];
                        if (fs == 0.0) continue;
                        double acc = 0.0;
                        if (g->kind == OR_FAN2D) {
                            acc = tr.lphi * fs * pv[c];
                        } else {
                            for (int r = r0; r <= r1; r++) {
                                double ft = Ft(g, tm, tp, r);
                                if (ft != 0.0) acc += tr.lphi * lth * fs * ft * pv[(size_t)r * g->ns + c];
                            }
                        }
                        x[((size_t)iz * g->ny + iy) * g->nx + ix] += acc;
                    }
                }
            }
        }
}

/* U = number of (view, voxel in mask) pairs with a non-empty footprint
 * (SURVEY §8d metric definition), over views first + k*stride. */
long long or_count_vv(const or_geom* g, int first, int stride, int count, const uint8_t* mask) {
    int NZ = nzv(g);
    double s_lo = chan_s(g, 0) - g->ds / 2, s_hi = chan_s(g, g->ns - 1) + g->ds / 2;
    double t_lo = row_t(g, 0) - g->dt / 2, t_hi = row_t(g, ntv(g) - 1) + g->dt / 2;
    long long total = 0;
#pragma omp parallel for reduction(+ : total) schedule(dynamic, 1)
    for (int k = 0; k < count; k++) {
        int v = first + k * stride;
        double beta = or_view_angle(g, v), zs = or_source_z(g, v);
        for (int iy = 0; iy < g->ny; iy++)
            for (int ix = 0; ix < g->nx; ix++) {
                or_trans tr;
                transaxial(g, beta, vox_x(g, ix), vox_y(g, iy), &tr);
                double a = tr.tau[0] > s_lo ? tr.tau[0] : s_lo, b = tr.tau[3] < s_hi ? tr.tau[3] : s_hi;
                if (!(b > a)) continue;
                for (int iz = 0; iz < NZ; iz++) {
                    if (mask && !mask[((size_t)iz * g->ny + iy) * g->nx + ix]) continue;
                    if (g->kind != OR_FAN2D) {
                        double tm, tp, lth;
                        axial_rect(g, &tr, vox_z(g, iz), zs, &tm, &tp, &lth);
                        double ta = tm > t_lo ? tm : t_lo, tb = tp < t_hi ? tp : t_hi;
                        if (!(tb > ta)) continue;
                    }
                    total++;
                }
            }
    }
    return total;
}

/* ---------------- O4: SQS denominator ---------------- */

/* D_L = A'(W (A 1_S)) over all views; S <- S and {D_L > 0}; D_L := 0 off S. */
void or_sqs_denom(const or_geom* g, const double* w, uint8_t* mask, double* dl) {
    size_t N = (size_t)nzv(g) * g->ny * g->nx;
    size_t cells = (size_t)g->na * ntv(g) * g->ns;
    double* one = (double*)malloc(N * sizeof(double));
    double* p = (double*)malloc(cells * sizeof(double));
    for (size_t j = 0; j < N; j++) one[j] = mask[j] ? 1.0 : 0.0;
    or_fwd(g, 0, 1, g->na, one, p);
    for (size_t i = 0; i < cells; i++) p[i] *= w[i];
    or_back(g, 0, 1, g->na, p, dl);
    for (size_t j = 0; j < N; j++) {
        if (!(mask[j] && dl[j] > 0.0)) {
            mask[j] = 0;
            dl[j] = 0.0;
        }
    }
    free(one);
    free(p);
}

/* ---------------- O5: Fair regulariser ---------------- */
/* psi(t) = delta^2 (|t|/delta - ln(1 + |t|/delta));  psi'(t) = t / (1 + |t|/delta);
 * omega(t) = 1 / (1 + |t|/delta)  (Huber curvature, G14).
 * R(x) = beta sum_{unordered pairs {j,k} in S, k in N(j)} w_jk psi(x_j - x_k),
 * w_jk = 1 / ||offset||; N = 8-neighbourhood in-plane (nbr = 8) or 26 in 3D. */

static double fair_psi(double t, double d) { double a = fabs(t) / d; return d * d * (a - log1p(a)); }

static int nbr_ok(const or_geom* g, int nbr, int oz) { return !(nbr == 8 && oz != 0) && !(nzv(g) == 1 && oz != 0); }

double or_reg_value(const or_geom* g, double beta, double delta, int nbr, const uint8_t* mask, const double* x) {
    int NZ = nzv(g);
    double total = 0.0;
    for (int iz = 0; iz < NZ; iz++)
        for (int iy = 0; iy < g->ny; iy++)
            for (int ix = 0; ix < g->nx; ix++) {
                size_t j = ((size_t)iz * g->ny + iy) * g->nx + ix;
                if (!mask[j]) continue;
                for (int oz = -1; oz <= 1; oz++)
                    for (int oy = -1; oy <= 1; oy++)
                        for (int ox = -1; ox <= 1; ox++) {
                            if (!nbr_ok(g, nbr, oz) || (ox == 0 && oy == 0 && oz == 0)) continue;
                            int kx = ix + ox, ky = iy + oy, kz = iz + oz;
                            if (kx < 0 || ky < 0 || kz < 0 || kx >= g->nx || ky >= g->ny || kz >= NZ) continue;
                            size_t k = ((size_t)kz * g->ny + ky) * g->nx + kx;
                            if (k <= j || !mask[k]) continue; /* each unordered pair once */
                            double w = 1.0 / sqrt((double)(ox * ox + oy * oy + oz * oz));
                            total += w * fair_psi(x[j] - x[k], delta);
                        }
            }
    return beta * total;
}

void or_reg_grad(const or_geom* g, double beta, double delta, int nbr, const uint8_t* mask, const double* x,
                 double* grad, double* curv) {
    int NZ = nzv(g);
#pragma omp parallel for
    for (int iz = 0; iz < NZ; iz++)
        for (int iy = 0; iy < g->ny; iy++)
            for (int ix = 0; ix < g->nx; ix++) {
                size_t j = ((size_t)iz * g->ny + iy) * g->nx + ix;
                double gr = 0.0, cu = 0.0;
                if (mask[j]) {
                    for (int oz = -1; oz <= 1; oz++)
                        for (int oy = -1; oy <= 1; oy++)
                            for (int ox = -1; ox <= 1; ox++) {
                                if (!nbr_ok(g, nbr, oz) || (ox == 0 && oy == 0 && oz == 0)) continue;
                                int kx = ix + ox, ky = iy + oy, kz = iz + oz;
                                if (kx < 0 || ky < 0 || kz < 0 || kx >= g->nx || ky >= g->ny || kz >= NZ) continue;
                                size_t k = ((size_t)kz * g->ny + ky) * g->nx + kx;
                                if (!mask[k]) continue;
                                double w = 1.0 / sqrt((double)(ox * ox + oy * oy + oz * oz));
                                double t = x[j] - x[k];
                                double om = 1.0 / (1.0 + fabs(t) / delta);
                                gr += w * t * om;
                                cu += w * om;
                            }
                }
                grad[j] = beta * gr;
                if (curv) curv[j] = 2.0 * beta * cu;
            }
}

/* ---------------- O6: cost ---------------- */
double or_cost(const or_geom* g, const double* y, const double* w, double beta, double delta, int nbr,
               const uint8_t* mask, const double* x) {
    size_t cells = (size_t)g->na * ntv(g) * g->ns;
    double* p = (double*)malloc(cells * sizeof(double));
    or_fwd(g, 0, 1, g->na, x, p);
    double d = 0.0;
    for (size_t i = 0; i < cells; i++) d += 0.5 * w[i] * (p[i] - y[i]) * (p[i] - y[i]);
    free(p);
    return d + or_reg_value(g, beta, delta, nbr, mask, x);
}

/* ---------------- O7: OS-LALM ---------------- */

/* Bit-reversal visiting order (pad to 2^ceil(log2 M), drop >= M, G11). */
void or_bit_reversal(int M, int* order) {
    int bits = 0;
    while ((1 << bits) < M) bits++;
    int n = 0;
    for (int i = 0; i < (1 << bits); i++) {
        int r = 0;
        for (int b = 0; b < bits; b++)
            if (i & (1 << b)) r |= 1 << (bits - 1 - b);
        if (r < M) order[n++] = r;
    }
}

/* rho_l (eq. rho_l_formula_qp): 1 if l = 0, else
 * max{ pi/(l+1) sqrt(1 - (pi/(2l+2))^2), rho_min }. */
double or_rho_l(long l, double rho_min) {
    if (l == 0) return 1.0;
    double a = M_PI / (l + 1.0), b = M_PI / (2.0 * l + 2.0);
    double r = a * sqrt(1.0 - b * b);
    return r > rho_min ? r : rho_min;
}

/* G = M * A_m'(W (A_m x - y)) for subset m (views v = m mod M). */
static void subset_grad(const or_geom* g, int M, int m, const double* y, const double* w, const double* x,
                        double* G, double* pbuf) {
    int count = (g->na - m + M - 1) / M;
    size_t cells = (size_t)ntv(g) * g->ns;
    or_fwd(g, m, M, count, x, pbuf);
    for (int k = 0; k < count; k++) {
        size_t off = (size_t)(m + k * M) * cells;
        for (size_t i = 0; i < cells; i++) {
            size_t q = (size_t)k * cells + i;
            pbuf[q] = M * w[off + i] * (pbuf[q] - y[off + i]);
        }
    }
    or_back(g, m, M, count, pbuf, G);
}

/* Exported for tests: M * A_m'(W (A_m x - y)). */
void or_subset_grad(const or_geom* g, int M, int m, const double* y, const double* w, const double* x,
                    double* G) {
    size_t cells = (size_t)ntv(g) * g->ns;
    int count = (g->na - m + M - 1) / M;
    double* pbuf = (double*)malloc((size_t)count * cells * sizeof(double));
    subset_grad(g, M, m, y, w, x, G, pbuf);
    free(pbuf);
}

/*
 * Inner constrained denoising by n warm-started FISTA iterations ("we solve this
 * inner constrained denoising problem using n iterations of ... FISTA ... starting from
 * the previous update as a warm start"; NEXT-1 reading in DESIGN.md):
 *   minimise  phi(x) = R(x) + (rho/2) ||x - z||^2_{D_L}  over x >= 0 (x = 0 off S),
 *   z = xk - s / (rho D_L),  grad f(v) = grad R(v) + rho D_L (v - xk) + s,
 * with the fixed diagonal Lipschitz metric P = rho D_L + 2 beta sum_{k in N(j) & S} w_jk
 * (Fair: psi'' <= 1) and Beck-Teboulle momentum:
 *   v0 = x0 = xk, t0 = 1;  x_i = max(0, v_{i-1} - P^-1 grad f(v_{i-1}));
 *   t_i = (1 + sqrt(1 + 4 t_{i-1}^2)) / 2;  v_i = x_i + ((t_{i-1} - 1)/t_i)(x_i - x_{i-1}).
 * s is the search direction rho G + (1 - rho) g.  Writes x_n to x_out.
 */
void or_inner_fista(const or_geom* g, double beta, double delta, int nbr, const uint8_t* mask, const double* dl,
                    double rho, const double* xk, const double* s, int n, double* x_out) {
    size_t N = (size_t)nzv(g) * g->ny * g->nx;
    int NZ = nzv(g);
    double* v = (double*)malloc(N * sizeof(double));
    double* xp = (double*)malloc(N * sizeof(double));
    double* xn = (double*)malloc(N * sizeof(double));
    double* gr = (double*)malloc(N * sizeof(double));
    double* P = (double*)malloc(N * sizeof(double));
    /* Lipschitz metric: rho D_L + 2 beta sum of neighbour weights inside S */
    for (int iz = 0; iz < NZ; iz++)
        for (int iy = 0; iy < g->ny; iy++)
            for (int ix = 0; ix < g->nx; ix++) {
                size_t j = ((size_t)iz * g->ny + iy) * g->nx + ix;
                double sw = 0.0;
                if (mask[j])
                    for (int oz = -1; oz <= 1; oz++)
                        for (int oy = -1; oy <= 1; oy++)
                            for (int ox = -1; ox <= 1; ox++) {
                                if (!nbr_ok(g, nbr, oz) || (ox == 0 && oy == 0 && oz == 0)) continue;
                                int kx = ix + ox, ky = iy + oy, kz = iz + oz;
                                if (kx < 0 || ky < 0 || kz < 0 || kx >= g->nx || ky >= g->ny || kz >= NZ) continue;
                                size_t k = ((size_t)kz * g->ny + ky) * g->nx + kx;
                                if (mask[k]) sw += 1.0 / sqrt((double)(ox * ox + oy * oy + oz * oz));
                            }
                P[j] = rho * dl[j] + 2.0 * beta * sw;
            }
    memcpy(v, xk, N * sizeof(double));
    memcpy(xp, xk, N * sizeof(double));
    double t = 1.0;
    for (int i = 1; i <= n; i++) {
        or_reg_grad(g, beta, delta, nbr, mask, v, gr, NULL);
        for (size_t j = 0; j < N; j++) {
            if (!mask[j]) { xn[j] = 0.0; continue; }
            double grad = gr[j] + rho * dl[j] * (v[j] - xk[j]) + s[j];
            double val = v[j] - grad / P[j];
            xn[j] = val > 0.0 ? val : 0.0;
        }
        double tn = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t));
        double mom = (t - 1.0) / tn;
        for (size_t j = 0; j < N; j++) {
            v[j] = xn[j] + mom * (xn[j] - xp[j]);
            xp[j] = xn[j];
        }
        t = tn;
    }
    memcpy(x_out, xp, N * sizeof(double));
    free(v); free(xp); free(xn); free(gr); free(P);
}

/*
 * OS-LALM run:
 *   x <- x0 (caller, 0 on S); G <- M A_{pi0}'(W(A x - y)); g <- G; l <- 0
 *   for k = 1..K, j = 0..M-1:
 *     rho <- FIXED ? rho_fixed : rho_l(l)
 *     x <- max(0, x - (rho G + (1-rho) g + gradR(x)) / (rho D_L + D_R(x)))   on S, 0 off S
 *     [if trailing == 0 and last step: stop]
 *     G+ <- M A_{pi[(j+1)%M]}'(W(A x - y))
 *     xi <- sum_S (g - G+)(G+ - G);  g <- (rho G+ + g)/(1 + rho);  G <- G+
 *     CONTINUATION: l <- (xi > 0) ? 0 : l + 1
 * mode 0 = FIXED, 1 = CONTINUATION.  trailing = 1 also computes the final
 * projection pair (so the state is ready for another iteration; x unchanged).
 * log (nullable) receives per inner step: rho, xi, restart flag (3 doubles).
 * g_out, G_out (nullable) receive the final split gradient and subset gradient.
 *
 * bb = 1: Barzilai-Borwein scaling (NEXT-2, supplement P:1472-1492).  The SQS
 * Hessian L_diag = D_L is replaced by H_k = alpha_k D_L, with alpha_k fitting the secant
 * equation y_k ~ H_k s_k in the L_diag^{-1}-weighted least-squares sense subject to
 * alpha <= 1 (eq. scale_factor_alpha_k):
 *     alpha_k = min(1, max(alpha_min, (y_k' s_k) / (s_k' D_L s_k)))   (sums over S),
 *     s_k = x^k - x^{k-1},  y_k = grad l(x^k) - grad l(x^{k-1}).
 * OS reading (DESIGN.md B-BB): k counts outer iterations; grad l is approximated by the
 * mean gbar_k of the M subset gradients M grad l_m computed during iteration k, and the
 * secant pair uses the points where those gradients were evaluated: s_k = xbar_k -
 * xbar_{k-1}, xbar_k = mean of the M inner iterates x^{k,j} (the image after inner step j,
 * at which the next subset gradient is computed), y_k = gbar_k - gbar_{k-1}.  With M = 1
 * xbar_k = x^k (the paper's s_k).  (Pairing gbar_k with the end point x^k instead makes
 * y_k's' <= 0 common with OS and collapses the iteration.)  alpha = 1 for iterations 1
 * and 2 (no secant pair yet); alpha_k (from iterations k-1, k) is used in iteration k + 1.
 * alpha_log (nullable) receives the alpha used in each outer iteration.
 */
void or_oslalm_run(const or_geom* g, const double* y, const double* w, const double* dl, const uint8_t* mask,
                   int M, int mode, double rho_fixed, double rho_min, double beta, double delta, int nbr,
                   int n_iter, int trailing, double* x, double* log, double* g_out, double* G_out, int inner,
                   int n_inner, int bb, double alpha_min, double* alpha_log) {
    size_t N = (size_t)nzv(g) * g->ny * g->nx;
    size_t cells = (size_t)ntv(g) * g->ns;
    int maxcount = (g->na + M - 1) / M;
    int* order = (int*)malloc(M * sizeof(int));
    or_bit_reversal(M, order);
    double* G = (double*)malloc(N * sizeof(double));
    double* Gp = (double*)malloc(N * sizeof(double));
    double* sg = (double*)malloc(N * sizeof(double));
    double* gr = (double*)malloc(N * sizeof(double));
    double* cu = (double*)malloc(N * sizeof(double));
    double* pbuf = (double*)malloc((size_t)maxcount * cells * sizeof(double));
    for (size_t j = 0; j < N; j++)
        if (!mask[j]) x[j] = 0.0;
    subset_grad(g, M, order[0], y, w, x, G, pbuf);
    memcpy(sg, G, N * sizeof(double));
    long l = 0;
    int step = 0;
    /* Barzilai-Borwein state: H = alpha D_L (alpha = 1: the plain SQS Hessian) */
    double alpha = 1.0;
    double* hd = (double*)malloc(N * sizeof(double));        /* alpha D_L */
    double* xprev = bb ? (double*)malloc(N * sizeof(double)) : NULL;   /* xbar_{k-1} */
    double* xbar = bb ? (double*)calloc(N, sizeof(double)) : NULL;
    double* gbar = bb ? (double*)calloc(N, sizeof(double)) : NULL;
    double* gprev = bb ? (double*)malloc(N * sizeof(double)) : NULL;
    for (int k = 1; k <= n_iter; k++) {
        for (size_t q = 0; q < N; q++) hd[q] = alpha * dl[q];
        if (alpha_log) alpha_log[k - 1] = alpha;
        for (int j = 0; j < M; j++, step++) {
            double rho = mode == 0 ? rho_fixed : or_rho_l(l, rho_min);
            if (inner == 0) {
                /* n = 1 SQS step with the Huber curvature of R at x (reading G14) */
                or_reg_grad(g, beta, delta, nbr, mask, x, gr, cu);
                for (size_t q = 0; q < N; q++) {
                    if (!mask[q]) { x[q] = 0.0; continue; }
                    double s = rho * G[q] + (1.0 - rho) * sg[q];
                    double xn = x[q] - (s + gr[q]) / (rho * hd[q] + cu[q]);
                    x[q] = xn > 0.0 ? xn : 0.0;
                }
            } else {
                /* n warm-started FISTA iterations on the inner problem (NEXT-1) */
                for (size_t q = 0; q < N; q++) cu[q] = rho * G[q] + (1.0 - rho) * sg[q];   /* s */
                memcpy(gr, x, N * sizeof(double));                                         /* x_k */
                or_inner_fista(g, beta, delta, nbr, mask, hd, rho, gr, cu, n_inner, x);
            }
            if (log) { log[3 * step] = rho; log[3 * step + 1] = 0.0; log[3 * step + 2] = 0.0; }
            if (!trailing && k == n_iter && j == M - 1) break;
            subset_grad(g, M, order[(j + 1) % M], y, w, x, Gp, pbuf);
            double xi = 0.0;
            for (size_t q = 0; q < N; q++)
                if (mask[q]) xi += (sg[q] - Gp[q]) * (Gp[q] - G[q]);
            for (size_t q = 0; q < N; q++) {
                sg[q] = (rho * Gp[q] + sg[q]) / (1.0 + rho);
                G[q] = Gp[q];
            }
            int restart = xi > 0.0;
            if (mode == 1) l = restart ? 0 : l + 1;
            if (log) { log[3 * step + 1] = xi; log[3 * step + 2] = restart; }
            if (bb)
                for (size_t q = 0; q < N; q++) {
                    gbar[q] += G[q] / M;   /* mean of the iteration's M grad l_m ... */
                    xbar[q] += x[q] / M;   /* ... and of the points they were evaluated at */
                }
        }
        if (bb && step < n_iter * M) {   /* end of outer iteration k (completed) */
            if (k >= 2) {
                double num = 0.0, den = 0.0;
                for (size_t q = 0; q < N; q++)
                    if (mask[q]) {
                        double sq = xbar[q] - xprev[q];
                        num += (gbar[q] - gprev[q]) * sq;
                        den += dl[q] * sq * sq;
                    }
                double a = den > 0.0 ? num / den : 1.0;
                alpha = a > 1.0 ? 1.0 : (a < alpha_min ? alpha_min : a);
            }
            memcpy(xprev, xbar, N * sizeof(double));
            memcpy(gprev, gbar, N * sizeof(double));
            memset(gbar, 0, N * sizeof(double));
            memset(xbar, 0, N * sizeof(double));
        }
    }
    if (g_out) memcpy(g_out, sg, N * sizeof(double));
    if (G_out) memcpy(G_out, G, N * sizeof(double));
    free(order); free(G); free(Gp); free(sg); free(gr); free(cu); free(pbuf); free(hd);
    free(xprev); free(xbar); free(gbar); free(gprev);
}

/* ---------------- NEXT-4: FBP / FDK initial image ---------------- */
/*
 * Filtered back-projection for the initial image x^0 ("initialized with a
 * standard filtered back-projection (FBP) reconstruction"; the paper does not say
 * which FBP — reading B-FBP in DESIGN.md: the textbook full-scan equiangular
 * fan-beam FBP (Kak & Slaney, eqs. 3.4.1), with the FDK cone-beam extension for a
 * cylindrical detector on a circular orbit):
 *   R'(gamma_k, t) = R(gamma_k, t) * D cos(gamma_k) * D / sqrt(D^2 + zeta^2),
 *                    zeta = t dso/dsd (row height at the rotation axis; 1 in 2D)
 *   Q(gamma_n, t)  = tau * sum_k R'(gamma_k, t) g((n - k) tau)     (row-wise)
 *   g(n tau)       = 1/(8 tau^2) (n = 0), 0 (n even), -1/(2 pi^2 sin^2(n tau)) (n odd)
 *   f(p)           = dbeta * sum_v Q_v(gamma(p), t(p)) / L(p)^2
 * with D = dso, tau = ds/dsd the angular channel pitch, L the in-plane source-voxel
 * distance, gamma(p) / t(p) the fan angle / detector row height of the voxel centre
 * (O1), linear interpolation in gamma and t (0 outside the detector), dbeta = 2 pi / na.
 * Helical scans (P:573, P:586 and P:1495 start the helical reconstructions from "the initial
 * FBP image"; which FBP is not said -- reading B-FBP-H in DESIGN.md): the same row-wise
 * filtering, and a voxel-driven back-projection over the views whose cone sees the voxel
 * (projected row coordinate inside [0, nt-1]), normalised by their number:
 *   f(p) = 2 pi * sum_{v seen} Q_v(gamma(p), t(p)) / L(p)^2 / #{v seen}
 * (with every view seen this is the circular-orbit formula, dbeta = 2 pi / na).
 * Returns 0, or -1 for a circular orbit that is not one full turn.
 */
int or_fbp(const or_geom* g, const double* p, double* x) {
    const int helical = g->kind == OR_CONE_HELICAL;
    if (!helical && fabs(g->orbit_deg - 360.0) > 1e-9) return -1;
    int NT = ntv(g), NZ = nzv(g);
    double D = g->dso, tau = g->ds / g->dsd;
    int ns = g->ns;
    size_t cells = (size_t)NT * ns;
    double* q = (double*)malloc((size_t)g->na * cells * sizeof(double));
    double* gk = (double*)malloc((2 * (size_t)ns - 1) * sizeof(double));
    for (int n = -(ns - 1); n <= ns - 1; n++) {
        double v;
        if (n == 0) v = 1.0 / (8.0 * tau * tau);
        else if (n % 2 == 0) v = 0.0;
        else { double s = sin(n * tau); v = -1.0 / (2.0 * M_PI * M_PI * s * s); }
        gk[n + ns - 1] = v;
    }
#pragma omp parallel for schedule(dynamic)
    for (int v = 0; v < g->na; v++) {
        double* rp = (double*)malloc((size_t)ns * sizeof(double));
        for (int r = 0; r < NT; r++) {
            double zeta = g->kind == OR_FAN2D ? 0.0 : row_t(g, r) * g->dso / g->dsd;
            for (int k = 0; k < ns; k++) {
                double gam = chan_s(g, k) / g->dsd;
                rp[k] = p[((size_t)v * NT + r) * ns + k] * D * cos(gam) * D / sqrt(D * D + zeta * zeta);
            }
            for (int n = 0; n < ns; n++) {
                double acc = 0.0;
                for (int k = 0; k < ns; k++) acc += rp[k] * gk[n - k + ns - 1];
                q[((size_t)v * NT + r) * ns + n] = tau * acc;
            }
        }
        free(rp);
    }
    double dbeta = 2.0 * M_PI / g->na;
    double c0 = (ns - 1) / 2.0 + g->offs, r0 = (NT - 1) / 2.0 + g->offt;
#pragma omp parallel for schedule(dynamic)
    for (int iy = 0; iy < g->ny; iy++)
        for (int iz = 0; iz < NZ; iz++)
            for (int ix = 0; ix < g->nx; ix++) {
                double xc = vox_x(g, ix), yc = vox_y(g, iy), zc = vox_z(g, iz), acc = 0.0;
                long long seen = 0;
                for (int v = 0; v < g->na; v++) {
                    double b = or_view_angle(g, v), sb = sin(b), cb = cos(b);
                    double along = D + xc * sb - yc * cb, perp = xc * cb + yc * sb;
                    double L2 = along * along + perp * perp;
                    double uc = atan2(perp, along) / tau + c0;         /* channel coordinate */
                    double ur = g->kind == OR_FAN2D ? 0.0 : (zc - or_source_z(g, v)) * g->dsd / sqrt(L2) / g->dt + r0;
                    if (helical) {
                        if (!(ur >= 0.0 && ur <= NT - 1)) continue;   /* the view does not see the voxel */
                        seen++;
                    }
                    int k0 = (int)floor(uc), r0i = (int)floor(ur);
                    double fk = uc - k0, fr = ur - r0i, val = 0.0;
                    for (int a = 0; a < 2; a++)
                        for (int bq = 0; bq < (NT > 1 ? 2 : 1); bq++) {
                            int k = k0 + a, r = NT > 1 ? r0i + bq : 0;
                            if (k < 0 || k >= ns || r < 0 || r >= NT) continue;
                            double wk = a ? fk : 1.0 - fk, wr = NT > 1 ? (bq ? fr : 1.0 - fr) : 1.0;
                            val += wk * wr * q[((size_t)v * NT + r) * ns + k];
                        }
                    acc += val / L2;
                }
                x[((size_t)iz * g->ny + iy) * g->nx + ix] =
                    helical ? (seen ? 2.0 * M_PI * acc / (double)seen : 0.0) : dbeta * acc;
            }
    free(q);
    free(gk);
    return 0;
}
