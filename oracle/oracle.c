/*
 * oracle/oracle.c -- CPU binary64 ORACLE for the SUPRA DAS -> B-mode hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product (paper_1711_06127_b200/, libsupra_bf.so) never links, imports
 * or calls it, and this file shares no code, header, table or constant
 * generator with the CUDA path.
 *
 * Plain, slow, obviously correct: scalar loops in the order the definitions
 * are written, IEEE binary64 throughout, compiled with -O2 -ffp-contract=off
 * against glibc libm.  Citations: P:n = /root/reference/PAPER.md line n,
 * S:n = /root/reference/SPEC.md line n, SURVEY = SURVEY.md section 8(c)
 * (the readings listed in DESIGN.md "Readings").
 *
 * Parity pins: every function below is pinned by a `-m "not gpu"` test in
 * tests/test_oracle_*.py (closed forms, invariants, special cases, brute
 * force).  None is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

enum { ORA_WIN_RECT = 0, ORA_WIN_HANN = 1, ORA_WIN_HAMMING = 2 };
enum { ORA_NORM_COUNT = 0, ORA_NORM_NONE = 1 };
enum { ORA_SC_LINEAR_2D = 0, ORA_SC_SECTOR_2D = 1, ORA_SC_PYRAMID_3D = 2 };

/* ------------------------------------------------------------------ */
/* Geometry.  Element (i,j) sits at ((i-(Nx-1)/2)*px, (j-(Ny-1)/2)*py, 0)
 * (TransducerGeometry invariant).  Channel ch = j*Nx + i (reading
 * #15).  Units: mm.                                                     */
void ora_element_positions(int nx, int ny, double px, double py, double *pos)
{
    for (int j = 0; j < ny; j++) {
        for (int i = 0; i < nx; i++) {
            int ch = j * nx + i;
            pos[3 * ch + 0] = (i - (nx - 1) / 2.0) * px;
            pos[3 * ch + 1] = (j - (ny - 1) / 2.0) * py;
            pos[3 * ch + 2] = 0.0;
        }
    }
}

/* Depth per output sample: z_k = k * c / (2 fs), in mm.  */
double ora_dr_mm(double c_mps, double fs_hz) { return 1000.0 * c_mps / (2.0 * fs_hz); }

/* Receive window over the dynamic aperture, u = rho / R in [0,1]
 * (reading #9: Hann is zero at the aperture edge).              */
static double ora_window(int kind, double u)
{
    if (kind == ORA_WIN_HANN) return 0.5 * (1.0 + cos(M_PI * u));
    if (kind == ORA_WIN_HAMMING) return 0.54 + 0.46 * cos(M_PI * u);
    return 1.0;
}

/* Zero-padded channel sample x~[i] ("out-of-range time indices
 * contribute zero"; reading #10).                                     */
static double ora_sample(const int16_t *x, long i, int S)
{
    if (i < 0 || i >= S) return 0.0;
    return (double)x[i];
}

/* Round-trip delay in samples for element position e and focal depth z on
 * the scanline (o, d):  tau = (z + |p - e|) * fs / c + t0 * fs,
 * p = o + z d  ("t_e(z_k) = (z_k + |p(z_k) - pos_e|)/c").        */
double ora_delay_samples(const double *o, const double *d, const double *e, double z_mm,
                         double fs_hz, double c_mps, double t0_s)
{
    double p0 = o[0] + z_mm * d[0];
    double p1 = o[1] + z_mm * d[1];
    double p2 = o[2] + z_mm * d[2];
    double dx = p0 - e[0], dy = p1 - e[1], dz = p2 - e[2];
    double r = sqrt(dx * dx + dy * dy + dz * dz);
    return ((z_mm + r) / 1000.0) * fs_hz / c_mps + t0_s * fs_hz;
}

typedef struct {
    int nx, ny;
    double pitch_x_mm, pitch_y_mm;
    int num_events, S;
    double fs_hz, c_mps, t0_s;
    int L;
    const double *origin_mm;   /* [L][3] */
    const double *direction;   /* [L][3] */
    const int32_t *line_event; /* [L]    */
    double f_number;
    int window, normalize;
    /* receive channel map ("only 64 channels usable"; S:102 active
     * aperture): nch = 0 -> channel ch is element ch; else raw holds nch
     * traces per event and chmap[ev*nch + ch] is the element channel ch
     * recorded (-1: unused).  The receive aperture of a line is the set of
     * elements its event recorded.                                       */
    int nch;
    const int32_t *chmap;
    /* fractional-delay lookup: 0 linear (reading #10), 1 nearest:
     * x~[floor(tau + 1/2)] (reading #32, ties round up)                  */
    int interp;
} ora_das_params;

/* Delay-and-sum with dynamic receive focusing (S:133,
 * S:153).  For line l and output sample k:
 *   z = k dr;  member(e) <=> (2F) rho_e <= k dr   (reading #6, inclusive)
 *   RF = sum_{members} w(rho/R) * ((1-f) x~[i0] + f x~[i0+1]) / N
 * with tau = i0 + f, R = z/(2F), N = #members (reading #7), 0 if N = 0.  */
static void ora_das_line(const ora_das_params *p, const double *pos, const int16_t *raw,
                         int l, double *rf)
{
    const double dr = 1000.0 * p->c_mps / (2.0 * p->fs_hz);
    const int C = p->nch > 0 ? p->nch : p->nx * p->ny;   /* traces per event */
    const int S = p->S;
    const double *o = p->origin_mm + 3 * l;
    const double *d = p->direction + 3 * l;
    const int ev = p->line_event[l];
    const int16_t *xev = raw + (size_t)ev * (size_t)C * (size_t)S;
    for (int k = 0; k < S; k++) {
        double z = k * dr;
        double sum = 0.0;
        int n = 0;
        for (int ch = 0; ch < C; ch++) {
            const int el = p->nch > 0 ? p->chmap[(size_t)ev * p->nch + ch] : ch;
            if (el < 0) continue;                 /* channel not recorded */
            const double *e = pos + 3 * el;
            double rho = hypot(e[0] - o[0], e[1] - o[1]);
            if (!((2.0 * p->f_number) * rho <= k * dr)) continue;
            n++;
            double tau = ora_delay_samples(o, d, e, z, p->fs_hz, p->c_mps, p->t0_s);
            double fl = floor(tau);
            long i0 = (long)fl;
            double f = tau - fl;
            const int16_t *x = xev + (size_t)ch * (size_t)S;
            double v = (p->interp == 1) ? ora_sample(x, (long)floor(tau + 0.5), S)
                                        : (1.0 - f) * ora_sample(x, i0, S) + f * ora_sample(x, i0 + 1, S);
            double R = z / (2.0 * p->f_number);
            double u = (R > 0.0) ? rho / R : 0.0;
            double w = ora_window(p->window, u);
            sum += w * v;
        }
        if (p->normalize == ORA_NORM_NONE) rf[k] = sum;
        else rf[k] = (n > 0) ? sum / n : 0.0;
    }
}

typedef struct {
    const ora_das_params *p;
    const double *pos;
    const int16_t *raw;
    const int32_t *lines;
    int nlines;
    double *rf;
    int t, nt;
} ora_job;

static void *ora_das_worker(void *arg)
{
    ora_job *j = (ora_job *)arg;
    for (int i = j->t; i < j->nlines; i += j->nt)
        ora_das_line(j->p, j->pos, j->raw, j->lines[i], j->rf + (size_t)i * j->p->S);
    return NULL;
}

/* Beamform the listed lines of one frame.  raw: [E][C][S] int16 (S:111,
 * time fastest).  rf: [nlines][S].  Threads split lines; every output cell
 * is computed by exactly one thread in a fixed order (deterministic).    */
int ora_das(const ora_das_params *p, const int16_t *raw, const int32_t *lines, int nlines,
            double *rf, int nthreads)
{
    const int C = p->nx * p->ny;
    double *pos = (double *)malloc(sizeof(double) * 3 * (size_t)C);
    if (!pos) return -1;
    ora_element_positions(p->nx, p->ny, p->pitch_x_mm, p->pitch_y_mm, pos);
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    ora_job jobs[256];
    for (int t = 0; t < nthreads; t++) {
        jobs[t] = (ora_job){p, pos, raw, lines, nlines, rf, t, nthreads};
        if (nthreads > 1) pthread_create(&th[t], NULL, ora_das_worker, &jobs[t]);
    }
    if (nthreads == 1) ora_das_worker(&jobs[0]);
    else for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
    free(pos);
    return 0;
}

/* ------------------------------------------------------------------ */
/* IQ demodulation low-pass: T-tap (odd) Hamming-windowed sinc with cutoff
 * fc ("windowed-sinc filter of cutoff bandwidth/2 (Hamming-windowed,
 * filter_length taps, zero-phase)"), DC gain normalised to 1 (reading #16).
 * h[j+P], j = -P..P, P = (T-1)/2.                                       */
void ora_fir_taps(int T, double fc_hz, double fs_hz, double *h)
{
    int P = (T - 1) / 2;
    double sum = 0.0;
    for (int j = -P; j <= P; j++) {
        double s = (j == 0) ? 2.0 * fc_hz / fs_hz : sin(2.0 * M_PI * fc_hz * j / fs_hz) / (M_PI * j);
        double w = (T > 1) ? 0.54 + 0.46 * cos(2.0 * M_PI * j / (T - 1)) : 1.0;
        h[j + P] = w * s;
        sum += w * s;
    }
    for (int j = 0; j < T; j++) h[j] /= sum;
}

/* Envelope by IQ demodulation:
 *   m[n] = RF[n] e^{-i 2 pi fd n / fs}  (0 <= n < S, else 0)
 *   b[k] = sum_{j=-P}^{P} h_j m[k-j];   env[k] = 2 |b[k]|
 * decimation d keeps k = d q, q = 0 .. S/d - 1 (floor).          */
int ora_iq_envelope(const double *rf, int S, double fs_hz, double fd_hz, double bw_hz, int T,
                    int dec, double *env)
{
    if (T < 1 || (T % 2) == 0 || dec < 1) return -1;
    int P = (T - 1) / 2;
    double *h = (double *)malloc(sizeof(double) * T);
    double *mre = (double *)malloc(sizeof(double) * (size_t)S);
    double *mim = (double *)malloc(sizeof(double) * (size_t)S);
    if (!h || !mre || !mim) { free(h); free(mre); free(mim); return -1; }
    ora_fir_taps(T, bw_hz / 2.0, fs_hz, h);
    for (int n = 0; n < S; n++) {
        double ph = 2.0 * M_PI * fd_hz * n / fs_hz;
        mre[n] = rf[n] * cos(ph);
        mim[n] = -rf[n] * sin(ph);
    }
    int nout = S / dec;
    for (int q = 0; q < nout; q++) {
        int k = q * dec;
        double bre = 0.0, bim = 0.0;
        for (int j = -P; j <= P; j++) {
            int n = k - j;
            if (n < 0 || n >= S) continue;
            bre += h[j + P] * mre[n];
            bim += h[j + P] * mim[n];
        }
        env[q] = 2.0 * sqrt(bre * bre + bim * bim);
    }
    free(h); free(mre); free(mim);
    return 0;
}

/* Frequency compounding through a bank of band-passes ("frequency
 * compounding through a bank of configurable bandpasses"; S:186-189 the
 * BandpassBank, "weighted sum of per-band iq_demodulate outputs; all
 * bands share one decimation factor so outputs align sample-for-sample"):
 *   env[q] = sum_{b=0}^{nb-1} w_b env_b[q],  env_b = ora_iq_envelope(rf, band b).
 * Bands are summed in order b = 0, 1, ...                                 */
int ora_compound(const double *rf, int S, double fs_hz, int nb, const double *fd_hz,
                 const double *bw_hz, const double *w, int T, int dec, double *env)
{
    if (nb < 1 || dec < 1) return -1;
    int nout = S / dec;
    double *eb = (double *)malloc(sizeof(double) * (size_t)(nout > 0 ? nout : 1));
    if (!eb) return -1;
    for (int q = 0; q < nout; q++) env[q] = 0.0;
    for (int b = 0; b < nb; b++) {
        if (ora_iq_envelope(rf, S, fs_hz, fd_hz[b], bw_hz[b], T, dec, eb) != 0) { free(eb); return -1; }
        for (int q = 0; q < nout; q++) env[q] += w[b] * eb[q];
    }
    free(eb);
    return 0;
}

/* Log compression:
 *   y = 0 if x = 0, else clamp((20 log10(x/ref) + DR)/DR, 0, 1).
 * ref_mode 0: ref = max over the n values given (the frame);
 * ref_mode 1: ref = ref_value.  ref = 0 (all-zero frame) -> all zeros.
 * Returns the reference used.                                            */
double ora_log_compress(const double *x, long n, int ref_mode, double ref_value, double dr_db,
                        double *y)
{
    double ref = ref_value;
    if (ref_mode == 0) {
        ref = 0.0;
        for (long i = 0; i < n; i++) if (x[i] > ref) ref = x[i];
    }
    for (long i = 0; i < n; i++) {
        if (x[i] == 0.0 || ref == 0.0) { y[i] = 0.0; continue; }
        double t = (20.0 * log10(x[i] / ref) + dr_db) / dr_db;
        y[i] = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
    }
    return ref;
}

/* u8 display code, round to nearest (reading #20).               */
void ora_to_u8(const double *y, long n, uint8_t *out)
{
    for (long i = 0; i < n; i++) out[i] = (uint8_t)floor(255.0 * y[i] + 0.5);
}

/* ------------------------------------------------------------------ */
/* Scan conversion.  Per output pixel
 * the scan geometry is inverted analytically (reading #13, #14, #21, #22):
 *   linear : u = (X - o0x) / ((oLx - o0x)/(L-1)),               v = Z/dr
 *   sector : u = atan2(X,Z)/dth + (L-1)/2,                      v = sqrt(X^2+Z^2)/dr
 *   pyramid: uy = atan2(Y,Z)/dthy + (Ly-1)/2,
 *            ux = atan2(X, sqrt(Y^2+Z^2))/dthx + (Lx-1)/2,      v = sqrt(X^2+Y^2+Z^2)/dr
 * valid iff every u in [0, L_axis-1] and v in [0, S-1];
 * i0 = min(floor(u), L-2), f = u - i0  (L = 1 -> i0 = 0, f = 0).
 * Pixel (ix, iy, iz) sits at origin + i*spacing; output index
 * (iz*ny + iy)*nx + ix.  The value is the bilinear/trilinear blend of the
 * log-compressed line image y[ly][lx][k] (reading #23).                 */
typedef struct {
    int kind;
    int Lx, Ly, S;
    double dr_mm;
    double line0_x_mm, lineL_x_mm; /* linear: origin x of first / last line */
    double fov_x_deg, fov_y_deg;
    int nx, ny, nz;
    double origin_mm[3], spacing_mm[3];
} ora_sc_params;

static void ora_axis(double u, int L, int32_t *i0, double *f)
{
    if (L == 1) { *i0 = 0; *f = 0.0; return; }
    double fl = floor(u);
    int32_t i = (int32_t)fl;
    if (i > L - 2) i = L - 2;
    *i0 = i;
    *f = u - i;
}

/* One pixel: returns validity and writes indices / fractions.            */
static int ora_sc_pixel(const ora_sc_params *p, int ix, int iy, int iz, int32_t *idx, double *fr)
{
    double X = p->origin_mm[0] + ix * p->spacing_mm[0];
    double Y = p->origin_mm[1] + iy * p->spacing_mm[1];
    double Z = p->origin_mm[2] + iz * p->spacing_mm[2];
    double ux = 0.0, uy = 0.0, v = 0.0;
    if (p->kind == ORA_SC_LINEAR_2D) {
        double pitch = (p->lineL_x_mm - p->line0_x_mm) / (p->Lx - 1);
        ux = (X - p->line0_x_mm) / pitch;
        v = Z / p->dr_mm;
    } else if (p->kind == ORA_SC_SECTOR_2D) {
        double fov = p->fov_x_deg * M_PI / 180.0;
        double dth = fov / (p->Lx - 1);
        ux = atan2(X, Z) / dth + (p->Lx - 1) / 2.0;
        v = sqrt(X * X + Z * Z) / p->dr_mm;
    } else {
        double fovx = p->fov_x_deg * M_PI / 180.0;
        double fovy = p->fov_y_deg * M_PI / 180.0;
        double dthx = fovx / (p->Lx - 1);
        double dthy = fovy / (p->Ly - 1);
        uy = atan2(Y, Z) / dthy + (p->Ly - 1) / 2.0;
        ux = atan2(X, sqrt(Y * Y + Z * Z)) / dthx + (p->Lx - 1) / 2.0;
        v = sqrt(X * X + Y * Y + Z * Z) / p->dr_mm;
    }
    int valid = (ux >= 0.0 && ux <= p->Lx - 1) && (v >= 0.0 && v <= p->S - 1);
    if (p->kind == ORA_SC_PYRAMID_3D) valid = valid && (uy >= 0.0 && uy <= p->Ly - 1);
    ora_axis(ux, p->Lx, &idx[0], &fr[0]);
    ora_axis(p->kind == ORA_SC_PYRAMID_3D ? uy : 0.0, p->kind == ORA_SC_PYRAMID_3D ? p->Ly : 1,
             &idx[1], &fr[1]);
    ora_axis(v, p->S, &idx[2], &fr[2]);
    return valid;
}

/* Table for every pixel: valid[n], idx[n][3] = (i0x, i0y, k0),
 * frac[n][3] = (fx, fy, fz).  Pixels not valid keep their indices (for
 * inspection) but are never blended.                                     */
void ora_sc_table(const ora_sc_params *p, uint8_t *valid, int32_t *idx, double *frac)
{
    long n = 0;
    for (int iz = 0; iz < p->nz; iz++)
        for (int iy = 0; iy < p->ny; iy++)
            for (int ix = 0; ix < p->nx; ix++, n++)
                valid[n] = (uint8_t)ora_sc_pixel(p, ix, iy, iz, idx + 3 * n, frac + 3 * n);
}

/* Blend: img[n] = sum_{a,b,c in {0,1}} wx_a wy_b wz_c y[iy0+b][ix0+a][k0+c]
 * with w_0 = 1-f, w_1 = f; invalid -> 0 and mask 0.
 * line_img: [Ly][Lx][S] for one frame.                                   */
void ora_scan_convert(const ora_sc_params *p, const double *line_img, double *img, uint8_t *mask)
{
    long n = 0;
    const int S = p->S, Lx = p->Lx;
    for (int iz = 0; iz < p->nz; iz++)
        for (int iy = 0; iy < p->ny; iy++)
            for (int ix = 0; ix < p->nx; ix++, n++) {
                int32_t idx[3];
                double fr[3];
                int ok = ora_sc_pixel(p, ix, iy, iz, idx, fr);
                if (mask) mask[n] = (uint8_t)ok;
                if (!ok) { img[n] = 0.0; continue; }
                double acc = 0.0;
                int nb = (p->kind == ORA_SC_PYRAMID_3D) ? 2 : 1;
                for (int b = 0; b < nb; b++)
                    for (int a = 0; a < 2; a++)
                        for (int c = 0; c < 2; c++) {
                            double wx = a ? fr[0] : 1.0 - fr[0];
                            double wy = (nb == 1) ? 1.0 : (b ? fr[1] : 1.0 - fr[1]);
                            double wz = c ? fr[2] : 1.0 - fr[2];
                            double w = wx * wy * wz;
                            if (w == 0.0) continue; /* also keeps i0+1 in range when L = 1 */
                            long li = (long)(idx[1] + b) * Lx + (idx[0] + a);
                            acc += w * line_img[li * S + idx[2] + c];
                        }
                img[n] = acc;
            }
}
