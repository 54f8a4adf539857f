/*
 * synth/synth.c -- point-scatterer channel-data generator (CPU, binary64).
 *
 * INPUT GENERATION ONLY (SPEC synth module).  It computes echo
 * arrival times of a forward model; it contains none of the method's
 * arithmetic (no delay-and-sum, envelope, compression or scan conversion).
 * The oracle and the CUDA path consume the same int16 buffer it produces.
 *
 * Model (reading #3): event ev with transmit reference o_ev, scatterer
 * q with reflectivity a, element e:
 *   arrival [samples] = (|q - o_ev| + |q - pos_e|) / 1000 * fs / c
 *   signal[n] += a / (|q - o_ev| |q - pos_e|) * g(n - arrival)
 *   g(t) = exp(-t^2 / (2 sigma^2)) cos(2 pi f0 t / fs),  |t| <= 4 sigma,
 *   sigma = fs / (2 pi sigma_f), sigma_f = fbw f0 / (2 sqrt(2 ln 2))
 * (Gaussian-enveloped cosine with -6 dB amplitude-spectrum fractional
 * bandwidth fbw, zero phase).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <pthread.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

typedef struct {
    int nx, ny;
    double pitch_x_mm, pitch_y_mm;
    int E, S;
    double fs_hz, c_mps, f0_hz, fbw;
    int nch;                 /* 0: channel = element; else traces per event */
    const int32_t *chmap;    /* [E][nch] element of each channel, -1 = unused (zero trace) */
} syn_params;

double syn_sigma_samples(double fs_hz, double f0_hz, double fbw)
{
    double sigma_f = fbw * f0_hz / (2.0 * sqrt(2.0 * log(2.0)));
    return fs_hz / (2.0 * M_PI * sigma_f);
}

typedef struct {
    const syn_params *p;
    const double *scat;
    int nscat;
    const double *tx;
    double *out;
    int t, nt;
} syn_job;

static void *syn_worker(void *arg)
{
    syn_job *j = (syn_job *)arg;
    const syn_params *p = j->p;
    const int C = p->nch > 0 ? p->nch : p->nx * p->ny, S = p->S;
    const double sig = syn_sigma_samples(p->fs_hz, p->f0_hz, p->fbw);
    const double half = 4.0 * sig;
    const double w0 = 2.0 * M_PI * p->f0_hz / p->fs_hz;
    const double smm = p->fs_hz / (1000.0 * p->c_mps);
    for (long tr = j->t; tr < (long)p->E * C; tr += j->nt) {
        int ev = (int)(tr / C), ch = (int)(tr % C);
        int el = p->nch > 0 ? p->chmap[(size_t)ev * p->nch + ch] : ch;
        int i = el % p->nx, jj = el / p->nx;
        double ex = (i - (p->nx - 1) / 2.0) * p->pitch_x_mm;
        double ey = (jj - (p->ny - 1) / 2.0) * p->pitch_y_mm;
        double *o = j->out + (size_t)tr * S;
        for (int n = 0; n < S; n++) o[n] = 0.0;
        if (el < 0) continue;
        const double *t = j->tx + 3 * ev;
        for (int s = 0; s < j->nscat; s++) {
            const double *q = j->scat + 4 * s;
            double dtx = sqrt((q[0] - t[0]) * (q[0] - t[0]) + (q[1] - t[1]) * (q[1] - t[1]) +
                              (q[2] - t[2]) * (q[2] - t[2]));
            double drx = sqrt((q[0] - ex) * (q[0] - ex) + (q[1] - ey) * (q[1] - ey) + q[2] * q[2]);
            if (dtx <= 0.0 || drx <= 0.0) continue;
            double arr = (dtx + drx) * smm;
            double amp = q[3] / (dtx * drx);
            long lo = (long)ceil(arr - half), hi = (long)floor(arr + half);
            if (lo < 0) lo = 0;
            if (hi > S - 1) hi = S - 1;
            for (long n = lo; n <= hi; n++) {
                double tt = n - arr;
                o[n] += amp * exp(-tt * tt / (2.0 * sig * sig)) * cos(w0 * tt);
            }
        }
    }
    return NULL;
}

/* Noiseless signal [E][C][S] (double).                                  */
void syn_frame(const syn_params *p, const double *scat, int nscat, const double *tx_origin,
               double *out, int nthreads)
{
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    syn_job jobs[256];
    for (int t = 0; t < nthreads; t++) {
        jobs[t] = (syn_job){p, scat, nscat, tx_origin, out, t, nthreads};
        if (nthreads > 1) pthread_create(&th[t], NULL, syn_worker, &jobs[t]);
    }
    if (nthreads == 1) syn_worker(&jobs[0]);
    else for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
}

/* Counter-based normal deviates (splitmix64 + Box-Muller), identical
 * recipe in synth_gpu.cu, so noise is reproducible from (seed, index).   */
static uint64_t syn_mix(uint64_t x)
{
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

double syn_gauss(uint64_t seed, uint64_t idx)
{
    uint64_t h1 = syn_mix((seed << 40) ^ (2 * idx));
    uint64_t h2 = syn_mix((seed << 40) ^ (2 * idx + 1));
    double u1 = ((h1 >> 11) + 1) * (1.0 / 9007199254740992.0);
    double u2 = (h2 >> 11) * (1.0 / 9007199254740992.0);
    return sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2);
}

/* int16 quantisation with 12 dB headroom: the noiseless peak maps to
 * 32767/4; optional white noise of std noise_rel * peak; round half even
 * (rint, default rounding mode).  Returns the peak.                      */
double syn_quantize(const double *sig, long n, double noise_rel, uint64_t seed, int16_t *out)
{
    double peak = 0.0;
    for (long i = 0; i < n; i++) if (fabs(sig[i]) > peak) peak = fabs(sig[i]);
    double scale = (peak > 0.0) ? (32767.0 / 4.0) / peak : 0.0;
    for (long i = 0; i < n; i++) {
        double x = sig[i];
        if (noise_rel > 0.0) x += noise_rel * peak * syn_gauss(seed, (uint64_t)i);
        double v = rint(x * scale);
        if (v > 32767.0) v = 32767.0;
        if (v < -32768.0) v = -32768.0;
        out[i] = (int16_t)v;
    }
    return peak;
}
