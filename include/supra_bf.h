/*
 * supra_bf.h -- C ABI of the B200-native SUPRA receive-beamforming hot path.
 *
 * The library implements the data-parallel steps of the software ultrasound
 * pipeline of Goebl, Navab, Hennersperger, "SUPRA: Open Source Software
 * Defined Ultrasound Processing for Real-Time Applications" (arXiv
 * 1711.06127), section 2 (P:95-100, P:117-123 of /root/reference/PAPER.md):
 *
 *   raw channel data --(delay-and-sum receive beamforming)--> RF
 *                    --(IQ envelope + log compression, fused)--> line image
 *                    --(scan conversion, separate kernel)--> B-mode image
 *
 * Citations: P:n = PAPER.md line n; S:n = SPEC.md line n (interfaces and
 * defaults only); "reading #n" = DESIGN.md "Readings",
 * where the paper is silent.  Units: mm, Hz, m/s, s, degrees.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  * All data buffers are CALLER-OWNED device memory on cfg.device,
 *    contiguous, in the layouts stated below.  The library never frees or
 *    retains them beyond the call and never allocates device or pinned memory
 *    per call, never synchronises the host with a stream, and passes every
 *    per-call tensor map by value as a kernel parameter -- so every call is
 *    capturable in a CUDA graph (a captured graph keeps its own copy of the
 *    parameters; tests/test_graph_gpu.py replays one over rotating buffers).
 *    Per (raw buffer, frames) the host encodes S/32 tensor maps once and
 *    keeps them in a small host-side cache (8 entries); a miss costs host
 *    time only.
 *  * Results are deterministic.  For every call with frames >= 2 the RF and
 *    line image of a frame are bitwise independent of the batch it is in
 *    (its position, the batch size, the launch shape: one summation order
 *    per configuration).  A call with frames = 1 and samples in
 *    {1024, 2048} uses a single-frame kernel that splits the aperture over
 *    warps; it agrees with the batched result to float32 rounding
 *    (normwise RF difference <= 1e-6).
 *  * Calls are asynchronous on `stream` (a cudaStream_t passed as void*; NULL
 *    = legacy default stream).  Validation errors are returned synchronously
 *    before anything is enqueued.  A device fault raised by an earlier launch
 *    surfaces as SUPRA_E_CUDA on a later call.
 *  * A handle owns its device tables and per-frame scratch; it must not be
 *    used concurrently from two streams (create one handle per stream/GPU).
 *    Two handles may read the same raw buffer (the paper's "two differently
 *    parametrized beamforming runs in parallel on the same input").
 *  * There is no CPU fallback: without a usable CUDA device `supra_bf_create`
 *    returns SUPRA_E_CUDA.
 */
#ifndef SUPRA_BF_H
#define SUPRA_BF_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SUPRA_BF_ABI_VERSION 2
#define SUPRA_MAX_BANDS 4   /* frequency-compounding bands */

typedef struct supra_bf *supra_bf_t;

typedef enum {
    SUPRA_OK = 0,
    SUPRA_E_PARAM = 2,    /* a parameter outside its declared range */
    SUPRA_E_STRUCT = 3,   /* NULL / shape / alignment / device mismatch, line_event out of range */
    SUPRA_E_RESOURCE = 4, /* device memory for tables or scratch could not be allocated */
    SUPRA_E_CUDA = 5      /* CUDA runtime / launch error, or no usable device */
} supra_status;

enum { SUPRA_WIN_RECT = 0, SUPRA_WIN_HANN = 1, SUPRA_WIN_HAMMING = 2 }; /* receive window */
enum { SUPRA_INTERP_LINEAR = 0, SUPRA_INTERP_NEAREST = 1 };           /* fractional-delay lookup */
enum { SUPRA_NORM_COUNT = 0, SUPRA_NORM_NONE = 1 };   /* sum / #members (reading #7) or plain sum */
enum { SUPRA_REF_FRAME_MAX = 0, SUPRA_REF_FIXED = 1 };/* log reference */
enum { SUPRA_T_I16 = 0, SUPRA_T_F32 = 1, SUPRA_T_U8 = 2 };
enum { SUPRA_SC_LINEAR_2D = 0, SUPRA_SC_SECTOR_2D = 1, SUPRA_SC_PYRAMID_3D = 2 };

/*
 * Configuration.  `supra_bf_create` copies every field and array; the caller
 * may free them afterwards.  Ranges checked at create (else SUPRA_E_PARAM):
 *   elements_x, elements_y >= 1 with elements_x * elements_y <= 65535 (and num_channels <= 65535),
 *   pitch > 0, center_frequency > 0;
 *   num_events >= 1; samples_per_channel a multiple of 32 in [32, 4096]
 *   (one TMA box holds a whole trace in 64-byte rows; 4096 = 16 tiles of 256
 *   samples held in registers per thread); input_type = SUPRA_T_I16;
 *   sample_frequency > 0; speed_of_sound in [1000, 2000];
 *   f_number > 0; window, normalize in their enums;
 *   fir_taps odd, 1..129; decimation d >= 1 with samples_per_channel / d
 *   >= 2 (the line image keeps k = d q, q < samples / d, and scan
 *   conversion treats it as samples/d samples spaced d dr);
 *   0 < demod_frequency - bw/2 and demod_frequency + bw/2 < fs/2 (S:188,
 *   S:196); dynamic_range_db > 0; reference_value > 0 when
 *   reference_mode = FIXED; spacing > 0 and out_dims >= 1;
 *   0 < fov < 180 degrees for SECTOR / PYRAMID;
 *   max_frames_per_call >= 1.
 * Scanline geometry must match sc_kind (else SUPRA_E_PARAM), because scan
 * conversion inverts it analytically (reading #13/#14):
 *   LINEAR_2D : num_lines_y = 1, num_lines_x >= 2, directions (0,0,1),
 *               origins (x_l, 0, 0) evenly spaced and increasing (1e-9 rel);
 *   SECTOR_2D : num_lines_y = 1, num_lines_x >= 2, origins 0, directions
 *               (sin t_l, 0, cos t_l), t_l = (l - (L-1)/2) fov_x/(L-1) (1e-9);
 *   PYRAMID_3D: num_lines_x, num_lines_y >= 2, origins 0, line l = ly*Lx + lx
 *               with direction (sin tx, cos tx sin ty, cos tx cos ty).
 * line_event[l] in [0, num_events) else SUPRA_E_STRUCT.
 */
typedef struct {
    int32_t abi_version;          /* SUPRA_BF_ABI_VERSION */
    int32_t device;               /* CUDA ordinal; every buffer must live on it */
    /* transducer: element (i,j) at ((i-(Nx-1)/2) px, (j-(Ny-1)/2) py, 0), channel j*Nx+i */
    int32_t elements_x, elements_y;
    double pitch_x_mm, pitch_y_mm;
    double center_frequency_hz;
    /* acquisition: raw frame [num_events][channels][samples], time fastest */
    int32_t num_events, samples_per_channel;
    int32_t input_type;           /* SUPRA_T_I16 */
    double sample_frequency_hz, speed_of_sound_mps;
    double t0_s;                  /* time of sample 0 after the transmit (reading #3); 0 = default */
    /* scanlines ("fully flexible scanline layout") */
    int32_t num_lines_x, num_lines_y;  /* L = Lx*Ly, l = ly*Lx + lx */
    const double *line_origin_mm;      /* [L][3], on the array face (z = 0) */
    const double *line_direction;      /* [L][3], unit within 1e-9 */
    const int32_t *line_event;         /* [L], multi-line map */
    /* receive beamforming */
    double f_number;
    int32_t window, normalize;
    /* envelope: demodulation at f_d, low-pass cutoff bw/2 */
    double demod_frequency_hz, demod_bandwidth_hz;
    int32_t fir_taps, decimation;
    /* log compression */
    double dynamic_range_db, reference_value;
    int32_t reference_mode, line_output_type;  /* line image: SUPRA_T_F32 (y in [0,1]) or SUPRA_T_U8 */
    /* scan conversion */
    int32_t sc_kind, sc_output_type;           /* output: SUPRA_T_F32 or SUPRA_T_U8 */
    int32_t out_dims[3];                       /* nx, ny, nz (ny = 1 for 2D) */
    double out_origin_mm[3], out_spacing_mm[3];/* pixel (ix,iy,iz) at origin + i*spacing */
    double fov_x_deg, fov_y_deg;
    int32_t max_frames_per_call;               /* sizes the per-frame scratch */
    /* frequency compounding through a bank of band-passes ("frequency
     * compounding through a bank of configurable bandpasses"; S:186-189,
     * S:210-218).  num_bands = 0: the single band (demod_frequency_hz,
     * demod_bandwidth_hz), weight 1.  num_bands = 1..SUPRA_MAX_BANDS: band b
     * demodulates at band_center_hz[b] with cutoff band_bandwidth_hz[b]/2
     * (same fir_taps and decimation for every band, so outputs align), and
     * env = sum_b band_weight[b] env_b.  Each band must lie inside (0, fs/2);
     * weights >= 0 and sum to 1 within 1e-9; else SUPRA_E_PARAM. */
    int32_t num_bands;
    double band_center_hz[SUPRA_MAX_BANDS];
    double band_bandwidth_hz[SUPRA_MAX_BANDS];
    double band_weight[SUPRA_MAX_BANDS];
    /* receive channel map (the 128-element probe of Table 1 with only
     * 64 usable channels; "an active-aperture width parameter").
     * num_channels = 0: one channel per element, ch = j*Nx + i (reading #15),
     * raw frames [num_events][Nx*Ny][samples].  num_channels >= 1: raw frames
     * are [num_events][num_channels][samples] and channel_element
     * [num_events][num_channels] gives the element channel ch of event e
     * recorded (-1: unused).  The receive aperture of a line is the set of
     * elements its event recorded; N(k) counts only those (reading #7).
     * An element listed twice in one event, or outside [-1, Nx*Ny), is
     * SUPRA_E_STRUCT. */
    int32_t num_channels;
    const int32_t *channel_element;
    /* fractional-delay sample lookup ("interpolation: {nearest,
     * linear}"): LINEAR (default) x~(tau) = (1-f) x~[i0] + f x~[i0+1];
     * NEAREST x~(tau) = x~[floor(tau + 1/2)] (reading #32). */
    int32_t interpolation;
} supra_bf_config;

/*
 * supra_bf_create -- validate `cfg`, build the per-configuration tables in
 * binary64 on the host, and upload them (the only host->device traffic the
 * library itself causes).  Tables: per-line aperture entries sorted by
 * aperture entry depth k_enter = min{k : (2F) rho <= k dr} (reading
 * #6), element offsets in sample units, complex FIR taps, and the
 * scan-conversion index/fraction table (reading #21/#22).
 *   cfg : host pointer, read only during the call.
 *   out : receives the handle on SUPRA_OK, NULL otherwise.
 * Errors: SUPRA_E_PARAM / SUPRA_E_STRUCT (see the config comment),
 * SUPRA_E_RESOURCE (cudaMalloc), SUPRA_E_CUDA (no device / runtime error).
 */
supra_status supra_bf_create(const supra_bf_config *cfg, supra_bf_t *out);

/*
 * supra_bf_beamform -- delay-and-sum receive beamforming with dynamic receive
 * focusing, optionally followed by the
 * fused IQ envelope and log compression (P:69,
 * P:122).  For line l, output sample k, z = k dr, dr = c/(2 fs):
 *   RF[l][k] = sum_{e : (2F) rho_le <= z} w(rho_le/R) x~_{ev(l),e}(tau_le(k)) / N
 *   tau = (z + |o_l + z d_l - pos_e|) fs/c + t0 fs, linear interpolation,
 *   zero outside [0, S) (reading #10), R = z/(2F), N = #members (0 -> 0).
 *   env[k] = 2 |sum_{j=-P..P} h_j RF[k-j] e^{-i w (k-j)}|  (w = 2 pi f_d / fs);
 *   with a band bank env[k] = sum_b weight_b env_b[k], env_b the same with
 *   (h^b, w_b) of band b (frequency compounding),
 *   y = 0 if env = 0, else clamp((20 log10(env/ref) + DR)/DR, 0, 1),
 *   ref = per-frame max of env (SUPRA_REF_FRAME_MAX) or reference_value.
 * Arguments:
 *   raw      : device, int16 [frames][num_events][channels][samples], 16-byte aligned
 *              (channels = num_channels, or Nx*Ny when num_channels = 0)
 *              (read through TMA tensor maps encoded on the host per
 *              (buffer, frames), cached, and passed as kernel parameters).
 *   frames   : 0 .. max_frames_per_call (0 = no-op).
 *   rf       : device float [frames][L][samples] or NULL.
 *   line_img : device [frames][L][samples / decimation] of line_output_type
 *              or NULL (non-NULL runs the fused envelope + log epilogue).
 *              RF keeps all samples; the line image keeps k = d q.
 *   stream   : cudaStream_t.
 * Errors: SUPRA_E_STRUCT if both outputs are NULL, raw is NULL/misaligned,
 * frames out of range, or a pointer is not device memory of cfg.device.
 */
supra_status supra_bf_beamform(supra_bf_t h, const void *raw, int32_t frames, float *rf,
                               void *line_img, void *stream);

/*
 * supra_bf_envelope_log -- the unfused epilogue on an RF buffer: IQ envelope
 * + log compression exactly as above, for `frames` frames.
 *   rf       : device float [frames][L][samples].
 *   line_img : device [frames][L][samples / decimation] of line_output_type.
 * Errors: SUPRA_E_STRUCT on NULL / frames out of range.
 */
supra_status supra_bf_envelope_log(supra_bf_t h, const float *rf, int32_t frames, void *line_img,
                                   void *stream);

/*
 * Split form of supra_bf_beamform for one volume sharded over GPUs by
 * scanline blocks (latency mode; each transmit event's data
 * is read only by its own lines, so a contiguous line range reads a
 * disjoint part of the input when event blocks align with the range).
 *
 * supra_bf_beamform_lines -- DAS + IQ envelope (the formulas of
 * supra_bf_beamform, without the log step) for lines
 * [line_first, line_first + line_count) of every frame.
 *   env       : device float [frames][L][samples / decimation]; only the range's rows are
 *               written (envelope, >= 0).
 *   frame_max : device float [frames]; receives the maximum of env over the
 *               range (0 for an all-zero range) -- all-reduce(max) it across
 *               ranks to get the frame-max reference of S:267.
 * Errors: SUPRA_E_STRUCT on NULL, a range outside [0, L), frames out of
 * range, raw misaligned, or a pointer that is not device memory.
 *
 * supra_bf_log_compress -- y = clamp((20 log10(env/ref) + DR)/DR, 0, 1)
 * (0 where env = 0 or ref = 0) on the same line range; ref =
 * frame_max[f] (device float [frames]) in SUPRA_REF_FRAME_MAX mode,
 * reference_value in SUPRA_REF_FIXED mode (frame_max may then be NULL).
 *   line_img  : device [frames][L][samples / decimation] of line_output_type; only the
 *               range's rows are written.  env and line_img may alias only
 *               when line_output_type is SUPRA_T_F32 (element-wise, in place).
 * Errors: SUPRA_E_STRUCT on NULL (frame_max NULL in FRAME_MAX mode), a range
 * outside [0, L), frames out of range.
 */
supra_status supra_bf_beamform_lines(supra_bf_t h, const void *raw, int32_t frames, int32_t line_first,
                                     int32_t line_count, float *env, float *frame_max, void *stream);
supra_status supra_bf_log_compress(supra_bf_t h, const float *env, int32_t frames, int32_t line_first,
                                   int32_t line_count, const float *frame_max, void *line_img,
                                   void *stream);

/*
 * supra_bf_scanconvert -- scan conversion in 2D and 3D (S:285-
 * 311): per output pixel/voxel the create-time table gives validity, integer
 * indices (built in binary64, bit-exact with the analytic inverse map) and
 * fractions; the log-compressed line image is blended bilinearly (2D) or
 * trilinearly (3D) (reading #23).  Invalid pixels are 0 with mask 0.
 *   line_img : device [frames][Ly][Lx][samples / decimation] of line_output_type.
 *   img      : device [frames][nz][ny][nx] of sc_output_type (x fastest).
 *   mask     : device uint8 [nz][ny][nx] or NULL (frame-independent).
 * Errors: SUPRA_E_STRUCT on NULL / frames out of range.
 */
supra_status supra_bf_scanconvert(supra_bf_t h, const void *line_img, int32_t frames, void *img,
                                  uint8_t *mask, void *stream);

/*
 * supra_bf_beamform_bmode -- the whole hot path in one call, raw channel data
 * to B-mode image, without materialising the line image: DAS + IQ envelope
 * into the handle's f32 line-domain scratch, then scan conversion that
 * log-compresses each interpolation corner on load (frame-max reference:
 * against the frame's envelope maximum; fixed reference: the
 * epilogue already wrote y).  The image is bitwise the one of
 * supra_bf_beamform(line_img = f32) + supra_bf_scanconvert; it saves the
 * finalisation pass over the line image.
 *   raw  : as supra_bf_beamform;  img, mask: as supra_bf_scanconvert.
 * Errors: SUPRA_E_STRUCT on NULL / misaligned raw / frames out of range /
 * pointers that are not device memory of cfg.device.
 */
supra_status supra_bf_beamform_bmode(supra_bf_t h, const void *raw, int32_t frames, void *img,
                                     uint8_t *mask, void *stream);

/*
 * supra_bf_destroy -- synchronise the device and free the handle's tables and
 * scratch.  NULL is a no-op.
 */
void supra_bf_destroy(supra_bf_t h);

/* ---- introspection (tests, bench) ------------------------------------ */

/* Human-readable text of the last error on this thread ("" if none). */
const char *supra_bf_last_error(void);

/*
 * supra_bf_sc_indices -- copy the scan-conversion table's integer part to
 * host memory for bit-exact comparison with an independent inverse map:
 * for every output pixel n (x fastest): valid[n] in {0,1} and
 * idx[3n..3n+2] = (i0x, i0y, k0) as int32 (undefined where valid = 0);
 * k0 indexes the (decimated) line image, samples / decimation long.
 *   valid : host uint8 [nz*ny*nx];  idx : host int32 [nz*ny*nx][3].
 * Synchronous.  Errors: SUPRA_E_STRUCT on NULL.
 */
supra_status supra_bf_sc_indices(supra_bf_t h, uint8_t *valid, int32_t *idx);

/*
 * supra_bf_info -- launch facts for the bench (host int64 [8]):
 *   [0] kernels launched per beamform call with line_img at max_frames_per_call
 *   (DAS, + a second DAS launch for frames % [1], + finalize in frame-max mode),
 *   [1] DAS frames batched per CTA, [2] DAS depth samples per pass, [3] referenced input
 *   bytes per frame (distinct int16 samples any tap reads x 2),
 *   [4] taps per frame, [5] scan-conversion table bytes, [6] valid output
 *   pixels, [7] kernels per scanconvert call.
 */
supra_status supra_bf_info(supra_bf_t h, int64_t *info8);

/*
 * supra_bf_stage_raw -- host->device input staging for the end-to-end path:
 * for every frame, event and channel, copy from src to the same positions of
 * dst only the sample range supra_bf_beamform reads -- the hull of
 * [floor tau(k_enter), floor tau(S-1) + 1] over the lines and aperture
 * members that use the trace (reading #6), widened by one
 * sample and rounded out to 16 bytes.  Samples outside those ranges are
 * left untouched in dst and are never read by supra_bf_beamform, so
 * beamforming dst gives exactly the result of beamforming a full copy of
 * src.  With src in page-locked host memory the device reads it over PCIe:
 * the transfer carries the referenced bytes only (C2: 41 % of a frame).
 * Arguments:
 *   src  : int16 [frames][num_events][channels][samples], 16-byte aligned;
 *          page-locked host memory (cudaHostAlloc / cudaMallocHost) or
 *          device memory of cfg.device.
 *   dst  : device int16, same shape, 16-byte aligned.
 *   frames : 0 .. max_frames_per_call.
 *   bytes_per_frame : NULL or host int64, set to the bytes copied per frame.
 *   stream : cudaStream_t (the copy is asynchronous on it).
 * Errors: SUPRA_E_STRUCT on a NULL handle/buffer, misalignment, frames out
 * of range, pageable src, or dst not device memory of cfg.device.
 */
supra_status supra_bf_stage_raw(supra_bf_t h, const void *src, void *dst, int32_t frames,
                                int64_t *bytes_per_frame, void *stream);

/*
 * supra_bf_set_das_events -- measurement hook for the bench: when non-NULL,
 * supra_bf_beamform records `before` and `after` (cudaEvent_t) on its stream
 * immediately around the DAS kernel launch, so the kernel's duration can be
 * timed with CUDA events on the stream it runs on.  NULL, NULL disables.
 * Errors: SUPRA_E_STRUCT on a NULL handle.
 */
supra_status supra_bf_set_das_events(supra_bf_t h, void *before, void *after);

#ifdef __cplusplus
}
#endif
#endif /* SUPRA_BF_H */
