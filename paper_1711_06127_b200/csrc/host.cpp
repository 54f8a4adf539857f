// host.cpp -- C-ABI host library: validation, binary64 setup tables, launches.
//
// Implements include/supra_bf.h.  Table construction runs once per
// configuration on the host in IEEE binary64 (compiled -ffp-contract=off) so
// every discontinuous decision -- aperture membership and scan-conversion
// indices -- is taken with the canonical expressions stated in DESIGN.md
// "Readings" (#6, #21, #22) and is bit-exact with any other binary64
// evaluation of the same definition.  Per-frame work runs in the sm_100a
// kernels (das.cu, epilogue.cu, scanconv.cu); there is no CPU fallback.
#include "supra_bf.h"
#include "internal.h"

#include <algorithm>
#include <cstdarg>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

using namespace supra;

namespace {

thread_local std::string g_err;

supra_status fail(supra_status s, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
supra_status fail(supra_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

constexpr double kPi = 3.14159265358979323846;

struct DeviceGuard {
  int prev = -1;
  bool ok = false;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    ok = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

}  // namespace

struct supra_bf {
  supra_bf_config cfg{};
  int L = 0, C = 0, S = 0, E = 0, G = 0;
  int dec = 1, Sd = 0;  // envelope decimation and line-image samples S / dec
  int ntiles = 0, entries_per_group = 0;
  int frames_per_cta = 1;
  size_t das_smem = 0;
  double dr_mm = 0.0, s_per_mm = 0.0;
  // device tables
  int32_t* d_line_group = nullptr;
  DasEntry* d_entries = nullptr;
  int32_t* d_nentries = nullptr;
  uint16_t* d_ncount = nullptr;
  float4* d_line_dir = nullptr;
  int32_t* d_line_event = nullptr;
  // mirror symmetry (DasArgs::cta / ech): CTA descriptor tables for MIR = 1,
  // 2, 4 lines per CTA (index 0, 1, 2; NULL if the layout lacks that order)
  // and the per-entry channel of each mirror variant
  int32_t* d_cta[3] = {nullptr, nullptr, nullptr};
  int32_t* d_ech = nullptr;
  uint32_t* d_stage_iv = nullptr;  // [E][C] 16-byte chunk range each trace's taps read (supra_bf_stage_raw)
  int64_t stage_bytes = 0;         // bytes supra_bf_stage_raw moves per frame
  int sym_order = 1;    // 1, 2 or 4 mirror lines that share one delay set
  bool sym_x = false;   // the 2-line tables pair x-mirrors (rows stay whole)
  int num_sms = 148;
  float2* d_fir = nullptr;
  unsigned* d_frame_max = nullptr;
  float* d_env = nullptr;
  ScAxis* d_ax = nullptr;
  ScAxis* d_az = nullptr;
  int32_t* d_blk_kmin = nullptr;
  int32_t* d_col_l0 = nullptr;
  int32_t* d_col_nl = nullptr;
  int slab_k = 2;
  int sc_tiled = 1;
  int sc_box_k = 4, sc_box_l = 1;
  ScRow* d_rows = nullptr;
  ScEntry* d_ent = nullptr;
  // host copies for introspection
  std::vector<ScAxis> h_ax, h_az;
  std::vector<ScRow> h_rows;
  std::vector<ScEntry> h_ent;
  int nbands = 1;
  float band_w[kMaxBands] = {1.f, 0.f, 0.f, 0.f};
  std::vector<float> fir_c, fir_s;  // [kMaxBands][kMaxHalfTaps + 1]
  cudaEvent_t ev_before = nullptr, ev_after = nullptr;
  // per-(raw buffer, frames, shape) row-cut tensor-map sets, HOST memory
  // only: each launch passes its set by value as a kernel parameter, so a
  // set can be re-encoded at any time without synchronisation (LRU of
  // kMapCache entries; a miss costs S/32 host encodes, never a device
  // allocation or a stall)
  static constexpr int kMapCache = 8;
  struct MapSet {
    const void* raw = nullptr;
    int F = 0, fb = 0, nt = 0;
    uint64_t used = 0;
    RawMaps maps;
  };
  std::vector<MapSet> mcache;
  uint64_t mclock = 0;
  int64_t info[8] = {0};
};

namespace {

template <class T>
cudaError_t upload(T** d, const std::vector<T>& h) {
  *d = nullptr;
  if (h.empty()) return cudaSuccess;
  cudaError_t e = cudaMalloc((void**)d, h.size() * sizeof(T));
  if (e != cudaSuccess) return e;
  return cudaMemcpy(*d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice);
}

void free_all(supra_bf* h) {
  void* ptrs[] = {h->d_cta[0], h->d_cta[1], h->d_cta[2], h->d_ech,
                  h->d_line_group, h->d_entries, h->d_nentries, h->d_ncount, h->d_line_dir, h->d_line_event,
                  h->d_fir, h->d_frame_max, h->d_env, h->d_ax, h->d_az, h->d_blk_kmin, h->d_col_l0, h->d_col_nl, h->d_rows, h->d_ent, h->d_stage_iv};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  h->mcache.clear();
}

// Element (i,j) position, S:30 (same definition the oracle writes out).
inline void elem_pos(const supra_bf_config& c, int ch, double* p) {
  int i = ch % c.elements_x, j = ch / c.elements_x;
  p[0] = (i - (c.elements_x - 1) / 2.0) * c.pitch_x_mm;
  p[1] = (j - (c.elements_y - 1) / 2.0) * c.pitch_y_mm;
  p[2] = 0.0;
}

// Canonical aperture predicate (reading #6): (2F) rho <= k dr, binary64.
inline bool member(double F, double rho, int k, double dr) { return (2.0 * F) * rho <= k * dr; }

int k_enter(double F, double rho, double dr, int S) {
  double g = std::ceil((2.0 * F) * rho / dr);
  long k = (g < 0) ? 0 : (g > S + 2.0 ? (long)S + 2 : (long)g);
  while (k > 0 && member(F, rho, (int)k - 1, dr)) k--;
  while (k <= S && !member(F, rho, (int)k, dr)) k++;
  return (int)std::min<long>(k, S);
}

// tau in samples for element e, line (o,d), output sample k (binary64).
double tau_d(const double* o, const double* d, const double* e, int k, double dr, double fs,
             double c, double t0) {
  double z = k * dr;
  double p0 = o[0] + z * d[0] - e[0], p1 = o[1] + z * d[1] - e[1], p2 = o[2] + z * d[2] - e[2];
  double r = std::sqrt(p0 * p0 + p1 * p1 + p2 * p2);
  return ((z + r) / 1000.0) * fs / c + t0 * fs;
}

supra_status validate(const supra_bf_config* c) {
  if (!c) return fail(SUPRA_E_STRUCT, "cfg is NULL");
  if (c->abi_version != SUPRA_BF_ABI_VERSION)
    return fail(SUPRA_E_PARAM, "abi_version %d != %d", c->abi_version, SUPRA_BF_ABI_VERSION);
  if (c->elements_x < 1 || c->elements_y < 1) return fail(SUPRA_E_PARAM, "elements must be >= 1");
  if ((int64_t)c->elements_x * c->elements_y > 65535 || c->num_channels > 65535)
    return fail(SUPRA_E_PARAM, "at most 65535 elements and channels per event");
  if (!(c->pitch_x_mm > 0) || !(c->pitch_y_mm > 0)) return fail(SUPRA_E_PARAM, "pitch must be > 0");
  if (!(c->center_frequency_hz > 0)) return fail(SUPRA_E_PARAM, "center_frequency must be > 0");
  if (c->num_events < 1) return fail(SUPRA_E_PARAM, "num_events must be >= 1");
  if (c->samples_per_channel < 32 || c->samples_per_channel % kRowSamples != 0 ||
      c->samples_per_channel > kMaxSamples)
    return fail(SUPRA_E_PARAM, "samples_per_channel must be a multiple of 32 in [32, 4096]");
  if (c->input_type != SUPRA_T_I16) return fail(SUPRA_E_PARAM, "input_type must be SUPRA_T_I16");
  if (!(c->sample_frequency_hz > 0)) return fail(SUPRA_E_PARAM, "sample_frequency must be > 0");
  if (!(c->speed_of_sound_mps >= 1000.0 && c->speed_of_sound_mps <= 2000.0))
    return fail(SUPRA_E_PARAM, "speed_of_sound must be in [1000, 2000] m/s (S:126)");
  if (!std::isfinite(c->t0_s)) return fail(SUPRA_E_PARAM, "t0 must be finite");
  if (c->num_lines_x < 1 || c->num_lines_y < 1) return fail(SUPRA_E_PARAM, "num_lines must be >= 1");
  if (!c->line_origin_mm || !c->line_direction || !c->line_event)
    return fail(SUPRA_E_STRUCT, "line arrays must not be NULL");
  if (!(c->f_number > 0)) return fail(SUPRA_E_PARAM, "f_number must be > 0 (S:126)");
  if (c->window < SUPRA_WIN_RECT || c->window > SUPRA_WIN_HAMMING) return fail(SUPRA_E_PARAM, "window");
  if (c->normalize != SUPRA_NORM_COUNT && c->normalize != SUPRA_NORM_NONE) return fail(SUPRA_E_PARAM, "normalize");
  if (c->interpolation != SUPRA_INTERP_LINEAR && c->interpolation != SUPRA_INTERP_NEAREST)
    return fail(SUPRA_E_PARAM, "interpolation must be LINEAR or NEAREST (S:125)");
  if (c->fir_taps < 1 || c->fir_taps > 129 || c->fir_taps % 2 == 0)
    return fail(SUPRA_E_PARAM, "fir_taps must be odd in [1, 129] (S:196)");
  if (c->decimation < 1 || c->samples_per_channel / c->decimation < 2)
    return fail(SUPRA_E_PARAM, "decimation must be >= 1 with samples_per_channel / decimation >= 2 (S:224)");
  double fd = c->demod_frequency_hz, bw = c->demod_bandwidth_hz;
  if (!(bw > 0) || !(fd - bw / 2 > 0) || !(fd + bw / 2 < c->sample_frequency_hz / 2))
    return fail(SUPRA_E_PARAM, "demodulation band must lie inside (0, fs/2) (S:188)");
  if (c->num_bands < 0 || c->num_bands > SUPRA_MAX_BANDS)
    return fail(SUPRA_E_PARAM, "num_bands must be in [0, %d]", SUPRA_MAX_BANDS);
  double wsum = 0.0;
  for (int b = 0; b < c->num_bands; b++) {
    const double bc = c->band_center_hz[b], bb = c->band_bandwidth_hz[b], bw_ = c->band_weight[b];
    if (!(bb > 0) || !(bc - bb / 2 > 0) || !(bc + bb / 2 < c->sample_frequency_hz / 2))
      return fail(SUPRA_E_PARAM, "band %d must lie inside (0, fs/2) (S:188)", b);
    if (!(bw_ >= 0) || !std::isfinite(bw_)) return fail(SUPRA_E_PARAM, "band weight %d must be >= 0", b);
    wsum += bw_;
  }
  if (c->num_bands > 0 && !(std::fabs(wsum - 1.0) <= 1e-9))
    return fail(SUPRA_E_PARAM, "band weights must sum to 1 within 1e-9 (S:187)");
  if (!(c->dynamic_range_db > 0)) return fail(SUPRA_E_PARAM, "dynamic_range_db must be > 0 (S:247)");
  if (c->reference_mode != SUPRA_REF_FRAME_MAX && c->reference_mode != SUPRA_REF_FIXED)
    return fail(SUPRA_E_PARAM, "reference_mode");
  if (c->reference_mode == SUPRA_REF_FIXED && !(c->reference_value > 0))
    return fail(SUPRA_E_PARAM, "fixed reference must be > 0 (S:247)");
  if (c->line_output_type != SUPRA_T_F32 && c->line_output_type != SUPRA_T_U8)
    return fail(SUPRA_E_PARAM, "line_output_type must be F32 or U8");
  if (c->sc_output_type != SUPRA_T_F32 && c->sc_output_type != SUPRA_T_U8)
    return fail(SUPRA_E_PARAM, "sc_output_type must be F32 or U8");
  if (c->sc_kind < SUPRA_SC_LINEAR_2D || c->sc_kind > SUPRA_SC_PYRAMID_3D) return fail(SUPRA_E_PARAM, "sc_kind");
  for (int i = 0; i < 3; i++) {
    if (c->out_dims[i] < 1) return fail(SUPRA_E_PARAM, "out_dims must be >= 1");
    if (!(c->out_spacing_mm[i] > 0)) return fail(SUPRA_E_PARAM, "out_spacing must be > 0 (S:296)");
    if (!std::isfinite(c->out_origin_mm[i])) return fail(SUPRA_E_PARAM, "out_origin must be finite");
  }
  if (c->max_frames_per_call < 1) return fail(SUPRA_E_PARAM, "max_frames_per_call must be >= 1");
  const int L = c->num_lines_x * c->num_lines_y;
  for (int l = 0; l < L; l++)
    if (c->line_event[l] < 0 || c->line_event[l] >= c->num_events)
      return fail(SUPRA_E_STRUCT, "line_event[%d] = %d out of [0, %d)", l, c->line_event[l], c->num_events);
  for (int l = 0; l < L; l++) {
    const double* d = c->line_direction + 3 * l;
    double n = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    if (!(std::fabs(n - 1.0) <= 1e-9)) return fail(SUPRA_E_PARAM, "line_direction[%d] not unit (S:37)", l);
    if (c->line_origin_mm[3 * l + 2] != 0.0) return fail(SUPRA_E_PARAM, "line origins must lie on the array face z = 0");
  }
  // geometry must match the scan-conversion inverse map
  const double tol = 1e-9;
  if (c->sc_kind == SUPRA_SC_LINEAR_2D) {
    if (c->num_lines_y != 1 || c->num_lines_x < 2) return fail(SUPRA_E_PARAM, "LINEAR_2D needs 1 x (>=2) lines");
    if (c->out_dims[1] != 1) return fail(SUPRA_E_PARAM, "2D output needs out_dims[1] = 1");
    double x0 = c->line_origin_mm[0], xL = c->line_origin_mm[3 * (L - 1)];
    if (!(xL > x0)) return fail(SUPRA_E_PARAM, "LINEAR_2D origins must increase");
    double span = xL - x0;
    for (int l = 0; l < L; l++) {
      const double* o = c->line_origin_mm + 3 * l;
      const double* d = c->line_direction + 3 * l;
      double xe = x0 + span * l / (L - 1);
      if (std::fabs(o[0] - xe) > tol * std::max(1.0, span) || o[1] != 0.0)
        return fail(SUPRA_E_PARAM, "LINEAR_2D origins must be evenly spaced on the x axis");
      if (std::fabs(d[0]) > tol || std::fabs(d[1]) > tol || std::fabs(d[2] - 1.0) > tol)
        return fail(SUPRA_E_PARAM, "LINEAR_2D directions must be (0,0,1)");
    }
  } else {
    const bool is3d = c->sc_kind == SUPRA_SC_PYRAMID_3D;
    if (!(c->fov_x_deg > 0 && c->fov_x_deg < 180)) return fail(SUPRA_E_PARAM, "fov_x must be in (0, 180) (S:64)");
    if (is3d && !(c->fov_y_deg > 0 && c->fov_y_deg < 180)) return fail(SUPRA_E_PARAM, "fov_y must be in (0, 180) (S:64)");
    if (c->num_lines_x < 2) return fail(SUPRA_E_PARAM, "phased layouts need >= 2 lines in x");
    if (!is3d && (c->num_lines_y != 1 || c->out_dims[1] != 1)) return fail(SUPRA_E_PARAM, "SECTOR_2D needs 1 line row and out_dims[1] = 1");
    if (is3d && c->num_lines_y < 2) return fail(SUPRA_E_PARAM, "PYRAMID_3D needs >= 2 lines in y");
    const double fx = c->fov_x_deg * kPi / 180.0, fy = c->fov_y_deg * kPi / 180.0;
    for (int l = 0; l < L; l++) {
      int lx = l % c->num_lines_x, ly = l / c->num_lines_x;
      double tx = (lx - (c->num_lines_x - 1) / 2.0) * (fx / (c->num_lines_x - 1));
      double ty = is3d ? (ly - (c->num_lines_y - 1) / 2.0) * (fy / (c->num_lines_y - 1)) : 0.0;
      double e[3] = {std::sin(tx), std::cos(tx) * std::sin(ty), std::cos(tx) * std::cos(ty)};
      const double* o = c->line_origin_mm + 3 * l;
      const double* d = c->line_direction + 3 * l;
      if (o[0] != 0.0 || o[1] != 0.0) return fail(SUPRA_E_PARAM, "phased line origins must be 0");
      for (int i = 0; i < 3; i++)
        if (std::fabs(d[i] - e[i]) > tol)
          return fail(SUPRA_E_PARAM, "line_direction[%d] off the uniform angle grid (reading #13/#14)", l);
    }
  }
  // receive channel map
  if (c->num_channels < 0) return fail(SUPRA_E_PARAM, "num_channels must be >= 0");
  if (c->num_channels > 0) {
    if (!c->channel_element) return fail(SUPRA_E_STRUCT, "channel_element must not be NULL when num_channels > 0");
    const int nel = c->elements_x * c->elements_y;
    std::vector<int> seen(nel, -1);
    for (int e = 0; e < c->num_events; e++)
      for (int ch = 0; ch < c->num_channels; ch++) {
        const int el = c->channel_element[(size_t)e * c->num_channels + ch];
        if (el < -1 || el >= nel) return fail(SUPRA_E_STRUCT, "channel_element[%d][%d] = %d out of range", e, ch, el);
        if (el >= 0) {
          if (seen[el] == e) return fail(SUPRA_E_STRUCT, "element %d recorded twice in event %d", el, e);
          seen[el] = e;
        }
      }
  }
  return SUPRA_OK;
}

// ---- mirror symmetry -------------------------------------------------
// A phased / matrix layout (every origin at 0) whose steering grid is
// symmetric about the x (y) axis pairs line (lx, ly) with (Lx-1-lx, ly)
// ((lx, Ly-1-ly)).  With element (i, j) <-> (Nx-1-i, j) ((i, Ny-1-j)) the
// mirrored line sees the mirrored element at exactly the same q-component
// products d.q, |q|^2 and rho (sign flips cancel in IEEE arithmetic), so
// its delays, weights, memberships and N(k) are bitwise those of the
// original: up to 4 lines share one delay set, and the DAS kernel computes
// the geometry once for all of them ("mirror lines").
// Every line is described as (canonical primary line, variant v): variant
// bit 0 = x-mirror, bit 1 = y-mirror; its taps are the primary's aperture
// entries in the primary's order, each read from the variant's mirrored
// channel -- so a line's result does not depend on how lines are grouped
// into CTAs.  Returns the CTA tables and entry channels, or sym_order = 1.
void build_mirror_tables(supra_bf* h, const std::vector<int32_t>& line_group,
                         const std::vector<std::vector<DasEntry>>& groups, const std::vector<int>& g_event,
                         std::vector<int32_t>& cta1, std::vector<int32_t>& cta2, std::vector<int32_t>& cta4,
                         std::vector<int32_t>& ech, int per) {
  const supra_bf_config& c = h->cfg;
  const int L = h->L, Lx = c.num_lines_x, Ly = c.num_lines_y, Nx = c.elements_x, Ny = c.elements_y;
  const int G = (int)groups.size();
  // channel of an element: identity, or the (uniform) channel map
  const int nel = Nx * Ny;
  std::vector<int> chan_of(nel, -1);
  bool ok = true;
  if (c.num_channels > 0) {
    for (int e = 1; e < c.num_events && ok; e++)
      ok = std::equal(c.channel_element, c.channel_element + c.num_channels,
                      c.channel_element + (size_t)e * c.num_channels);
    for (int ch = 0; ch < c.num_channels && ok; ch++)
      if (c.channel_element[ch] >= 0) chan_of[c.channel_element[ch]] = ch;
  } else {
    for (int e = 0; e < nel; e++) chan_of[e] = e;
  }
  for (int l = 0; l < L && ok; l++)
    ok = c.line_origin_mm[3 * l] == 0.0 && c.line_origin_mm[3 * l + 1] == 0.0 && c.line_origin_mm[3 * l + 2] == 0.0;
  auto mirror_el = [&](int e, int v) {
    int i = e % Nx, j = e / Nx;
    if (v & 1) i = Nx - 1 - i;
    if (v & 2) j = Ny - 1 - j;
    return j * Nx + i;
  };
  auto mirror_line = [&](int l, int v) {
    int lx = l % Lx, ly = l / Lx;
    if (v & 1) lx = Lx - 1 - lx;
    if (v & 2) ly = Ly - 1 - ly;
    return ly * Lx + lx;
  };
  auto fdir = [&](int l, int k) { return (float)c.line_direction[3 * l + k]; };
  auto sym_ok = [&](int v) {
    if (!ok) return false;
    if ((v & 1) && Lx % 2) return false;
    if ((v & 2) && (Ly % 2 || Ly < 2)) return false;
    for (int l = 0; l < L; l++) {
      const int m = mirror_line(l, v);
      const float ex = (v & 1) ? -fdir(l, 0) : fdir(l, 0), ey = (v & 2) ? -fdir(l, 1) : fdir(l, 1);
      if (fdir(m, 0) != ex || fdir(m, 1) != ey || fdir(m, 2) != fdir(l, 2)) return false;
      if (line_group[m] != line_group[l]) return false;
    }
    // the recorded element set is closed under the mirror
    for (int e = 0; e < nel; e++)
      if ((chan_of[e] >= 0) != (chan_of[mirror_el(e, v)] >= 0)) return false;
    return true;
  };
  const bool sx = sym_ok(1), sy = sym_ok(2);
  const int vmask = (sx ? 1 : 0) | (sy ? 2 : 0);
  h->sym_order = (sx ? 2 : 1) * (sy ? 2 : 1);
  h->sym_x = sx;
  // canonical primary and variant of every line
  std::vector<int> prim(L), var(L);
  for (int l = 0; l < L; l++) {
    const int lx = l % Lx, ly = l / Lx;
    int v = 0;
    if ((vmask & 1) && lx >= Lx / 2) v |= 1;
    if ((vmask & 2) && ly >= Ly / 2) v |= 2;
    var[l] = v;
    prim[l] = mirror_line(l, v);
  }
  // entry channels per variant (variant 0 = the entry's own channel)
  ech.assign((size_t)G * per * 4, 0);
  for (int g = 0; g < G; g++)
    for (size_t j = 0; j < groups[g].size(); j++) {
      const int ch = groups[g][j].elem;
      const int el = c.num_channels > 0 ? c.channel_element[(size_t)g_event[g] * c.num_channels + ch] : ch;
      for (int v = 0; v < 4; v++) {
        const int mc = (v & ~vmask) ? ch : chan_of[mirror_el(el, v)];
        ech[((size_t)g * per + j) * 4 + v] = mc < 0 ? ch : mc;
      }
    }
  auto push = [](std::vector<int32_t>& t, int p, const int* ls, const int* vs, int n) {
    t.push_back(p);
    for (int i = 0; i < 4; i++) t.push_back(i < n ? ls[i] : ls[0]);
    for (int i = 0; i < 4; i++) t.push_back(i < n ? vs[i] : vs[0]);
  };
  cta1.clear(); cta2.clear(); cta4.clear();
  for (int l = 0; l < L; l++) push(cta1, prim[l], &l, &var[l], 1);
  if (h->sym_order >= 2) {
    // pairs along one mirrored axis (x if available): slots {l, mirror(l)}
    const int vb = (vmask & 1) ? 1 : 2;
    for (int l = 0; l < L; l++) {
      if (var[l] & vb) continue;  // l is the first slot of its pair
      const int ls[2] = {l, mirror_line(l, vb)}, vs[2] = {var[l], var[l] | vb};
      push(cta2, prim[l], ls, vs, 2);
    }
  }
  if (h->sym_order == 4)
    for (int l = 0; l < L; l++) {
      if (var[l]) continue;
      const int ls[4] = {l, mirror_line(l, 1), mirror_line(l, 2), mirror_line(l, 3)}, vs[4] = {0, 1, 2, 3};
      push(cta4, l, ls, vs, 4);
    }
}

// ---- DAS tables ------------------------------------------------------
supra_status build_das_tables(supra_bf* h) {
  const supra_bf_config& c = h->cfg;
  const int L = h->L, C = h->C, S = h->S;
  const double dr = h->dr_mm, sc = h->s_per_mm, F = c.f_number;
  // line groups: lines with bitwise-identical origins (and, with a channel
  // map, events that recorded the same channel -> element map) share an
  // aperture table
  std::map<std::vector<double>, int> gid;
  std::vector<int32_t> line_group(L);
  std::vector<const double*> g_origin;
  std::vector<int> g_event;  // an event of the group (its channel map row)
  for (int l = 0; l < L; l++) {
    std::vector<double> key(c.line_origin_mm + 3 * l, c.line_origin_mm + 3 * l + 3);
    if (c.num_channels > 0) {
      const int32_t* row = c.channel_element + (size_t)c.line_event[l] * c.num_channels;
      key.insert(key.end(), row, row + c.num_channels);
    }
    auto it = gid.find(key);
    if (it == gid.end()) {
      it = gid.emplace(key, (int)g_origin.size()).first;
      g_origin.push_back(c.line_origin_mm + 3 * l);
      g_event.push_back(c.line_event[l]);
    }
    line_group[l] = it->second;
  }
  const int G = (int)g_origin.size();
  h->G = G;
  std::vector<std::vector<DasEntry>> groups(G);
  size_t maxn = 0;
  for (int g = 0; g < G; g++) {
    const double* o = g_origin[g];
    auto& v = groups[g];
    for (int ch = 0; ch < C; ch++) {
      const int el = c.num_channels > 0 ? c.channel_element[(size_t)g_event[g] * c.num_channels + ch] : ch;
      if (el < 0) continue;  // channel unused in this event
      double e[3];
      elem_pos(c, el, e);
      double rho = std::hypot(e[0] - o[0], e[1] - o[1]);
      int ke = k_enter(F, rho, dr, S);
      if (ke >= S) continue;  // never in the aperture within the record
      DasEntry d{};
      double q0 = (o[0] - e[0]) * sc, q1 = (o[1] - e[1]) * sc, q2 = (o[2] - e[2]) * sc;
      d.qx = (float)q0;
      d.qy = (float)q1;
      d.qz = (float)q2;
      d.A = (float)(q0 * q0 + q1 * q1 + q2 * q2);
      d.cu = (float)(4.0 * F * rho * sc);
      d.elem = ch;
      d.kenter = ke;
      v.push_back(d);
    }
    std::stable_sort(v.begin(), v.end(),
                     [](const DasEntry& a, const DasEntry& b) { return a.kenter < b.kenter; });
    maxn = std::max(maxn, v.size());
  }
  const int per = (int)std::max<size_t>(32, (maxn + 31) / 32 * 32);
  h->entries_per_group = per;
  h->ntiles = (S + kTileK - 1) / kTileK;
  std::vector<DasEntry> flat((size_t)G * per);
  std::vector<int32_t> nentries(G);
  std::vector<uint16_t> ncount((size_t)G * S);
  for (int g = 0; g < G; g++) {
    // ascending k_enter; the kernel takes the prefix of entries that are
    // members within a depth pass and interleaves its two ends itself
    const int n = (int)groups[g].size();
    for (int j = 0; j < per; j++) {
      DasEntry d{};
      if (j < n) d = groups[g][j];
      else { d.kenter = 0x7fffffff; }
      flat[(size_t)g * per + j] = d;
    }
    nentries[g] = (int)groups[g].size();
    // N(k) = #entries with k_enter <= k (the aperture count of reading #7)
    size_t j = 0;
    for (int k = 0; k < S; k++) {
      while (j < groups[g].size() && groups[g][j].kenter <= k) j++;
      ncount[(size_t)g * S + k] = (uint16_t)j;
    }
  }
  std::vector<float4> dirs(L);
  std::vector<int32_t> ev(c.line_event, c.line_event + L);
  for (int l = 0; l < L; l++)
    dirs[l] = make_float4((float)c.line_direction[3 * l], (float)c.line_direction[3 * l + 1],
                          (float)c.line_direction[3 * l + 2], 0.f);
  // FIR per band: Hamming-windowed sinc low-pass, cutoff bw/2, DC gain 1
  // (reading #16), rotated to the complex band-pass g_j = h_j e^{+i w j}
  // (reading #18), w = 2 pi f_d / fs.  num_bands = 0: the single
  // (demod_frequency, demod_bandwidth) band with weight 1; else the bank
  // (frequency compounding).
  const int T = c.fir_taps, P = (T - 1) / 2;
  const double fs = c.sample_frequency_hz;
  h->nbands = c.num_bands > 0 ? c.num_bands : 1;
  std::vector<float2> fir((size_t)h->nbands * T);
  h->fir_c.assign((size_t)kMaxBands * (kMaxHalfTaps + 1), 0.f);
  h->fir_s.assign((size_t)kMaxBands * (kMaxHalfTaps + 1), 0.f);
  for (int b = 0; b < h->nbands; b++) {
    const double fd = c.num_bands > 0 ? c.band_center_hz[b] : c.demod_frequency_hz;
    const double fc = (c.num_bands > 0 ? c.band_bandwidth_hz[b] : c.demod_bandwidth_hz) / 2.0;
    h->band_w[b] = c.num_bands > 0 ? (float)c.band_weight[b] : 1.0f;
    std::vector<double> hd(T);
    double sum = 0;
    for (int j = -P; j <= P; j++) {
      double s = (j == 0) ? 2.0 * fc / fs : std::sin(2.0 * kPi * fc * j / fs) / (kPi * j);
      double w = (T > 1) ? 0.54 + 0.46 * std::cos(2.0 * kPi * j / (T - 1)) : 1.0;
      hd[j + P] = w * s;
      sum += w * s;
    }
    const double om = 2.0 * kPi * fd / fs;
    for (int j = -P; j <= P; j++) {
      double hj = hd[j + P] / sum;
      fir[(size_t)b * T + j + P] = make_float2((float)(hj * std::cos(om * j)), (float)(hj * std::sin(om * j)));
    }
    for (int j = 0; j <= P; j++) {
      h->fir_c[(size_t)b * (kMaxHalfTaps + 1) + j] = fir[(size_t)b * T + j + P].x;
      h->fir_s[(size_t)b * (kMaxHalfTaps + 1) + j] = fir[(size_t)b * T + j + P].y;
    }
  }
  std::vector<int32_t> cta1, cta2, cta4, ech;
  build_mirror_tables(h, line_group, groups, g_event, cta1, cta2, cta4, ech, per);
  cudaError_t e;
  if ((e = upload(&h->d_cta[0], cta1)) != cudaSuccess || (e = upload(&h->d_cta[1], cta2)) != cudaSuccess ||
      (e = upload(&h->d_cta[2], cta4)) != cudaSuccess || (e = upload(&h->d_ech, ech)) != cudaSuccess)
    return fail(e == cudaErrorMemoryAllocation ? SUPRA_E_RESOURCE : SUPRA_E_CUDA, "table upload: %s",
                cudaGetErrorString(e));
  if ((e = upload(&h->d_line_group, line_group)) != cudaSuccess ||
      (e = upload(&h->d_entries, flat)) != cudaSuccess || (e = upload(&h->d_nentries, nentries)) != cudaSuccess ||
      (e = upload(&h->d_ncount, ncount)) != cudaSuccess ||
      (e = upload(&h->d_line_dir, dirs)) != cudaSuccess || (e = upload(&h->d_line_event, ev)) != cudaSuccess ||
      (e = upload(&h->d_fir, fir)) != cudaSuccess)
    return fail(e == cudaErrorMemoryAllocation ? SUPRA_E_RESOURCE : SUPRA_E_CUDA, "table upload: %s",
                cudaGetErrorString(e));
  // Work accounting for the bench: taps and referenced input bytes.  For a
  // (line, entry) the referenced samples over k in [k_enter, S) are the
  // contiguous range [floor tau(k_enter), floor tau(S-1) + 1] (d tau / dk in
  // [0, 1]), clipped to [0, S); multi-line events take the union.
  int64_t taps = 0;
  std::vector<std::vector<std::pair<long, long>>> iv((size_t)h->E * C);
  for (int l = 0; l < L; l++) {
    const double* o = c.line_origin_mm + 3 * l;
    const double* d = c.line_direction + 3 * l;
    for (auto& de : groups[line_group[l]]) {
      taps += S - de.kenter;
      double e3[3];  // de.elem is the channel; its element from the map
      elem_pos(c, c.num_channels > 0 ? c.channel_element[(size_t)c.line_event[l] * c.num_channels + de.elem] : de.elem,
               e3);
      long a = (long)std::floor(tau_d(o, d, e3, de.kenter, dr, fs, c.speed_of_sound_mps, c.t0_s));
      long b = (long)std::floor(tau_d(o, d, e3, S - 1, dr, fs, c.speed_of_sound_mps, c.t0_s)) + 1;
      a = std::max(a, 0L);
      b = std::min(b, (long)S - 1);
      if (b >= a) iv[(size_t)c.line_event[l] * C + de.elem].push_back({a, b});
    }
  }
  int64_t ref = 0;
  for (auto& v : iv) {
    if (v.empty()) continue;
    std::sort(v.begin(), v.end());
    long ca = v[0].first, cb = v[0].second;
    for (size_t i = 1; i < v.size(); i++) {
      if (v[i].first <= cb + 1) cb = std::max(cb, v[i].second);
      else { ref += cb - ca + 1; ca = v[i].first; cb = v[i].second; }
    }
    ref += cb - ca + 1;
  }
  h->info[3] = ref * 2;
  h->info[4] = taps;
  // staging ranges (supra_bf_stage_raw): per trace the hull of its
  // referenced samples, widened by one sample each side (the device's float
  // tau may floor one sample off the binary64 value at an integer) and
  // rounded out to 16-byte chunks
  std::vector<uint32_t> siv((size_t)h->E * C, 0u);
  int64_t sbytes = 0;
  for (size_t t = 0; t < iv.size(); t++) {
    if (iv[t].empty()) continue;
    long lo = iv[t][0].first, hi = iv[t][0].second;
    for (auto& pr : iv[t]) { lo = std::min(lo, pr.first); hi = std::max(hi, pr.second); }
    const long c0 = std::max(0L, lo - 1) / 8, c1 = std::min((long)S, hi + 2 + 7) / 8;
    siv[t] = (uint32_t)c0 | ((uint32_t)c1 << 16);
    sbytes += (c1 - c0) * 16;
  }
  h->stage_bytes = sbytes;
  if ((e = upload(&h->d_stage_iv, siv)) != cudaSuccess)
    return fail(e == cudaErrorMemoryAllocation ? SUPRA_E_RESOURCE : SUPRA_E_CUDA, "table upload: %s",
                cudaGetErrorString(e));
  return SUPRA_OK;
}

// ---- scan-conversion tables (reading #21/#22; same definition as the
// analytic inverse map written out in DESIGN.md) -------------------------
void sc_axis(double u, int L, int32_t* i0, double* f) {
  if (L == 1) { *i0 = 0; *f = 0.0; return; }
  double fl = std::floor(u);
  int32_t i = (int32_t)fl;
  if (i > L - 2) i = L - 2;
  *i0 = i;
  *f = u - i;
}

supra_status build_sc_tables(supra_bf* h) {
  const supra_bf_config& c = h->cfg;
  const int nx = c.out_dims[0], ny = c.out_dims[1], nz = c.out_dims[2];
  // the line image holds S / dec samples spaced dec * dr
  const int Lx = c.num_lines_x, Ly = c.num_lines_y, S = h->Sd;
  const double dr = h->dr_mm * h->dec;
  int64_t nvalid = 0;
  cudaError_t e = cudaSuccess;
  if (c.sc_kind == SUPRA_SC_LINEAR_2D) {
    const double x0 = c.line_origin_mm[0], xL = c.line_origin_mm[3 * (Lx - 1)];
    const double pitch = (xL - x0) / (Lx - 1);
    h->h_ax.resize(nx);
    h->h_az.resize(nz);
    int64_t vx = 0, vz = 0;
    for (int ix = 0; ix < nx; ix++) {
      double X = c.out_origin_mm[0] + ix * c.out_spacing_mm[0];
      double u = (X - x0) / pitch;
      int32_t i0;
      double f;
      sc_axis(u, Lx, &i0, &f);
      bool ok = u >= 0.0 && u <= Lx - 1;
      h->h_ax[ix] = ScAxis{ok ? i0 : -1, (float)f};
      vx += ok;
    }
    for (int iz = 0; iz < nz; iz++) {
      double Z = c.out_origin_mm[2] + iz * c.out_spacing_mm[2];
      double v = Z / dr;
      int32_t k0;
      double f;
      sc_axis(v, S, &k0, &f);
      bool ok = v >= 0.0 && v <= S - 1;
      h->h_az[iz] = ScAxis{ok ? k0 : -1, (float)f};
      vz += ok;
    }
    nvalid = vx * vz;
    // per block of kScRows output rows: the k range its valid rows touch
    const int nb = (nz + kScRows - 1) / kScRows;
    std::vector<int32_t> kmin(nb, -1);
    int span = 2;
    for (int b = 0; b < nb; b++) {
      int lo = -1, hi = -1;
      for (int iz = b * kScRows; iz < std::min(nz, (b + 1) * kScRows); iz++) {
        int k0 = h->h_az[iz].i0;
        if (k0 < 0) continue;
        if (lo < 0 || k0 < lo) lo = k0;
        if (k0 > hi) hi = k0;
      }
      kmin[b] = lo;
      if (lo >= 0) span = std::max(span, hi - lo + 2);
    }
    h->slab_k = span | 1;  // odd: slab rows of consecutive lines start in distinct banks
    // per 256-column tile: the lines its valid columns touch (i0 .. i0 + 1)
    const int nc = (nx + 255) / 256;
    std::vector<int32_t> cl0(nc, 0), cnl(nc, 0);
    for (int cb = 0; cb < nc; cb++) {
      int lo = -1, hi = -1;
      for (int ix = cb * 256; ix < std::min(nx, (cb + 1) * 256); ix++) {
        int i0 = h->h_ax[ix].i0;
        if (i0 < 0) continue;
        if (lo < 0 || i0 < lo) lo = i0;
        if (i0 + 1 > hi) hi = i0 + 1;
      }
      if (lo >= 0) { cl0[cb] = lo; cnl[cb] = hi - lo + 1; }
    }
    int maxnl = 0;
    for (int v : cnl) maxnl = std::max(maxnl, v);
    // per 32-column warp group: lines touched (the tiled kernel's per-warp depth lerp)
    int maxwl = 0;
    for (int w0 = 0; w0 < nx; w0 += 32) {
      int lo = -1, hi = -1;
      for (int ix = w0; ix < std::min(nx, w0 + 32); ix++) {
        int i0 = h->h_ax[ix].i0;
        if (i0 < 0) continue;
        if (lo < 0 || i0 < lo) lo = i0;
        if (i0 + 1 > hi) hi = i0 + 1;
      }
      if (lo >= 0) maxwl = std::max(maxwl, hi - lo + 1);
    }
    h->sc_tiled = (maxnl <= kScMaxLines && h->slab_k + 3 <= kScMaxK && maxwl <= kScWarpLinesMax - 1) ? 1 : 0;  // else direct kernel
    h->sc_box_l = std::max(1, maxnl);
    h->sc_box_k = std::min(kScMaxK, (h->slab_k + 3 + 3) & ~3);   // 16-byte rows, + alignment slack
    if ((e = upload(&h->d_blk_kmin, kmin)) != cudaSuccess || (e = upload(&h->d_col_l0, cl0)) != cudaSuccess ||
        (e = upload(&h->d_col_nl, cnl)) != cudaSuccess)
      return fail(SUPRA_E_RESOURCE, "sc upload: %s", cudaGetErrorString(e));
    if ((e = upload(&h->d_ax, h->h_ax)) != cudaSuccess || (e = upload(&h->d_az, h->h_az)) != cudaSuccess)
      return fail(e == cudaErrorMemoryAllocation ? SUPRA_E_RESOURCE : SUPRA_E_CUDA, "sc upload: %s",
                  cudaGetErrorString(e));
    h->info[5] = (int64_t)(nx + nz) * sizeof(ScAxis);
  } else {
    const bool is3d = c.sc_kind == SUPRA_SC_PYRAMID_3D;
    const double fovx = c.fov_x_deg * kPi / 180.0, fovy = c.fov_y_deg * kPi / 180.0;
    const double dthx = fovx / (Lx - 1), dthy = is3d ? fovy / (Ly - 1) : 1.0;
    h->h_rows.assign((size_t)nz * ny, ScRow{0, 0, 0, 0.f});
    h->h_ent.clear();
    std::vector<ScEntry> rowbuf(nx);
    auto unorm16 = [](double f) { return (uint32_t)std::lrint(std::min(1.0, std::max(0.0, f)) * 65535.0); };
    for (int iz = 0; iz < nz; iz++) {
      const double Z = c.out_origin_mm[2] + iz * c.out_spacing_mm[2];
      for (int iy = 0; iy < ny; iy++) {
        const double Y = c.out_origin_mm[1] + iy * c.out_spacing_mm[1];
        int lo = -1, hi = -1;
        double fy_row = 0.0;
        for (int ix = 0; ix < nx; ix++) {
          const double X = c.out_origin_mm[0] + ix * c.out_spacing_mm[0];
          double ux, uy = 0.0, v;
          if (!is3d) {
            ux = std::atan2(X, Z) / dthx + (Lx - 1) / 2.0;
            v = std::sqrt(X * X + Z * Z) / dr;
          } else {
            uy = std::atan2(Y, Z) / dthy + (Ly - 1) / 2.0;
            ux = std::atan2(X, std::sqrt(Y * Y + Z * Z)) / dthx + (Lx - 1) / 2.0;
            v = std::sqrt(X * X + Y * Y + Z * Z) / dr;
          }
          bool ok = (ux >= 0.0 && ux <= Lx - 1) && (v >= 0.0 && v <= S - 1);
          if (is3d) ok = ok && (uy >= 0.0 && uy <= Ly - 1);
          int32_t i0x, i0y, k0;
          double fx, fy, fz;
          sc_axis(ux, Lx, &i0x, &fx);
          sc_axis(uy, is3d ? Ly : 1, &i0y, &fy);
          sc_axis(v, S, &k0, &fz);
          rowbuf[ix] = ScEntry{ok ? (uint32_t)((i0y * Lx + i0x) * S + k0) : kScInvalid,
                               unorm16(fx) | (unorm16(fz) << 16)};
          if (ok) {
            if (lo < 0) lo = ix;
            hi = ix + 1;
            nvalid++;
            fy_row = fy;  // u_y depends on (Y, Z) only: one value per row
          }
        }
        ScRow& r = h->h_rows[(size_t)iz * ny + iy];
        if (h->h_ent.size() + nx > 0xFFFFFFFFull) return fail(SUPRA_E_RESOURCE, "scan-conversion table too large");
        if (lo >= 0) {
          r = ScRow{lo, hi, (uint32_t)h->h_ent.size(), (float)fy_row};
          h->h_ent.insert(h->h_ent.end(), rowbuf.begin() + lo, rowbuf.begin() + hi);
        } else {
          r = ScRow{0, 0, (uint32_t)h->h_ent.size(), 0.f};
        }
      }
    }
    if ((e = upload(&h->d_rows, h->h_rows)) != cudaSuccess || (e = upload(&h->d_ent, h->h_ent)) != cudaSuccess)
      return fail(e == cudaErrorMemoryAllocation ? SUPRA_E_RESOURCE : SUPRA_E_CUDA, "sc upload: %s",
                  cudaGetErrorString(e));
    h->info[5] = (int64_t)h->h_rows.size() * sizeof(ScRow) + (int64_t)h->h_ent.size() * sizeof(ScEntry);
  }
  h->info[6] = nvalid;
  h->info[7] = 1;
  return SUPRA_OK;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  }
  return fn;
}

// raw [F][E][C][S] int16 viewed as u32 sample pairs in rows of 16 pairs:
// dims {16, S/32, C, E, F}; box {16, rows, 1, 1, fb} -- one TMA per
// (aperture entry, depth pass, frame group) fetches the pass's trace window;
// out-of-bounds rows (before 0 or past S) and frames (>= F) read as zero.
// rows_in_range < S/32 cuts the time extent (rows past it read as zeros).
bool make_raw_map(CUtensorMap* m, const void* raw, int F, int E, int C, int S, int rows, int fb,
                  int rows_in_range = -1) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t R = rows_in_range > 0 ? (cuuint64_t)rows_in_range : (cuuint64_t)S / kRowSamples;
  cuuint64_t dims[5] = {16, R, (cuuint64_t)C, (cuuint64_t)E, (cuuint64_t)F};
  cuuint64_t strides[4] = {(cuuint64_t)kRowSamples * 2, (cuuint64_t)S * 2, (cuuint64_t)C * S * 2,
                           (cuuint64_t)E * C * S * 2};
  cuuint32_t box[5] = {16, (cuuint32_t)rows, 1, 1, (cuuint32_t)fb};
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 5, const_cast<void*>(raw), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Row-cut map set (RawMaps, a kernel parameter): m[r-1] = make_raw_map with
// only r time rows in range.  Cached on the host per (raw, F, fb, nt); NULL
// on failure (the kernel then uses its single map).
const RawMaps* row_cut_maps(supra_bf* h, const void* raw, int F, int fb, int nt) {
  h->mclock++;
  supra_bf::MapSet* victim = nullptr;
  for (auto& m : h->mcache) {
    if (m.raw == raw && m.F == F && m.fb == fb && m.nt == nt) {
      m.used = h->mclock;
      return &m.maps;
    }
    if (!victim || m.used < victim->used) victim = &m;
  }
  if ((int)h->mcache.size() < supra_bf::kMapCache) {
    h->mcache.emplace_back();
    victim = &h->mcache.back();
  }
  victim->raw = nullptr;
  const int R = h->S / kRowSamples;
  for (int r = 1; r <= R; r++)
    if (!make_raw_map(&victim->maps.m[r - 1], raw, F, h->E, h->C, h->S, das_rows_nt(nt), fb, r)) return nullptr;
  victim->raw = raw;
  victim->F = F;
  victim->fb = fb;
  victim->nt = nt;
  victim->used = h->mclock;
  return &victim->maps;
}

bool is_device_ptr(const void* p, int dev) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) && a.device == dev;
}

supra_status check_launch(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return SUPRA_OK;
  return fail(SUPRA_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

void fill_log(const supra_bf* h, int& fixed, float& k1, float& k0) {
  fixed = h->cfg.reference_mode == SUPRA_REF_FIXED;
  double kk1 = 20.0 * std::log10(2.0) / h->cfg.dynamic_range_db;
  k1 = (float)kk1;
  k0 = fixed ? (float)(1.0 - kk1 * std::log2(h->cfg.reference_value)) : 1.0f;
}

}  // namespace

// DAS launch shape for `frames` frames of `nlines` lines.  Frames per CTA:
// the largest feasible (das_shape; the geometry is shared by more frames --
// smaller groups measured slower even where they fill the GPU better, e.g.
// Table-1 shapes at 64 frames FB = 8: 0.85 vs 0.65 ms).  Mirror lines per CTA
// m <= mir_max: the m with the smallest modelled time -- per CTA and tap the
// cost is G + vf * C issue slots (G ~ 13: geometry and per-entry
// bookkeeping, shared by the vf = m x frames virtual frames; C ~ 5: per-frame
// loads, conversions and FMAs), and the busiest SM runs ceil(CTAs / SMs)
// of them, a lone CTA at ~1/1.8 of the rate of two (C4p, 512 lines, one
// volume: m = 1, 2, 4 -> 0.87, 0.55, 0.76 ms, so m = 2).  Results do not
// depend on the choice (fixed per-sample member order; mirror variants
// beamform every line as (primary, variant)).
static DasShape pick_shape(supra_bf* h, int frames, int mir_max, int nlines) {
  const supra_bf_config& c = h->cfg;
  int force = 0;
#ifdef SUPRA_DEV_KNOBS
  if (const char* ev = std::getenv("SUPRA_BF_MIR")) force = std::atoi(ev);  // A/B measurements only
#endif
  DasShape best{0, 0, 1};
  double tbest = 0.0;
  for (int m = 4; m >= 1; m /= 2) {
    if (m > mir_max || (force && force != m)) continue;
    const DasShape sh = das_shape(h->frames_per_cta, h->S, frames, h->entries_per_group, c.fir_taps, m);
    if (sh.fb == 0) continue;
    const int fbr = sh.fb / m;
    const long ncta = (long)(nlines / m) * ((frames + fbr - 1) / fbr);
    const double per_sm = (double)((ncta + h->num_sms - 1) / h->num_sms);
    const double t = std::max(per_sm, 1.8) * (13.0 + 5.0 * sh.fb);
    if (best.fb == 0 || t < tbest) {
      best = sh;
      tbest = t;
    }
  }
  return best.fb ? best : das_shape(h->frames_per_cta, h->S, frames, h->entries_per_group, c.fir_taps, 1);
}

// Largest mirror order usable for lines [line0, line0 + nlines): the whole
// volume takes the layout's order; whole rows of lines take x-mirror pairs.
// t0 != 0 (or nearest-sample lookup) uses one line per CTA.
static int mirror_max(const supra_bf* h, int line0, int nlines, float t0fs) {
  if (t0fs != 0.f || h->sym_order == 1) return 1;
  if (line0 == 0 && nlines == h->L) return h->sym_order;
  const int Lx = h->cfg.num_lines_x;
  if (h->sym_x && line0 % Lx == 0 && nlines % Lx == 0) return 2;
  return 1;
}

extern "C" {

const char* supra_bf_last_error(void) { return g_err.c_str(); }

supra_status supra_bf_create(const supra_bf_config* cfg, supra_bf_t* out) {
  g_err.clear();
  if (!out) return fail(SUPRA_E_STRUCT, "out is NULL");
  *out = nullptr;
  supra_status s = validate(cfg);
  if (s != SUPRA_OK) return s;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(SUPRA_E_CUDA, "no CUDA device available (there is no CPU fallback)");
  }
  if (cfg->device < 0 || cfg->device >= ndev) return fail(SUPRA_E_STRUCT, "device %d not present", cfg->device);
  DeviceGuard dg(cfg->device);
  if (!dg.ok) return fail(SUPRA_E_CUDA, "cudaSetDevice(%d) failed", cfg->device);
  if ((int64_t)cfg->num_lines_x * cfg->num_lines_y * cfg->samples_per_channel >= (1LL << 31))
    return fail(SUPRA_E_PARAM, "L * samples_per_channel must be < 2^31");
  supra_bf* h = new supra_bf();
  h->cfg = *cfg;  // the line arrays are read by the builders below, then dropped
  h->L = cfg->num_lines_x * cfg->num_lines_y;
  h->C = cfg->num_channels > 0 ? cfg->num_channels : cfg->elements_x * cfg->elements_y;
  h->S = cfg->samples_per_channel;
  h->dec = cfg->decimation;
  h->Sd = h->S / h->dec;
  h->E = cfg->num_events;
  h->dr_mm = 1000.0 * cfg->speed_of_sound_mps / (2.0 * cfg->sample_frequency_hz);
  h->s_per_mm = cfg->sample_frequency_hz / (1000.0 * cfg->speed_of_sound_mps);
  s = build_das_tables(h);
  if (s == SUPRA_OK) s = build_sc_tables(h);
  h->cfg.line_origin_mm = nullptr;
  h->cfg.line_direction = nullptr;
  h->cfg.line_event = nullptr;
  if (s != SUPRA_OK) {
    free_all(h);
    delete h;
    return s;
  }
  // DAS launch shape
  const int maxF = cfg->max_frames_per_call;
  h->frames_per_cta = 16;  // upper bound; das_shape() picks per call
#ifdef SUPRA_DEV_KNOBS
  if (const char* ev = std::getenv("SUPRA_BF_FRAMES_PER_CTA")) {  // A/B measurements only
    int v = std::atoi(ev);
    if (v == 1 || v == 2 || v == 4 || v == 8 || v == 16) h->frames_per_cta = v;
  }
#endif
  h->mcache.reserve(supra_bf::kMapCache);  // entries never move (launches point into them)
  {
    int nsm = 0;
    if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, cfg->device) == cudaSuccess && nsm > 0)
      h->num_sms = nsm;
  }
  const bool t0zero = (float)(cfg->t0_s * cfg->sample_frequency_hz +
                              (cfg->interpolation == SUPRA_INTERP_NEAREST ? 0.5 : 0.0)) == 0.f;
  const DasShape sh = pick_shape(h, maxF, t0zero ? h->sym_order : 1, h->L);
  cudaError_t e = cudaMalloc((void**)&h->d_frame_max, sizeof(unsigned) * maxF);
  // f32 line-domain scratch [maxF][L][S/dec]: the envelope of a frame-max
  // call with a u8 line image, and supra_bf_beamform_bmode's envelope / y
  if (e == cudaSuccess) e = cudaMalloc((void**)&h->d_env, sizeof(float) * (size_t)maxF * h->L * h->Sd);
  if (e != cudaSuccess) {
    free_all(h);
    delete h;
    return fail(SUPRA_E_RESOURCE, "scratch allocation: %s", cudaGetErrorString(e));
  }
  // kernels per beamform call at max_frames_per_call: DAS (+ remainder DAS) (+ finalize)
  h->info[0] = 1 + (maxF % (sh.fb / sh.mir) != 0) + (cfg->reference_mode == SUPRA_REF_FRAME_MAX);
  h->info[1] = sh.fb / sh.mir;
  h->info[2] = (int64_t)sh.nt * kTileK;
  *out = h;
  return SUPRA_OK;
}

void supra_bf_destroy(supra_bf_t h) {
  if (!h) return;
  DeviceGuard dg(h->cfg.device);
  cudaDeviceSynchronize();
  free_all(h);
  delete h;
}

supra_status supra_bf_set_das_events(supra_bf_t h, void* before, void* after) {
  if (!h) return fail(SUPRA_E_STRUCT, "handle is NULL");
  h->ev_before = (cudaEvent_t)before;
  h->ev_after = (cudaEvent_t)after;
  return SUPRA_OK;
}

supra_status supra_bf_stage_raw(supra_bf_t h, const void* src, void* dst, int32_t frames, int64_t* bytes_per_frame,
                                void* stream) {
  g_err.clear();
  if (!h) return fail(SUPRA_E_STRUCT, "handle is NULL");
  if (bytes_per_frame) *bytes_per_frame = h->stage_bytes;
  if (frames < 0 || frames > h->cfg.max_frames_per_call)
    return fail(SUPRA_E_STRUCT, "frames %d outside [0, %d]", frames, h->cfg.max_frames_per_call);
  if (!src || !dst) return fail(SUPRA_E_STRUCT, "src and dst must not be NULL");
  if (((uintptr_t)src & 15) || ((uintptr_t)dst & 15)) return fail(SUPRA_E_STRUCT, "src / dst must be 16-byte aligned");
  if (frames == 0) return SUPRA_OK;
  DeviceGuard dg(h->cfg.device);
  if (!is_device_ptr(dst, h->cfg.device)) return fail(SUPRA_E_STRUCT, "dst is not device memory of device %d", h->cfg.device);
  cudaPointerAttributes pa;
  if (cudaPointerGetAttributes(&pa, src) != cudaSuccess) {
    cudaGetLastError();
    return fail(SUPRA_E_STRUCT, "src is neither device nor page-locked host memory");
  }
  const bool src_ok = pa.type == cudaMemoryTypeHost || ((pa.type == cudaMemoryTypeDevice || pa.type == cudaMemoryTypeManaged) &&
                                                        pa.device == h->cfg.device);
  if (!src_ok) return fail(SUPRA_E_STRUCT, "src is neither page-locked host memory nor device memory of device %d",
                           h->cfg.device);
  const void* s = pa.type == cudaMemoryTypeHost && pa.devicePointer ? pa.devicePointer : src;
  return check_launch(launch_stage_raw(s, dst, h->d_stage_iv, h->E * h->C, h->S, frames, (cudaStream_t)stream),
                      "stage kernel");
}

supra_status supra_bf_info(supra_bf_t h, int64_t* info8) {
  if (!h || !info8) return fail(SUPRA_E_STRUCT, "NULL argument");
  std::memcpy(info8, h->info, sizeof h->info);
  return SUPRA_OK;
}

// env_ext != NULL: envelope-only mode for a line range (supra_bf_beamform_lines):
// the envelope goes to env_ext, per-frame maxima to fmax_ext, no log pass.
// y_ext != NULL (fixed reference only): the log-compressed line image goes
// to y_ext as f32 whatever line_output_type is (supra_bf_beamform_bmode).
static supra_status run_das(supra_bf_t h, const void* raw, int32_t frames, int line0, int nlines, float* rf,
                            void* line_img, float* env_ext, float* fmax_ext, cudaStream_t st,
                            float* y_ext = nullptr) {
  const supra_bf_config& c = h->cfg;
  DasArgs a{};
  a.line0 = line0;
  a.nlines = nlines;
  a.raw = (const int16_t*)raw;
  a.F = frames;
  a.E = h->E;
  a.C = h->C;
  a.S = h->S;
  a.Sd = h->Sd;
  a.dec = h->dec;
  a.L = h->L;
  a.entries_per_group = h->entries_per_group;
  a.ech = h->d_ech;
  a.line_group = h->d_line_group;
  a.entries = h->d_entries;
  a.nentries = h->d_nentries;
  a.ncount = h->d_ncount;
  a.line_dir = h->d_line_dir;
  a.line_event = h->d_line_event;
  // nearest-sample lookup x~[floor(tau + 1/2)]: shift tau by 1/2, drop the fraction
  const bool nearest = c.interpolation == SUPRA_INTERP_NEAREST;
  a.t0fs = (float)(c.t0_s * c.sample_frequency_hz + (nearest ? 0.5 : 0.0));
  a.fr_scale = nearest ? 0.f : 1.f;
  a.win_a = c.window == SUPRA_WIN_HANN ? 0.5f : (c.window == SUPRA_WIN_HAMMING ? 0.54f : 1.0f);
  a.win_b = c.window == SUPRA_WIN_HANN ? 0.5f : (c.window == SUPRA_WIN_HAMMING ? 0.46f : 0.0f);
  a.normalize = c.normalize;
  a.rf = rf;
  a.do_epilogue = line_img != nullptr;
  // measurement only: 1 = TMA pipeline without the tap loop, 2 = tap loop without TMA
#ifdef SUPRA_DEV_KNOBS
  // measurement builds only (python -m paper_1711_06127_b200.build --variant=dev -DSUPRA_DEV_KNOBS):
  // SUPRA_BF_DEBUG=1 skips the tap loop, =2 the TMA staging
  a.debug_skip = std::getenv("SUPRA_BF_DEBUG") ? std::atoi(std::getenv("SUPRA_BF_DEBUG")) : 0;
#else
  a.debug_skip = 0;
#endif
  a.fir = h->d_fir;
  a.fir_taps = c.fir_taps;
  a.nbands = h->nbands;
  for (int b = 0; b < kMaxBands; b++) {
    a.band_w[b] = h->band_w[b];
    for (int j = 0; j <= kMaxHalfTaps; j++) {
      a.fir_c[b][j] = h->fir_c[(size_t)b * (kMaxHalfTaps + 1) + j];
      a.fir_s[b][j] = h->fir_s[(size_t)b * (kMaxHalfTaps + 1) + j];
    }
  }
  fill_log(h, a.ref_fixed, a.log_k1, a.log_k0);
  a.y_type = c.line_output_type;
  if (y_ext) {
    a.do_epilogue = 1;
    a.y_out = y_ext;
    a.y_type = SUPRA_T_F32;
  } else if (env_ext) {
    a.do_epilogue = 1;
    a.ref_fixed = 0;
    a.env_out = env_ext;
    a.frame_max = (unsigned*)fmax_ext;  // non-negative floats: bit order = value order
    cudaError_t e = cudaMemsetAsync(fmax_ext, 0, sizeof(float) * frames, st);
    if (e != cudaSuccess) return check_launch(e, "memset frame_max");
  } else if (line_img) {
    if (a.ref_fixed) {
      a.y_out = line_img;
    } else {
      a.env_out = (c.line_output_type == SUPRA_T_F32) ? (float*)line_img : h->d_env;
      a.frame_max = h->d_frame_max;
      cudaError_t e = cudaMemsetAsync(h->d_frame_max, 0, sizeof(unsigned) * frames, st);
      if (e != cudaSuccess) return check_launch(e, "memset frame_max");
    }
  }
  {
    const void* out = a.ref_fixed ? a.y_out : (const void*)a.env_out;
    a.vec_out = out != nullptr && ((uintptr_t)out & 15) == 0;
  }
  // Mirror lines and frames per CTA (build_mirror_tables, pick_shape):
  // results do not depend on the choice.  Mirror lines for whole-volume
  // calls with t0 = 0 only.
  const int mmax = mirror_max(h, line0, nlines, a.t0fs);
  const DasShape sh = pick_shape(h, frames, mmax, nlines);
  const int fbr = sh.fb / sh.mir;  // frames per CTA
  a.cta = h->d_cta[sh.mir == 4 ? 2 : (sh.mir == 2 ? 1 : 0)];
  a.cta_base = line0 / sh.mir;
  // Frames in groups of fbr per CTA; a remainder (frames % fbr) runs as a
  // second, programmatically-serialised launch with its own (smaller) shape
  // that fills the SMs the first grid's tail leaves idle.
  const int Fmain = (frames / fbr) * fbr;
  const int rem = frames - Fmain;
  const DasShape sh2 = rem ? pick_shape(h, rem, mmax, nlines) : sh;
  const int fbr2 = sh2.fb / sh2.mir;
  const size_t frame_bytes = (size_t)h->E * h->C * h->S * sizeof(int16_t);
  CUtensorMap tm, tm2;
  if (!make_raw_map(&tm, raw, Fmain, h->E, h->C, h->S, das_rows_nt(sh.nt), fbr) ||
      (rem && !make_raw_map(&tm2, (const char*)raw + Fmain * frame_bytes, rem, h->E, h->C, h->S,
                            das_rows_nt(sh2.nt), fbr2)))
    return fail(SUPRA_E_CUDA, "cuTensorMapEncodeTiled failed for the raw buffer");
  a.fbase = 0;
  a.Fmap = Fmain;
  a.pdl_trigger = rem > 0;
  a.pdl_wait_end = 0;
  // exact trace windows for the multi-pass / multi-frame kernel (the
  // single-frame kernel's windows run to the end of the record anyway)
  bool exact = true;
#ifdef SUPRA_DEV_KNOBS
  if (std::getenv("SUPRA_BF_NO_ROWCUT")) exact = false;  // A/B measurements only
#endif
  // the warp-split kernel only for a single-frame call; remainders of a
  // multi-frame call use das_fused_kernel (batch-independent results)
  // (not for mirror-symmetric layouts: there every launch, whatever its
  // lines per CTA, gives bitwise the same result)
  const bool warp_ok = frames == 1 && h->sym_order == 1;
  const bool warp1 = warp_ok && das_warp_ok(sh.fb, h->S, a.t0fs);
  static const RawMaps kNoMaps{};
  const RawMaps* m1 = (exact && !warp1) ? row_cut_maps(h, raw, Fmain, fbr, sh.nt) : nullptr;
  a.row_cut = m1 != nullptr;
  if (h->ev_before) cudaEventRecord(h->ev_before, st);
  supra_status s = check_launch(launch_das(tm, a, m1 ? *m1 : kNoMaps, sh, warp_ok, st), "das kernel");
  if (s == SUPRA_OK && rem) {
    DasArgs a2 = a;
    a2.fbase = Fmain;
    a2.Fmap = rem;
    a2.pdl_trigger = 0;
    a2.pdl_wait_end = 1;
    const RawMaps* m2 = exact ? row_cut_maps(h, (const char*)raw + Fmain * frame_bytes, rem, fbr2, sh2.nt)
                              : nullptr;
    a2.row_cut = m2 != nullptr;
    a2.cta = h->d_cta[sh2.mir == 4 ? 2 : (sh2.mir == 2 ? 1 : 0)];
    a2.cta_base = line0 / sh2.mir;
    s = check_launch(launch_das(tm2, a2, m2 ? *m2 : kNoMaps, sh2, false, st), "das kernel (remainder frames)");
  }
  if (h->ev_after) cudaEventRecord(h->ev_after, st);
  if (s != SUPRA_OK || !line_img || a.ref_fixed || env_ext) return s;
  FinalizeArgs fa{};
  fa.env = a.env_out;
  fa.per_frame = (long long)h->L * h->Sd;
  fa.frame_stride = fa.per_frame;
  fa.F = frames;
  fa.frame_max = h->d_frame_max;
  fa.DR_k = a.log_k1;
  fa.y_out = line_img;
  fa.y_type = c.line_output_type;
  return check_launch(launch_finalize(fa, st), "finalize kernel");
}

supra_status supra_bf_beamform(supra_bf_t h, const void* raw, int32_t frames, float* rf, void* line_img,
                               void* stream) {
  g_err.clear();
  if (!h) return fail(SUPRA_E_STRUCT, "handle is NULL");
  if (frames < 0 || frames > h->cfg.max_frames_per_call)
    return fail(SUPRA_E_STRUCT, "frames %d outside [0, %d]", frames, h->cfg.max_frames_per_call);
  if (!rf && !line_img) return fail(SUPRA_E_STRUCT, "both rf and line_img are NULL");
  if (frames == 0) return SUPRA_OK;
  if (!raw || ((uintptr_t)raw & 15)) return fail(SUPRA_E_STRUCT, "raw must be a 16-byte aligned device pointer");
  DeviceGuard dg(h->cfg.device);
  const int dev = h->cfg.device;
  if (!is_device_ptr(raw, dev)) return fail(SUPRA_E_STRUCT, "raw is not device memory of device %d", dev);
  if (rf && !is_device_ptr(rf, dev)) return fail(SUPRA_E_STRUCT, "rf is not device memory of device %d", dev);
  if (line_img && !is_device_ptr(line_img, dev))
    return fail(SUPRA_E_STRUCT, "line_img is not device memory of device %d", dev);
  cudaError_t pe = cudaGetLastError();
  if (pe != cudaSuccess) return fail(SUPRA_E_CUDA, "pending CUDA error: %s", cudaGetErrorString(pe));
  return run_das(h, raw, frames, 0, h->L, rf, line_img, nullptr, nullptr, (cudaStream_t)stream);
}

supra_status supra_bf_beamform_lines(supra_bf_t h, const void* raw, int32_t frames, int32_t line_first,
                                     int32_t line_count, float* env, float* frame_max, void* stream) {
  g_err.clear();
  if (!h) return fail(SUPRA_E_STRUCT, "handle is NULL");
  if (frames < 0 || frames > h->cfg.max_frames_per_call)
    return fail(SUPRA_E_STRUCT, "frames %d outside [0, %d]", frames, h->cfg.max_frames_per_call);
  if (line_first < 0 || line_count < 0 || line_first + (int64_t)line_count > h->L)
    return fail(SUPRA_E_STRUCT, "line range [%d, %d + %d) outside [0, %d)", line_first, line_first, line_count,
                h->L);
  if (!env || !frame_max) return fail(SUPRA_E_STRUCT, "env and frame_max must not be NULL");
  if (frames == 0 || line_count == 0) {
    if (frames > 0) {
      DeviceGuard dg(h->cfg.device);
      return check_launch(cudaMemsetAsync(frame_max, 0, sizeof(float) * frames, (cudaStream_t)stream),
                          "memset frame_max");
    }
    return SUPRA_OK;
  }
  if (!raw || ((uintptr_t)raw & 15)) return fail(SUPRA_E_STRUCT, "raw must be a 16-byte aligned device pointer");
  DeviceGuard dg(h->cfg.device);
  const int dev = h->cfg.device;
  if (!is_device_ptr(raw, dev) || !is_device_ptr(env, dev) || !is_device_ptr(frame_max, dev))
    return fail(SUPRA_E_STRUCT, "raw / env / frame_max are not device memory of device %d", dev);
  cudaError_t pe = cudaGetLastError();
  if (pe != cudaSuccess) return fail(SUPRA_E_CUDA, "pending CUDA error: %s", cudaGetErrorString(pe));
  return run_das(h, raw, frames, line_first, line_count, nullptr, nullptr, env, frame_max, (cudaStream_t)stream);
}

supra_status supra_bf_log_compress(supra_bf_t h, const float* env, int32_t frames, int32_t line_first,
                                   int32_t line_count, const float* frame_max, void* line_img, void* stream) {
  g_err.clear();
  if (!h) return fail(SUPRA_E_STRUCT, "handle is NULL");
  if (frames < 0 || frames > h->cfg.max_frames_per_call)
    return fail(SUPRA_E_STRUCT, "frames %d outside [0, %d]", frames, h->cfg.max_frames_per_call);
  if (line_first < 0 || line_count < 0 || line_first + (int64_t)line_count > h->L)
    return fail(SUPRA_E_STRUCT, "line range [%d, %d + %d) outside [0, %d)", line_first, line_first, line_count,
                h->L);
  if (!env || !line_img) return fail(SUPRA_E_STRUCT, "env and line_img must not be NULL");
  const supra_bf_config& c = h->cfg;
  if (!frame_max && c.reference_mode != SUPRA_REF_FIXED)
    return fail(SUPRA_E_STRUCT, "frame_max is NULL but reference_mode is FRAME_MAX");
  if (frames == 0 || line_count == 0) return SUPRA_OK;
  DeviceGuard dg(c.device);
  const int dev = c.device;
  if (!is_device_ptr(env, dev) || !is_device_ptr(line_img, dev) || (frame_max && !is_device_ptr(frame_max, dev)))
    return fail(SUPRA_E_STRUCT, "env / frame_max / line_img are not device memory of device %d", dev);
  int fixed;
  float k1, k0;
  fill_log(h, fixed, k1, k0);
  FinalizeArgs fa{};
  fa.env = env;
  fa.per_frame = (long long)line_count * h->Sd;
  fa.frame_stride = (long long)h->L * h->Sd;
  fa.offset = (long long)line_first * h->Sd;
  fa.F = frames;
  fa.frame_max = fixed ? nullptr : (const unsigned*)frame_max;
  fa.fixed_ref = (float)c.reference_value;
  fa.DR_k = k1;
  fa.y_out = line_img;
  fa.y_type = c.line_output_type;
  return check_launch(launch_finalize(fa, (cudaStream_t)stream), "log kernel");
}

supra_status supra_bf_envelope_log(supra_bf_t h, const float* rf, int32_t frames, void* line_img, void* stream) {
  g_err.clear();
  if (!h) return fail(SUPRA_E_STRUCT, "handle is NULL");
  if (frames < 0 || frames > h->cfg.max_frames_per_call)
    return fail(SUPRA_E_STRUCT, "frames %d outside [0, %d]", frames, h->cfg.max_frames_per_call);
  if (!rf || !line_img) return fail(SUPRA_E_STRUCT, "rf and line_img must not be NULL");
  if (frames == 0) return SUPRA_OK;
  DeviceGuard dg(h->cfg.device);
  const int dev = h->cfg.device;
  if (!is_device_ptr(rf, dev) || !is_device_ptr(line_img, dev))
    return fail(SUPRA_E_STRUCT, "rf / line_img are not device memory of device %d", dev);
  cudaStream_t st = (cudaStream_t)stream;
  const supra_bf_config& c = h->cfg;
  EnvArgs a{};
  a.rf = rf;
  a.F = frames;
  a.L = h->L;
  a.S = h->S;
  a.Sd = h->Sd;
  a.dec = h->dec;
  a.fir = h->d_fir;
  a.fir_taps = c.fir_taps;
  a.nbands = h->nbands;
  for (int b = 0; b < kMaxBands; b++) a.band_w[b] = h->band_w[b];
  fill_log(h, a.ref_fixed, a.log_k1, a.log_k0);
  a.y_type = c.line_output_type;
  if (a.ref_fixed) {
    a.y_out = line_img;
  } else {
    a.env_out = (c.line_output_type == SUPRA_T_F32) ? (float*)line_img : h->d_env;
    a.frame_max = h->d_frame_max;
    cudaError_t e = cudaMemsetAsync(h->d_frame_max, 0, sizeof(unsigned) * frames, st);
    if (e != cudaSuccess) return check_launch(e, "memset frame_max");
  }
  supra_status s = check_launch(launch_envlog(a, st), "envlog kernel");
  if (s != SUPRA_OK || a.ref_fixed) return s;
  FinalizeArgs fa{};
  fa.env = a.env_out;
  fa.per_frame = (long long)h->L * h->Sd;
  fa.frame_stride = fa.per_frame;
  fa.F = frames;
  fa.frame_max = h->d_frame_max;
  fa.DR_k = a.log_k1;
  fa.y_out = line_img;
  fa.y_type = c.line_output_type;
  return check_launch(launch_finalize(fa, st), "finalize kernel");
}

static supra_status run_sc(supra_bf_t h, const void* line_img, int in_type, const unsigned* frame_max,
                           int32_t frames, void* img, uint8_t* mask, cudaStream_t st) {
  const supra_bf_config& c = h->cfg;
  ScArgs a{};
  a.line_img = line_img;
  a.in_type = in_type;
  a.frame_max = frame_max;
  a.DR_k = (float)(20.0 * std::log10(2.0) / c.dynamic_range_db);
  a.F = frames;
  a.Lx = c.num_lines_x;
  a.Ly = c.num_lines_y;
  a.S = h->Sd;  // line-image samples (S / decimation)
  a.nx = c.out_dims[0];
  a.ny = c.out_dims[1];
  a.nz = c.out_dims[2];
  a.img = img;
  a.out_type = c.sc_output_type;
  a.mask = mask;
  a.ax = h->d_ax;
  a.az = h->d_az;
  a.blk_kmin = h->d_blk_kmin;
  a.slab_k = h->slab_k;
  a.col_l0 = h->d_col_l0;
  a.col_nl = h->d_col_nl;
  a.tiled = h->sc_tiled;
  a.slab_box_k = h->sc_box_k;
  a.slab_box_l = h->sc_box_l;
  a.rows = h->d_rows;
  a.ent = h->d_ent;
  a.is3d = c.sc_kind == SUPRA_SC_PYRAMID_3D;
  // bulk-copy staging of the slab: 16-byte aligned line segments (f32; a
  // u8 line image needs the tensor copy below, else the kernel's own loads)
  const bool in8 = in_type == SUPRA_T_U8;
  const int esz = in8 ? 1 : 4;
  const bool slab_ok = c.sc_kind == SUPRA_SC_LINEAR_2D && h->sc_tiled && (h->Sd * esz) % 16 == 0 &&
                       ((uintptr_t)line_img & 15) == 0;
  a.slab_tma = (slab_ok && !in8) ? 1 : 0;
  // u8: segments start 16-byte aligned (k & ~15), box width a multiple of 16
  if (in8) a.slab_box_k = std::min(256, (h->slab_k + 15 + 15) & ~15);
  // one 2-D tensor map over the [frames Lx][Sd] line image: a single TMA per
  // (tile, frame) instead of one bulk copy per line (fallback if the encode
  // fails)
  CUtensorMap slab_map;
  const CUtensorMap* sm = nullptr;
  if (slab_ok && frames > 0) {
    EncodeTiledFn fn = encode_fn();
    cuuint64_t dims[2] = {(cuuint64_t)h->Sd, (cuuint64_t)frames * c.num_lines_x};
    cuuint64_t strides[1] = {(cuuint64_t)h->Sd * esz};
    cuuint32_t box[2] = {(cuuint32_t)a.slab_box_k, (cuuint32_t)h->sc_box_l};
    cuuint32_t es[2] = {1, 1};
    if (fn && fn(&slab_map, in8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                 const_cast<void*>(line_img), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS) {
      sm = &slab_map;
      a.slab_tma = 2;
    }
  }
  if (c.sc_kind == SUPRA_SC_LINEAR_2D) return check_launch(launch_sc_linear(a, sm, st), "sc_linear kernel");
  const int lbytes = (int)std::min<int64_t>(INT32_MAX, (int64_t)h->L * h->Sd * (in_type == SUPRA_T_U8 ? 1 : 4));
  return check_launch(launch_sc_table(a, lbytes, st), "sc_table kernel");
}

supra_status supra_bf_scanconvert(supra_bf_t h, const void* line_img, int32_t frames, void* img, uint8_t* mask,
                                  void* stream) {
  g_err.clear();
  if (!h) return fail(SUPRA_E_STRUCT, "handle is NULL");
  if (frames < 0 || frames > h->cfg.max_frames_per_call)
    return fail(SUPRA_E_STRUCT, "frames %d outside [0, %d]", frames, h->cfg.max_frames_per_call);
  if (!line_img || !img) return fail(SUPRA_E_STRUCT, "line_img and img must not be NULL");
  if (frames == 0) return SUPRA_OK;
  DeviceGuard dg(h->cfg.device);
  const int dev = h->cfg.device;
  if (!is_device_ptr(line_img, dev) || !is_device_ptr(img, dev) || (mask && !is_device_ptr(mask, dev)))
    return fail(SUPRA_E_STRUCT, "line_img / img / mask are not device memory of device %d", dev);
  return run_sc(h, line_img, h->cfg.line_output_type, nullptr, frames, img, mask, (cudaStream_t)stream);
}

supra_status supra_bf_beamform_bmode(supra_bf_t h, const void* raw, int32_t frames, void* img, uint8_t* mask,
                                     void* stream) {
  g_err.clear();
  if (!h) return fail(SUPRA_E_STRUCT, "handle is NULL");
  if (frames < 0 || frames > h->cfg.max_frames_per_call)
    return fail(SUPRA_E_STRUCT, "frames %d outside [0, %d]", frames, h->cfg.max_frames_per_call);
  if (!raw || !img) return fail(SUPRA_E_STRUCT, "raw and img must not be NULL");
  if (frames == 0) return SUPRA_OK;
  if ((uintptr_t)raw & 15) return fail(SUPRA_E_STRUCT, "raw must be a 16-byte aligned device pointer");
  DeviceGuard dg(h->cfg.device);
  const int dev = h->cfg.device;
  if (!is_device_ptr(raw, dev) || !is_device_ptr(img, dev) || (mask && !is_device_ptr(mask, dev)))
    return fail(SUPRA_E_STRUCT, "raw / img / mask are not device memory of device %d", dev);
  cudaError_t pe = cudaGetLastError();
  if (pe != cudaSuccess) return fail(SUPRA_E_CUDA, "pending CUDA error: %s", cudaGetErrorString(pe));
  cudaStream_t st = (cudaStream_t)stream;
  const bool fixed = h->cfg.reference_mode == SUPRA_REF_FIXED;
  // DAS + envelope (frame max) into the handle's f32 scratch -- or, with a
  // fixed reference, DAS + envelope + log straight into it -- then scan
  // conversion from the scratch (log-compressing each corner on load)
  supra_status s = run_das(h, raw, frames, 0, h->L, nullptr, nullptr, fixed ? nullptr : h->d_env,
                           fixed ? nullptr : (float*)h->d_frame_max, st, fixed ? h->d_env : nullptr);
  if (s != SUPRA_OK) return s;
  return run_sc(h, h->d_env, SUPRA_T_F32, fixed ? nullptr : h->d_frame_max, frames, img, mask, st);
}

supra_status supra_bf_sc_indices(supra_bf_t h, uint8_t* valid, int32_t* idx) {
  if (!h || !valid || !idx) return fail(SUPRA_E_STRUCT, "NULL argument");
  const supra_bf_config& c = h->cfg;
  // entries encode base = (i0y Lx + i0x) Sd + k0 over the (decimated)
  // line image (build_sc_tables)
  const int nx = c.out_dims[0], ny = c.out_dims[1], nz = c.out_dims[2], S = h->Sd, Lx = c.num_lines_x;
  size_t n = 0;
  for (int iz = 0; iz < nz; iz++)
    for (int iy = 0; iy < ny; iy++)
      for (int ix = 0; ix < nx; ix++, n++) {
        idx[3 * n] = idx[3 * n + 1] = idx[3 * n + 2] = 0;
        if (c.sc_kind == SUPRA_SC_LINEAR_2D) {
          const ScAxis &ax = h->h_ax[ix], &az = h->h_az[iz];
          valid[n] = ax.i0 >= 0 && az.i0 >= 0;
          idx[3 * n] = ax.i0;
          idx[3 * n + 2] = az.i0;
        } else {
          const ScRow& r = h->h_rows[(size_t)iz * ny + iy];
          valid[n] = 0;
          if (ix >= r.xlo && ix < r.xhi) {
            const uint32_t b = h->h_ent[r.off + (ix - r.xlo)].base;
            if (b != kScInvalid) {
              valid[n] = 1;
              idx[3 * n + 2] = b % S;
              const int li = (int)(b / S);
              idx[3 * n] = li % Lx;
              idx[3 * n + 1] = li / Lx;
            }
          }
        }
      }
  return SUPRA_OK;
}

}  // extern "C"
