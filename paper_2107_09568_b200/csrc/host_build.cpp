// host_build.cpp — host side of iga_build_tables: validation, I_coo (Eq. 56),
// DofMap (reading R10), full symmetric CSR pattern and the atomic-free gather
// lists of K4 (reading R9), Gauss rules and the interpolation operator (R1).
// Everything here is integer/topology work done once per handle.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <type_traits>
#include <omp.h>
#include "internal.h"

namespace iga {

static thread_local char g_err[1024] = "";
void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
const char *get_error() { return g_err; }

// n-point Gauss–Legendre rule mapped to [0,1], nodes ascending (Newton on P_n).
iga_status upload_topology(Handle &h) {
  auto up = [&](void **dst, const void *src, size_t bytes) -> bool {
    if (cudaMalloc(dst, std::max<size_t>(bytes, 8)) != cudaSuccess) { set_error("cudaMalloc(%zu) failed", bytes); return false; }
    if (bytes && cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice) != cudaSuccess) { set_error("H2D copy failed"); return false; }
    return true;
  };
  std::vector<int32_t> pinfo(3 * (h.n_patches + 1), 0);
  for (int pi = 0; pi <= h.n_patches; ++pi) {
    pinfo[3 * pi] = h.pcol[pi] / IGA_KCHUNK;
    if (pi < h.n_patches) {
      pinfo[3 * pi + 1] = h.patches[pi].ctrl_off;
      pinfo[3 * pi + 2] = h.patches[pi].n_ctrl;
    }
  }
  if (!up((void **)&h.d_node_map, h.node_map.data(), h.node_map.size() * 4) ||
      !up((void **)&h.d_pairA, h.pairA.data(), h.pairA.size() * 4) ||
      !up((void **)&h.d_pairB, h.pairB.data(), h.pairB.size() * 4) ||
      !up((void **)&h.d_brow_ptr, h.brow_ptr.data(), h.brow_ptr.size() * 8) ||
      !up((void **)&h.d_bcol, h.bcol.data(), h.bcol.size() * 4) ||
      !up((void **)&h.d_rowinfo, h.rowinfo.data(), h.rowinfo.size() * 8) ||
      !up((void **)&h.d_emap, h.emap.data(), h.emap.size() * 4) ||
      !up((void **)&h.d_k4d, h.k4d.data(), h.k4d.size() * sizeof(K4Desc)) ||
      !up((void **)&h.d_slot_tr, h.slot_tr.data(), h.slot_tr.size()) ||
      !up((void **)&h.d_k5_pair, h.k5_pair.data(), h.k5_pair.size() * 4) ||
      !up((void **)&h.d_k5_col, h.k5_col.data(), h.k5_col.size() * 4) ||
      !up((void **)&h.d_tperm, h.tperm.data(), h.tperm.size()) ||
      !up((void **)&h.d_cperm, h.cperm.data(), h.cperm.size() * 2) ||
      !up((void **)&h.d_rowdesc, h.rowdesc.data(), h.rowdesc.size() * sizeof(int4)) ||
      !up((void **)&h.d_g1len, h.g1len.data(), h.g1len.size() * 2) ||
      !up((void **)&h.d_g2len, h.g2len.data(), h.g2len.size() * 2) ||
      !up((void **)&h.d_g1slot, h.g1slot.data(), h.g1slot.size() * 4) ||
      !up((void **)&h.d_g2slot, h.g2slot.data(), h.g2slot.size() * 4) ||
      !up((void **)&h.d_sA_ptr, h.sA_ptr.data(), h.sA_ptr.size() * 4) ||
      !up((void **)&h.d_sA_slot, h.sA_slot.data(), h.sA_slot.size() * 4) ||
      !up((void **)&h.d_inv_ptr, h.inv_ptr.data(), h.inv_ptr.size() * 8) ||
      !up((void **)&h.d_inv_ent, h.inv_ent.data(), h.inv_ent.size() * 4) ||
      !up((void **)&h.d_patch_info, pinfo.data(), pinfo.size() * 4) ||
      !up((void **)&h.d_k5_gphys, h.k5_gphys.data(), h.k5_gphys.size() * 4) ||
      !up((void **)&h.d_k5_mode, h.k5_mode.data(), h.k5_mode.size()) ||
      !up((void **)&h.d_k5_extra, h.k5_extra.data(), h.k5_extra.size() * 4))
    return IGA_ENOMEM;
  if (cudaMalloc((void **)&h.d_side, std::max<size_t>(8, (size_t)h.n_slot_cap * h.d * h.d * 8)) != cudaSuccess) {
    set_error("cudaMalloc of the multi-contribution slots failed");
    return IGA_ENOMEM;
  }
  // the epilogue maps live on the device only from here on
  std::vector<int64_t>().swap(h.rowinfo);
  std::vector<int32_t>().swap(h.emap);
  std::vector<MultiBlock>().swap(h.mblk);
  std::vector<int32_t>().swap(h.mslot0);
  std::vector<int32_t>().swap(h.mperm);
  std::vector<int64_t>().swap(h.inv_ptr);
  std::vector<int32_t>().swap(h.inv_ent);
  std::vector<uint8_t>().swap(h.slot_tr);
  std::vector<K4Desc>().swap(h.k4d);
  return IGA_OK;
}

void gauss_legendre01(int n, double *x, double *w) {
  const double pi = 3.14159265358979323846;
  for (int i = 0; i < (n + 1) / 2; ++i) {
    double z = std::cos(pi * (i + 0.75) / (n + 0.5)), pp = 1.0;
    for (int it = 0; it < 100; ++it) {
      double p1 = 1.0, p2 = 0.0;
      for (int j = 1; j <= n; ++j) {
        double p3 = p2;
        p2 = p1;
        p1 = ((2.0 * j - 1.0) * z * p2 - (j - 1.0) * p3) / j;
      }
      pp = n * (z * p1 - p2) / (z * z - 1.0);
      double z1 = z;
      z = z1 - p1 / pp;
      if (std::fabs(z - z1) < 1e-16) break;
    }
    double wi = 2.0 / ((1.0 - z * z) * pp * pp);
    // z > 0 is the (i)-th largest root
    x[n - 1 - i] = 0.5 * (1.0 + z);
    x[i] = 0.5 * (1.0 - z);
    w[n - 1 - i] = 0.5 * wi;
    w[i] = 0.5 * wi;
  }
}

static double binom(int n, int k) {
  double r = 1.0;
  for (int i = 1; i <= k; ++i) r = r * (n - k + i) / i;
  return r;
}

// Gauss–Jordan inverse with partial pivoting (n <= 5).
static bool invert(int n, const double *a, double *inv) {
  double m[5][10];
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < 2 * n; ++j) m[i][j] = j < n ? a[i * n + j] : (j - n == i ? 1.0 : 0.0);
  for (int c = 0; c < n; ++c) {
    int piv = c;
    for (int r = c + 1; r < n; ++r)
      if (std::fabs(m[r][c]) > std::fabs(m[piv][c])) piv = r;
    if (std::fabs(m[piv][c]) < 1e-300) return false;
    for (int j = 0; j < 2 * n; ++j) std::swap(m[c][j], m[piv][j]);
    double f = 1.0 / m[c][c];
    for (int j = 0; j < 2 * n; ++j) m[c][j] *= f;
    for (int r = 0; r < n; ++r)
      if (r != c) {
        double g = m[r][c];
        for (int j = 0; j < 2 * n; ++j) m[r][j] -= g * m[c][j];
      }
  }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) inv[i * n + j] = m[i][j + n];
  return true;
}

// ---------------------------------------------------------------------------
// validation of one spline's knots (open, normalised, multiplicities)
static bool check_knots(const iga_spline &s, int k, const char *what, int idx,
                        std::vector<double> &U, std::vector<int> &el) {
  int p = s.degree[k], nk = s.n_knots[k];
  if (p < 1 || p > IGA_MAXP) { set_error("%s %d: degree[%d]=%d outside [1,%d]", what, idx, k, p, IGA_MAXP); return false; }
  if (nk < 2 * (p + 1) || !s.knots[k]) { set_error("%s %d: too few knots in direction %d", what, idx, k); return false; }
  U.assign(s.knots[k], s.knots[k] + nk);
  for (int i = 0; i + 1 < nk; ++i)
    if (!(U[i] <= U[i + 1])) { set_error("%s %d: knots of direction %d not non-decreasing", what, idx, k); return false; }
  for (int i = 0; i <= p; ++i)
    if (U[i] != 0.0 || U[nk - 1 - i] != 1.0) { set_error("%s %d: knot vector %d not open on [0,1]", what, idx, k); return false; }
  if (!(U[p + 1] > 0.0) || !(U[nk - p - 2] < 1.0)) { set_error("%s %d: end knot multiplicity > degree+1 in direction %d", what, idx, k); return false; }
  for (int i = p + 1; i < nk - p - 1;) {
    int j = i;
    while (j + 1 < nk - p - 1 && U[j + 1] == U[i]) ++j;
    if (j - i + 1 > p) { set_error("%s %d: interior knot multiplicity > degree in direction %d", what, idx, k); return false; }
    i = j + 1;
  }
  el.clear();
  for (int i = p; i < nk - p - 1; ++i)
    if (U[i] < U[i + 1]) el.push_back(i);
  return true;
}

struct UF {
  std::vector<int64_t> par;
  explicit UF(int64_t n) : par(n) { std::iota(par.begin(), par.end(), 0); }
  int64_t find(int64_t x) {
    while (par[x] != x) { par[x] = par[par[x]]; x = par[x]; }
    return x;
  }
  void unite(int64_t a, int64_t b) {
    a = find(a); b = find(b);
    if (a == b) return;
    if (a < b) par[b] = a; else par[a] = b;
  }
};

// the macro map ℳ = F (Eq. 4): knots, elements per direction, NURBS weights
iga_status parse_macro(Handle &h, const iga_spline *macro, int d) {
  if (!macro) { set_error("no macro topology"); return IGA_EINVAL; }
  if (macro->dim != d) { set_error("macro dim %d != tile dim %d", macro->dim, d); return IGA_EINVAL; }
  h.n_cp = 1;
  h.n_tiles = 1;
  for (int k = 0; k < 3; ++k) { h.pm[k] = 0; h.mn[k] = 1; h.mel[k] = 1; }
  for (int k = 0; k < d; ++k) {
    if (!check_knots(*macro, k, "macro", 0, h.mknots[k], h.mel_span[k])) return IGA_EINVAL;
    h.pm[k] = macro->degree[k];
    h.mn[k] = macro->n_knots[k] - macro->degree[k] - 1;
    h.mel[k] = (int)h.mel_span[k].size();
    h.n_cp *= h.mn[k];
    h.n_tiles *= h.mel[k];
  }
  h.mweights.clear();
  if (macro->weights) {   // NURBS macro map (NEXT N4)
    h.mweights.assign(macro->weights, macro->weights + h.n_cp);
    for (double w : h.mweights)
      if (!(w > 0.0)) { set_error("macro weights must be positive"); return IGA_EINVAL; }
  }
  return IGA_OK;
}

// projection degrees per direction (Eq. 21 with p_π per direction, the twist's 3, 3, 4)
iga_status set_degrees(Handle &h, const int *q) {
  h.q = 0;
  h.iso = true;
  h.npi = 1;
  for (int k = 0; k < 3; ++k) h.qv[k] = 0;
  for (int k = 0; k < h.d; ++k) {
    if (q[k] < 0 || q[k] > IGA_MAXQ) { set_error("q[%d]=%d outside [0,%d]", k, q[k], IGA_MAXQ); return IGA_EINVAL; }
    h.qv[k] = q[k];
    h.q = std::max(h.q, q[k]);
    h.iso = h.iso && q[k] == q[0];
    h.npi *= q[k] + 1;
  }
  h.nk = h.d * h.d * h.npi;
  h.kstride = (h.nk + IGA_KCHUNK - 1) / IGA_KCHUNK * IGA_KCHUNK;
  // Eq. 38-reduced contraction layout
  auto up = [](int x, int m) { return (x + m - 1) / m * m; };
  h.n_p1 = h.d * (h.d + 1) / 2;
  h.n_p2 = h.d * (h.d - 1) / 2;
  h.tpc = h.d == 3 ? 8 : 16;
  const int k1 = up(h.n_p1 * h.npi, 4), k2 = up(h.n_p2 * h.npi, 4);
  h.k3_split = k1 / 4;
  h.k3_steps = (k1 + k2) / 4;
  h.ks3 = up(k1 + k2, IGA_KCHUNK);
  h.k5_split = up(h.n_p1 * h.npi, 8);
  h.k5_kap = h.k5_split + up(h.n_p2 * h.npi, 8);
  return IGA_OK;
}

iga_status build_host(Handle &h, const iga_spline *tile, int n_patches, const iga_interface *ifc,
                      int n_ifc, const iga_spline *macro, const int *q, int n_gauss, const iga_shard *shard) {
  if (!tile || n_patches <= 0 || !macro || !q) { set_error("no tile patches, macro topology or q"); return IGA_EINVAL; }
  const int d = tile[0].dim;
  if (d != 2 && d != 3) { set_error("dim must be 2 or 3 (got %d)", d); return IGA_EINVAL; }
  if (macro->dim != d) { set_error("macro dim %d != tile dim %d", macro->dim, d); return IGA_EINVAL; }
  h.d = d;
  {
    const iga_status st = set_degrees(h, q);
    if (st != IGA_OK) return st;
  }
  h.p = tile[0].degree[0];
  h.n_patches = n_patches;
  h.patches.resize(n_patches);
  int off = 0;
  for (int pi = 0; pi < n_patches; ++pi) {
    const iga_spline &s = tile[pi];
    PatchInfo &P = h.patches[pi];
    if (s.dim != d) { set_error("tile patch %d: dim %d != %d", pi, s.dim, d); return IGA_EINVAL; }
    P.n_ctrl = 1;
    P.n_spans = 1;
    for (int k = 0; k < 3; ++k) { P.deg[k] = 0; P.n[k] = 1; P.n_span[k] = 1; }
    for (int k = 0; k < d; ++k) {
      if (!check_knots(s, k, "tile patch", pi, P.knots[k], P.el_span[k])) return IGA_EINVAL;
      if (s.degree[k] != h.p) { set_error("tile patch %d: all tile directions/patches must share degree p=%d", pi, h.p); return IGA_EINVAL; }
      P.deg[k] = s.degree[k];
      P.n[k] = s.n_knots[k] - s.degree[k] - 1;
      P.n_span[k] = (int)P.el_span[k].size();
      P.n_ctrl *= P.n[k];
      P.n_spans *= P.n_span[k];
    }
    if (!s.ctrl) { set_error("tile patch %d: no control points", pi); return IGA_EINVAL; }
    if (s.weights) { set_error("tile patch %d: rational (NURBS) tile patches are not supported", pi); return IGA_EINVAL; }
    P.ctrl.assign(s.ctrl, s.ctrl + (size_t)P.n_ctrl * d);
    for (double c : P.ctrl)
      if (!(c >= -1e-12 && c <= 1.0 + 1e-12)) { set_error("tile patch %d: control point outside [0,1]^d (Eq. 10 condition)", pi); return IGA_EINVAL; }
    P.ctrl_off = off;
    off += P.n_ctrl;
  }
  h.n_local_ctrl = off;
  {
    const iga_status st = parse_macro(h, macro, d);
    if (st != IGA_OK) return st;
  }
  h.n_g = n_gauss > 0 ? n_gauss : h.p + (h.q + 2) / 2;   // R3 with the largest q_k
  if (h.n_g > 12) { set_error("n_gauss=%d > 12", h.n_g); return IGA_EINVAL; }

  // ---- I_coo per patch (Eq. 56; R8: supports share a knot span) -------------
  h.M = 0;
  h.pairA.clear();
  h.pairB.clear();
  int span_off = 0;
  for (int pi = 0; pi < n_patches; ++pi) {
    PatchInfo &P = h.patches[pi];
    // 1D: function a is nonzero on knot spans a..a+p; spans must be elements
    std::vector<std::vector<char>> share(d);
    for (int k = 0; k < d; ++k) {
      int n = P.n[k], p = P.deg[k];
      share[k].assign((size_t)n * n, 0);
      for (int s : P.el_span[k])
        for (int a = std::max(0, s - p); a <= std::min(n - 1, s); ++a)
          for (int b = std::max(0, s - p); b <= std::min(n - 1, s); ++b) share[k][(size_t)a * n + b] = 1;
    }
    P.row_off = (int)h.M;
    int cnt = 0;
    for (int A = 0; A < P.n_ctrl; ++A) {
      int ia[3] = {A % P.n[0], (A / P.n[0]) % P.n[1], A / (P.n[0] * P.n[1])};
      for (int B = A; B < P.n_ctrl; ++B) {
        int ib[3] = {B % P.n[0], (B / P.n[0]) % P.n[1], B / (P.n[0] * P.n[1])};
        bool ok = true;
        for (int k = 0; k < d && ok; ++k) ok = share[k][(size_t)ia[k] * P.n[k] + ib[k]];
        if (ok) {
          h.pairA.push_back(P.ctrl_off + A);
          h.pairB.push_back(P.ctrl_off + B);
          ++cnt;
        }
      }
    }
    P.n_nz = cnt;
    h.M += cnt;
    P.span_off = span_off;
    span_off += P.n_spans;
  }

  // ---- DofMap (R10) ------------------------------------------------------------
  const double TOL = 1e-10;
  auto pos = [&](int loc, int k) -> double {
    for (int pi = n_patches - 1; pi >= 0; --pi)
      if (loc >= h.patches[pi].ctrl_off) return h.patches[pi].ctrl[(size_t)(loc - h.patches[pi].ctrl_off) * d + k];
    return 0.0;
  };
  auto close = [&](int a, int b, const double *shift) {
    for (int k = 0; k < d; ++k)
      if (std::fabs(pos(a, k) - shift[k] - pos(b, k)) > TOL) return false;
    return true;
  };
  std::vector<std::pair<int, int>> intra;
  for (int f = 0; f < n_ifc; ++f) {
    const iga_interface &I = ifc[f];
    if (I.patch_a < 0 || I.patch_a >= n_patches || I.patch_b < 0 || I.patch_b >= n_patches || I.dir_a < 0 ||
        I.dir_a >= d || I.dir_b < 0 || I.dir_b >= d) { set_error("interface %d: bad patch/direction", f); return IGA_EINVAL; }
    auto members = [&](int pi, int dir, int side) {
      std::vector<int> m;
      const PatchInfo &P = h.patches[pi];
      int want = side ? P.n[dir] - 1 : 0;
      for (int A = 0; A < P.n_ctrl; ++A) {
        int ii[3] = {A % P.n[0], (A / P.n[0]) % P.n[1], A / (P.n[0] * P.n[1])};
        if (ii[dir] == want) m.push_back(P.ctrl_off + A);
      }
      return m;
    };
    auto ma = members(I.patch_a, I.dir_a, I.side_a), mb = members(I.patch_b, I.dir_b, I.side_b);
    double zero[3] = {0, 0, 0};
    for (int a : ma) {
      int hit = -1, nh = 0;
      for (int b : mb)
        if (close(a, b, zero)) { hit = b; ++nh; }
      if (nh != 1) { set_error("interface %d: control point %d of patch %d has %d partners", f, a, I.patch_a, nh); return IGA_ENONCONFORMING; }
      intra.push_back({a, hit});
    }
  }
  std::vector<std::vector<std::pair<int, int>>> inter(d);
  for (int k = 0; k < d; ++k) {
    std::vector<int> hi, lo;
    for (int a = 0; a < h.n_local_ctrl; ++a) {
      if (std::fabs(pos(a, k) - 1.0) <= TOL) hi.push_back(a);
      if (std::fabs(pos(a, k)) <= TOL) lo.push_back(a);
    }
    if (hi.size() != lo.size()) { set_error("tile faces xi_%d=0 and xi_%d=1 carry %zu vs %zu control points", k, k, lo.size(), hi.size()); return IGA_ENONCONFORMING; }
    double e[3] = {0, 0, 0};
    e[k] = 1.0;
    for (int a : hi) {
      int hit = -1, nh = 0;
      for (int b : lo)
        if (close(a, b, e)) { hit = b; ++nh; }
      if (nh != 1) { set_error("tile face xi_%d=1: control point %d has %d partners on xi_%d=0", k, a, nh, k); return IGA_ENONCONFORMING; }
      inter[k].push_back({a, hit});
    }
  }
  const int64_t nl = h.n_local_ctrl, nt = h.n_tiles;
  if (nt * nl >= (int64_t(1) << 31)) { set_error("n_tiles * n_local_ctrl exceeds int32"); return IGA_ELIMIT; }
  UF uf(nt * nl);
  int64_t stride[3] = {1, h.mel[0], (int64_t)h.mel[0] * h.mel[1]};
  for (int64_t t = 0; t < nt; ++t) {
    for (auto &pr : intra) uf.unite(t * nl + pr.first, t * nl + pr.second);
    int64_t tk[3] = {t % h.mel[0], (t / h.mel[0]) % h.mel[1], t / stride[2]};
    for (int k = 0; k < d; ++k)
      if (tk[k] < h.mel[k] - 1)
        for (auto &pr : inter[k]) uf.unite(t * nl + pr.first, (t + stride[k]) * nl + pr.second);
  }
  h.node_map.assign(nt * nl, -1);
  {
    std::vector<int32_t> id(nt * nl, -1);
    int64_t next = 0;
    for (int64_t f = 0; f < nt * nl; ++f) {
      int64_t r = uf.find(f);
      if (id[r] < 0) id[r] = (int32_t)next++;
      h.node_map[f] = id[r];
    }
    h.n_nodes = next;
  }
  h.n_dof = h.n_nodes * d;
  for (int64_t t = 0; t < nt; ++t)
    for (int pi = 0; pi < n_patches; ++pi) {
      const PatchInfo &P = h.patches[pi];
      std::vector<int32_t> ids(h.node_map.begin() + t * nl + P.ctrl_off, h.node_map.begin() + t * nl + P.ctrl_off + P.n_ctrl);
      std::sort(ids.begin(), ids.end());
      for (size_t i = 1; i < ids.size(); ++i)
        if (ids[i] == ids[i - 1]) { set_error("tile %lld patch %d: two control points merged", (long long)t, pi); return IGA_ENONCONFORMING; }
    }

  // ---- shard: slab of macro-element layers along the slowest direction
  // plus one halo layer; owned rows = nodes first appearing in the slab (a contiguous
  // id range, since ids follow first appearance over tiles).  Every tile containing an
  // owned node lies in the slab or the halo layer, so owned rows are complete.
  h.n_tiles_glob = nt;
  h.n_nodes_glob = h.n_nodes;
  {
    int64_t tb = 0, te_own = nt, te = nt, n0 = 0, n1 = h.n_nodes;
    if (shard && shard->n_shards > 1) {
      const int kd = d - 1;
      const int64_t layers = h.mel[kd], layer = nt / layers;
      if (shard->shard < 0 || shard->shard >= shard->n_shards || shard->n_shards > layers) {
        set_error("shard %d of %d: need 0 <= shard < n_shards <= %lld element layers", shard->shard, shard->n_shards,
                  (long long)layers);
        return IGA_EINVAL;
      }
      const int64_t l0 = shard->shard * layers / shard->n_shards, l1 = (shard->shard + 1) * layers / shard->n_shards;
      tb = l0 * layer;
      te_own = l1 * layer;
      te = std::min(nt, te_own + layer);
      int32_t mx = -1;
      for (int64_t f = 0; f < tb * nl; ++f) mx = std::max(mx, h.node_map[f]);
      n0 = mx + 1;
      for (int64_t f = tb * nl; f < te_own * nl; ++f) mx = std::max(mx, h.node_map[f]);
      n1 = mx + 1;
      h.n_shards = shard->n_shards;
      h.shard = shard->shard;
    }
    h.t_base = tb;
    h.n_tiles_own = te_own - tb;
    h.n_tiles = te - tb;
    h.node_base = n0;
    h.n_nodes = n1 - n0;
    if (tb != 0 || te != nt)
      h.node_map = std::vector<int32_t>(h.node_map.begin() + tb * nl, h.node_map.begin() + te * nl);
  }

  // ---- pattern (R9) and the K3 fused-epilogue maps ------------------------------
  // Every (tile t, table row r) with I = node(A_r), J = node(B_r) contributes the local
  // block L to K(I,J) and Lᵀ to K(J,I).  Blocks with exactly one contribution are
  // written straight from the K3 epilogue (emap holds rank(J in row I) | rank(I in row
  // J) << 16); blocks with several contributions (tile faces, patch interfaces) get
  // one side slot per contribution and are summed in a fixed order by K4.
  // (local tiles lt = t - t_base; owned rows i = I - node_base; columns stay global)
  const int64_t lnt = h.n_tiles, n0 = h.node_base;
  if (lnt * h.M >= (int64_t(1) << 40)) { set_error("n_tiles * table rows exceeds 2^40"); return IGA_ELIMIT; }
  const int64_t nn = h.n_nodes;
  auto own = [&](int64_t I) { return I >= n0 && I < n0 + nn; };
  std::vector<int64_t> cnt(nn + 1, 0);
  std::vector<std::atomic<int64_t>> acnt(nn);
  for (auto &a : acnt) a.store(0, std::memory_order_relaxed);
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < lnt; ++t)
    for (int64_t r = 0; r < h.M; ++r) {
      int32_t I = h.node_map[t * nl + h.pairA[r]], J = h.node_map[t * nl + h.pairB[r]];
      if (own(I)) acnt[I - n0].fetch_add(1, std::memory_order_relaxed);
      if (I != J && own(J)) acnt[J - n0].fetch_add(1, std::memory_order_relaxed);
    }
  for (int64_t i = 0; i < nn; ++i) cnt[i + 1] = cnt[i] + acnt[i].load(std::memory_order_relaxed);
  h.n_contrib = cnt[nn];
  // key = J << 40 | t*M + r  << 1 | transposed   (transposed: this row's node is B's)
  std::vector<uint64_t> keys(h.n_contrib);
  for (int64_t i = 0; i < nn; ++i) acnt[i].store(cnt[i], std::memory_order_relaxed);
  std::vector<uint64_t> kcol(h.n_contrib);   // J per key (sort by (J, code))
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < lnt; ++t)
    for (int64_t r = 0; r < h.M; ++r) {
      int32_t I = h.node_map[t * nl + h.pairA[r]], J = h.node_map[t * nl + h.pairB[r]];
      uint64_t code = (uint64_t)(t * h.M + r) << 1;
      if (own(I)) {
        const int64_t k = acnt[I - n0].fetch_add(1, std::memory_order_relaxed);
        keys[k] = code;
        kcol[k] = (uint64_t)J;
      }
      if (I != J && own(J)) {
        const int64_t k = acnt[J - n0].fetch_add(1, std::memory_order_relaxed);
        keys[k] = code | 1u;
        kcol[k] = (uint64_t)I;
      }
    }
  std::vector<int64_t> nnzb(nn + 1, 0);
  int bad_cnt = 0;
#pragma omp parallel reduction(+ : bad_cnt)
  {
    std::vector<std::pair<uint64_t, uint64_t>> tmp;
#pragma omp for schedule(dynamic, 1024)
    for (int64_t i = 0; i < nn; ++i) {
      const int64_t k0 = cnt[i], k1 = cnt[i + 1];
      tmp.resize(k1 - k0);
      for (int64_t k = k0; k < k1; ++k) tmp[k - k0] = {kcol[k], keys[k]};
      std::sort(tmp.begin(), tmp.end());
      for (int64_t k = k0; k < k1; ++k) { kcol[k] = tmp[k - k0].first; keys[k] = tmp[k - k0].second; }
      int64_t nb = 0;
      for (int64_t k = k0; k < k1; ++k)
        if (k == k0 || kcol[k] != kcol[k - 1]) ++nb;
      if (nb >= 32768) ++bad_cnt;
      nnzb[i + 1] = nb;
    }
  }
  if (bad_cnt) { set_error("a block row has >= 32768 blocks (emap rank width)"); return IGA_ELIMIT; }
  h.brow_ptr.assign(nn + 1, 0);
  for (int64_t i = 0; i < nn; ++i) h.brow_ptr[i + 1] = h.brow_ptr[i] + nnzb[i + 1];
  h.n_blocks = h.brow_ptr[nn];
  h.nnz = h.n_blocks * d * d;
  if (h.n_blocks >= (int64_t(1) << 39)) { set_error("too many blocks"); return IGA_ELIMIT; }
  h.bcol.assign(h.n_blocks, 0);
  h.emap.assign(lnt * h.M, 0);
  uint16_t *e16 = reinterpret_cast<uint16_t *>(h.emap.data());
  std::vector<int64_t> mcount(nn + 1, 0), scount(nn + 1, 0), ntrue(nn + 1, 0);
  // pass 1: block columns, direct ranks, multi-block counts (canonical I <= J)
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t i = 0; i < nn; ++i) {
    int64_t b = h.brow_ptr[i] - 1;
    for (int64_t k = cnt[i]; k < cnt[i + 1];) {
      int64_t k1 = k + 1;
      while (k1 < cnt[i + 1] && kcol[k1] == kcol[k]) ++k1;
      ++b;
      const int64_t J = (int64_t)kcol[k];
      h.bcol[b] = (int32_t)J;
      if (k1 - k == 1) {
        const uint64_t code = keys[k] >> 1;
        e16[2 * code + (keys[k] & 1u)] = (uint16_t)(b - h.brow_ptr[i]);
      } else if (J >= i + n0 || !own(J)) {   // canonical row of a shared block
        mcount[i + 1] += 1;
        scount[i + 1] += (k1 - k + 1) & ~int64_t(1);   // slot ranges start at even slots (K4's 16-B loads)
        ntrue[i + 1] += k1 - k;
      }
      k = k1;
    }
  }
  for (int64_t i = 0; i < nn; ++i) {
    mcount[i + 1] += mcount[i];
    scount[i + 1] += scount[i];
    ntrue[i + 1] += ntrue[i];
  }
  h.n_multi = mcount[nn];
  h.n_slots = ntrue[nn];       // contributions
  h.n_slot_cap = scount[nn];   // side slots allocated (each block's range starts at an even slot)
  if (h.n_slot_cap >= (int64_t(1) << 31) - 1) { set_error("too many multi-contribution slots"); return IGA_ELIMIT; }
  h.mblk.assign(h.n_multi, MultiBlock{});
  h.mslot0.assign(h.n_multi + 1, 0);
  h.slot_tr.assign(h.n_slot_cap, 0);
  h.mslot0[h.n_multi] = (int32_t)h.n_slot_cap;
  std::vector<int32_t> nslots(h.n_multi);   // contributions per multi block (its slot range may end in a pad slot)
  auto rank_in_row = [&](int64_t row, int64_t col) -> int64_t {
    const int32_t *bb = h.bcol.data() + h.brow_ptr[row], *ee = h.bcol.data() + h.brow_ptr[row + 1];
    return std::lower_bound(bb, ee, (int32_t)col) - bb;
  };
  // pass 2: multi blocks and their slots (needs all of bcol)
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t i = 0; i < nn; ++i) {
    int64_t m = mcount[i], sl = scount[i], b = h.brow_ptr[i] - 1;
    for (int64_t k = cnt[i]; k < cnt[i + 1];) {
      int64_t k1 = k + 1;
      while (k1 < cnt[i + 1] && kcol[k1] == kcol[k]) ++k1;
      ++b;
      const int64_t J = (int64_t)kcol[k];
      if (k1 - k > 1 && (J >= i + n0 || !own(J))) {
        MultiBlock &mb = h.mblk[m];
        mb.off_ij = (int64_t)d * d * h.brow_ptr[i] + (int64_t)d * (b - h.brow_ptr[i]);
        mb.stride_i = (int32_t)(d * (h.brow_ptr[i + 1] - h.brow_ptr[i]));
        if (own(J)) {
          const int64_t j = J - n0;
          mb.off_ji = (int64_t)d * d * h.brow_ptr[j] + (int64_t)d * rank_in_row(j, i + n0);
          mb.stride_j = (int32_t)(d * (h.brow_ptr[j + 1] - h.brow_ptr[j]));
        } else {   // row J belongs to another shard
          mb.off_ji = -1;
          mb.stride_j = 0;
        }
        h.mslot0[m] = (int32_t)sl;
        for (int64_t kk = k; kk < k1; ++kk, ++sl) {
          h.slot_tr[sl] = (uint8_t)(keys[kk] & 1u);
          h.emap[keys[kk] >> 1] = -(int32_t)(sl + 1);
        }
        nslots[m] = (int32_t)(k1 - k);
        sl += (k1 - k) & 1;   // pad to an even slot
        ++m;
      }
      k = k1;
    }
  }
  std::vector<uint64_t>().swap(keys);
  std::vector<uint64_t>().swap(kcol);
  {   // K4 transposed pass order: multi blocks sorted by (J, I) = (row of K(J,I), its column)
    std::vector<int64_t> rowJ(h.n_multi), colI(h.n_multi);
#pragma omp parallel for schedule(static)
    for (int64_t m = 0; m < h.n_multi; ++m) {
      const MultiBlock &mb = h.mblk[m];
      // off_ji = d²·brow_ptr[J] + d·rank: recover J by binary search in brow_ptr
      const int64_t b = (mb.off_ji / d) / d;   // block index lower bound of row J
      const int64_t J = mb.off_ji < 0 ? INT64_MAX
                                      : std::upper_bound(h.brow_ptr.begin(), h.brow_ptr.end(), b) - h.brow_ptr.begin() - 1;
      rowJ[m] = J;
      colI[m] = mb.off_ij;   // (I, J) order already sorts by I within row J
    }
    h.mperm.resize(h.n_multi);
    std::iota(h.mperm.begin(), h.mperm.end(), 0);
    std::stable_sort(h.mperm.begin(), h.mperm.end(), [&](int32_t x, int32_t y) {
      return rowJ[x] != rowJ[y] ? rowJ[x] < rowJ[y] : colI[x] < colI[y];
    });
    h.k4d.assign(2 * h.n_multi, K4Desc{});
    int bad_ns = 0;
#pragma omp parallel for schedule(static) reduction(+ : bad_ns)
    for (int64_t m = 0; m < h.n_multi; ++m)
      if (nslots[m] >= K4_MAX_NS) ++bad_ns;
    if (bad_ns) { set_error("a shared block has >= %d contributions", K4_MAX_NS); return IGA_ELIMIT; }
#pragma omp parallel for schedule(static)
    for (int64_t m = 0; m < h.n_multi; ++m) {
      const MultiBlock &b1 = h.mblk[m];
      const int64_t mt = h.mperm[m];
      const MultiBlock &b2 = h.mblk[mt];
      const bool dg1 = b1.off_ij == b1.off_ji, dg2 = b2.off_ij == b2.off_ji;
      h.k4d[m] = k4_desc(b1.off_ij, b1.stride_i, h.mslot0[m], nslots[m], dg1);
      // diagonal blocks are complete after pass 1; off_ji < 0: row J belongs to another shard
      h.k4d[h.n_multi + m] = k4_desc(b2.off_ji >= 0 && !dg2 ? b2.off_ji : -1, b2.stride_j, h.mslot0[mt], nslots[mt], false);
    }
  }
  h.rowinfo.assign(lnt * nl, 0);
#pragma omp parallel for schedule(static)
  for (int64_t f = 0; f < lnt * nl; ++f) {
    const int64_t I = h.node_map[f];
    h.rowinfo[f] = own(I) ? (h.brow_ptr[I - n0] << 24) | (h.brow_ptr[I - n0 + 1] - h.brow_ptr[I - n0]) : -1;
  }

  // ---- operand layouts: K3 A rows, coefficient rows, K5a padded reduction columns --
  h.Mpad = (h.M + IGA_K3_BM * IGA_K3_CL - 1) / (IGA_K3_BM * IGA_K3_CL) * (IGA_K3_BM * IGA_K3_CL);
  h.Npad = (lnt + h.tpc - 1) / h.tpc * IGA_GEMM_BN;   // blocks of tpc tiles (sym layout)
  h.pcol.assign(n_patches + 1, 0);
  h.max_patch_ctrl = 0;
  for (int pi = 0; pi < n_patches; ++pi) {
    h.pcol[pi + 1] = h.pcol[pi] + (h.patches[pi].n_nz + IGA_KCHUNK - 1) / IGA_KCHUNK * IGA_KCHUNK;
    h.max_patch_ctrl = std::max(h.max_patch_ctrl, h.patches[pi].n_ctrl);
  }
  if (h.max_patch_ctrl >= 32768) { set_error("tile patch with >= 32768 control points"); return IGA_ELIMIT; }
  h.Kp = h.pcol[n_patches];
  // K3 epilogue, transposed pass: within each 64-row block, rows ordered by (B, A) so that
  // neighbouring threads write neighbouring blocks of CSR row node(B)
  auto block_perm = [&](auto &perm, int BMb, int64_t rows) {
    perm.assign(rows, 0);
    for (int64_t m0 = 0; m0 < rows; m0 += BMb) {
      std::vector<int> idx(BMb);
      std::iota(idx.begin(), idx.end(), 0);
      std::stable_sort(idx.begin(), idx.end(), [&](int x, int y) {
        const int64_t rx = m0 + x, ry = m0 + y;
        if (rx >= h.M || ry >= h.M) return rx < h.M && ry >= h.M;
        return h.pairB[rx] != h.pairB[ry] ? h.pairB[rx] < h.pairB[ry] : h.pairA[rx] < h.pairA[ry];
      });
      for (int k = 0; k < BMb; ++k) perm[m0 + k] = (typename std::decay_t<decltype(perm)>::value_type)idx[k];
    }
  };
  block_perm(h.tperm, IGA_K3_BM, h.Mpad);
  // clustered K3 (IGA_K3_CL > 1): the transposed pass pools the CL row blocks of a cluster, so
  // the (J,I) blocks of one CSR row J that come from neighbouring A (neighbouring row blocks)
  // leave as one run
  block_perm(h.cperm, IGA_K3_BM * IGA_K3_CL, h.Mpad);
  // per-row scatter descriptor (row pair and its (B, A)-order partner), one 16-byte load
  h.rowdesc.assign(h.Mpad, int4{-1, -1, 0, 0});
  for (int64_t r = 0; r < h.Mpad; ++r) {
    const int64_t m0 = r / IGA_K3_BM * IGA_K3_BM, rt = m0 + h.tperm[r];
    int4 &q = h.rowdesc[r];
    q.z = h.tperm[r];
    if (r < h.M) q.x = h.pairA[r] | (h.pairB[r] << 16);
    if (rt < h.M) q.y = h.pairA[rt] | (h.pairB[rt] << 16);
  }
  // matrix-free apply maps (tile-independent, NEXT N1)
  {
    h.g1len.assign(h.Mpad, 0);
    h.g2len.assign(h.Mpad, 0);
    h.g1slot.assign(h.Mpad, -1);
    h.g2slot.assign(h.Mpad, -1);
    std::vector<int32_t> key;   // local control point receiving each slot
    for (int64_t m0 = 0; m0 < h.Mpad; m0 += IGA_K3_BM) {
      for (int e = 0; e < IGA_K3_BM && m0 + e < h.M;) {   // runs of equal A in row order
        int f = e + 1;
        while (f < IGA_K3_BM && m0 + f < h.M && h.pairA[m0 + f] == h.pairA[m0 + e]) ++f;
        for (int x = e; x < f; ++x) h.g1len[m0 + x] = (uint16_t)((f - e) | ((x - e) << 8));   // length | position << 8
        h.g1slot[m0 + e] = (int32_t)key.size();
        key.push_back(h.pairA[m0 + e]);
        e = f;
      }
      for (int q = 0; q < IGA_K3_BM;) {   // runs of equal B in tperm order (diagonal rows add 0)
        const int64_t r = m0 + h.tperm[m0 + q];
        if (r >= h.M) break;
        int f = q + 1;
        while (f < IGA_K3_BM && m0 + h.tperm[m0 + f] < h.M && h.pairB[m0 + h.tperm[m0 + f]] == h.pairB[r]) ++f;
        for (int x = q; x < f; ++x) h.g2len[m0 + x] = (uint16_t)((f - q) | ((x - q) << 8));
        h.g2slot[m0 + q] = (int32_t)key.size();
        key.push_back(h.pairB[r]);
        q = f;
      }
    }
    h.P = (int64_t)key.size();
    h.sA_ptr.assign(nl + 1, 0);
    for (int32_t k : key) h.sA_ptr[k + 1]++;
    for (int64_t a = 0; a < nl; ++a) h.sA_ptr[a + 1] += h.sA_ptr[a];
    h.sA_slot.assign(h.P, 0);
    std::vector<int32_t> fill(h.sA_ptr.begin(), h.sA_ptr.end() - 1);
    for (int64_t p = 0; p < h.P; ++p) h.sA_slot[fill[key[p]]++] = (int32_t)p;
    // owned node -> (local tile, A) occurrences, sorted by (tile, A)
    h.inv_ptr.assign(nn + 1, 0);
    for (int64_t f = 0; f < lnt * nl; ++f)
      if (own(h.node_map[f])) h.inv_ptr[h.node_map[f] - n0 + 1]++;
    for (int64_t i = 0; i < nn; ++i) h.inv_ptr[i + 1] += h.inv_ptr[i];
    h.inv_ent.assign(h.inv_ptr[nn], 0);
    std::vector<int64_t> fi(h.inv_ptr.begin(), h.inv_ptr.end() - 1);
    for (int64_t f = 0; f < lnt * nl; ++f)
      if (own(h.node_map[f])) h.inv_ent[fi[h.node_map[f] - n0]++] = (int32_t)f;
  }
  h.k5_pair.assign(h.Kp, -1);
  h.k5_col.assign(h.M, 0);
  for (int pi = 0; pi < n_patches; ++pi) {
    const PatchInfo &P = h.patches[pi];
    for (int i = 0; i < P.n_nz; ++i) {
      const int64_t r = P.row_off + i;
      h.k5_pair[h.pcol[pi] + i] = (h.pairA[r] - P.ctrl_off) | ((h.pairB[r] - P.ctrl_off) << 16);
      h.k5_col[r] = h.pcol[pi] + i;
    }
  }
  // K5a CTA height IGA_K3_BM κ rows
  h.k5_rows = (h.k5_kap + IGA_K5_BM - 1) / IGA_K5_BM * IGA_K5_BM;
  {   // K5a κ-group placement (longest-processing-time first over blocks, then sub-partitions):
      // block b, sub-partition q holds the warps q + 4h (h < W/4), two 8-row groups each
    constexpr int W = IGA_K5_BM / 16, SL = 2 * (W / 4);   // warps per block, slots per sub-partition
    const int G1 = h.k5_split / 8, G2 = (h.k5_kap - h.k5_split) / 8, nbk = (int)(h.k5_rows / IGA_K5_BM);
    std::vector<int> sload(nbk * 4, 0), bload(nbk, 0);
    std::vector<std::vector<int>> slot(nbk * 4);
    for (int g = 0; g < G1 + G2; ++g) {
      const int w = g < G1 ? (d == 3 ? 2 : 3) : 1;   // DMMAs per k-step: 6 : 3 (3D), 6 : 2 (2D)
      int bb = -1, ss = -1;
      for (int b = 0; b < nbk; ++b) {
        bool free_ = false;
        for (int q = 0; q < 4; ++q) free_ = free_ || (int)slot[b * 4 + q].size() < SL;
        if (free_ && (bb < 0 || bload[b] < bload[bb])) bb = b;
      }
      for (int q = 0; q < 4; ++q)
        if ((int)slot[bb * 4 + q].size() < SL && (ss < 0 || sload[bb * 4 + q] < sload[bb * 4 + ss])) ss = q;
      slot[bb * 4 + ss].push_back(g);
      sload[bb * 4 + ss] += w;
      bload[bb] += w;
    }
    h.k5_gphys.assign(h.k5_rows / 8, 0);   // unused tail groups: 0 (never read)
    h.k5_mode.assign(nbk * W, 0);
    auto part = [&](int g) { return g < 0 ? 0 : (g < G1 ? 1 : 2); };
    for (int b = 0; b < nbk; ++b)
      for (int q = 0; q < 4; ++q) {
        std::vector<int> v = slot[b * 4 + q];   // part-1 groups first (heavier), empty slots last
        while ((int)v.size() < SL) v.push_back(-1);
        std::stable_sort(v.begin(), v.end(), [&](int x, int y) {
          const int px = part(x) == 0 ? 3 : part(x), py = part(y) == 0 ? 3 : part(y);
          return px < py;
        });
        for (int hh = 0; hh < W / 4; ++hh) {   // warp q + 4hh: the hh-th heaviest with the hh-th lightest
          const int warp = q + 4 * hh;
          int g0 = v[hh], g1 = v[SL - 1 - hh];
          if (part(g1) != 0 && (part(g0) == 0 || part(g1) < part(g0))) std::swap(g0, g1);
          h.k5_mode[b * W + warp] = (uint8_t)(part(g0) * 3 + part(g1));
          if (g0 >= 0) h.k5_gphys[g0] = (b * W + warp) * 2;
          if (g1 >= 0) h.k5_gphys[g1] = (b * W + warp) * 2 + 1;
        }
      }
    // K5g column split (3D; part-1 group = 6 column tiles, part-2 = 3): LPT leaves loads
    // (m+3, m, m, m) DMMAs per k-step when the unit count is 1 mod 4 (cfg5: 42/39/39/39).
    // The heavy sub-partition keeps columns 0-3 of one of its part-1 groups (mode 9/10) and
    // hands columns 4 and 5 to one warp on each of two light sub-partitions (mode 11/12,
    // an extra single-column piece): 40/40/40/39.  K5g only (K5a has no modes 9-12).
    h.k5_extra.assign(nbk * W, -1);
#ifndef IGA_EXPERIMENT_NO_K5G
    if (d == 3 && sens_xw_fits(h))
      for (int b = 0; b < nbk; ++b) {
        int L[4], hq = 0;
        for (int q = 0; q < 4; ++q) L[q] = 3 * sload[b * 4 + q];
        for (int q = 1; q < 4; ++q) if (L[q] > L[hq]) hq = q;
        int nlow = 0;
        for (int q = 0; q < 4; ++q) nlow += q != hq && L[q] == L[hq] - 3;
        if (nlow != 3) continue;
        int wh = -1;   // heavy warp with a part-1 first group: prefer (1,2)
        for (int hh = 0; hh < W / 4 && wh < 0; ++hh) if (h.k5_mode[b * W + hq + 4 * hh] == 5) wh = hq + 4 * hh;
        for (int hh = 0; hh < W / 4 && wh < 0; ++hh) if (h.k5_mode[b * W + hq + 4 * hh] == 4) wh = hq + 4 * hh;
        if (wh < 0) continue;
        int wl[2], nl_ = 0;   // one light warp of mode (2,2) or (1,2) on two light sub-partitions
        for (int q = 0; q < 4 && nl_ < 2; ++q) {
          if (q == hq) continue;
          int w = -1;
          for (int hh = 0; hh < W / 4 && w < 0; ++hh) if (h.k5_mode[b * W + q + 4 * hh] == 8) w = q + 4 * hh;
          for (int hh = 0; hh < W / 4 && w < 0; ++hh) if (h.k5_mode[b * W + q + 4 * hh] == 5 && q + 4 * hh != wh) w = q + 4 * hh;
          if (w >= 0) wl[nl_++] = w;
        }
        if (nl_ < 2) continue;
        h.k5_mode[b * W + wh] = h.k5_mode[b * W + wh] == 5 ? 10 : 9;
        for (int i = 0; i < 2; ++i) {
          h.k5_mode[b * W + wl[i]] = h.k5_mode[b * W + wl[i]] == 8 ? 11 : 12;
          h.k5_extra[b * W + wl[i]] = (wh * 2) | ((4 + i) << 16);
        }
      }
#endif
  }

  if (k5x_smem_bytes(d, h.max_patch_ctrl) > 227 * 1024) { set_error("tile patch too large for the K5 shared-memory staging (%d control points)", h.max_patch_ctrl); return IGA_ELIMIT; }

  // ---- projection operator (R1: interpolation at the q_k+1 Gauss nodes) -----------
  {
    const iga_status st = set_projection(h, 0);
    if (st != IGA_OK) return st;
  }
  return IGA_OK;
}

// Π1 for an m-point Gauss rule in one direction (Eqs. 23-24: M_π d = r_π with
// [M_π]_kl = Σ_i w_i N_k(x_i) N_l(x_i), (r_π)_k = Σ_i w_i N_k(x_i) f(x_i), tensorised):
// Pi1 = (VᵀWV)⁻¹VᵀW, V[i][c] = B_c^q(x_i).  m = q+1 reduces to V⁻¹ (interpolation at the
// Gauss nodes, reading R1), computed directly.
static iga_status projection_1d(int q, int m, double *x, double *P) {
  const int q1 = q + 1;
  double w[IGA_MAXM], V[IGA_MAXM * (IGA_MAXQ + 1)];
  gauss_legendre01(m, x, w);
  for (int i = 0; i < m; ++i)
    for (int c = 0; c <= q; ++c) V[i * q1 + c] = binom(q, c) * std::pow(x[i], c) * std::pow(1.0 - x[i], q - c);
  if (m == q1) {
    if (!invert(q1, V, P)) { set_error("singular interpolation matrix"); return IGA_EINVAL; }
    return IGA_OK;
  }
  double Mpi[(IGA_MAXQ + 1) * (IGA_MAXQ + 1)], Minv[(IGA_MAXQ + 1) * (IGA_MAXQ + 1)];
  for (int k = 0; k < q1; ++k)
    for (int l = 0; l < q1; ++l) {
      double v = 0.0;
      for (int i = 0; i < m; ++i) v += w[i] * V[i * q1 + k] * V[i * q1 + l];
      Mpi[k * q1 + l] = v;
    }
  if (!invert(q1, Mpi, Minv)) { set_error("singular projection mass matrix"); return IGA_EINVAL; }
  for (int c = 0; c < q1; ++c)
    for (int i = 0; i < m; ++i) {
      double v = 0.0;
      for (int k = 0; k < q1; ++k) v += Minv[c * q1 + k] * V[i * q1 + k];
      P[c * m + i] = v * w[i];
    }
  return IGA_OK;
}

iga_status set_projection_v(Handle &h, const int *mv) {
  int ns = 1;
  bool iso = true;
  for (int k = 0; k < h.d; ++k) {
    if (mv[k] < h.qv[k] + 1 || mv[k] > IGA_MAXM) {
      set_error("projection points m=%d outside [q+1=%d, %d] (direction %d)", mv[k], h.qv[k] + 1, IGA_MAXM, k);
      return IGA_EINVAL;
    }
    ns *= mv[k];
    iso = iso && mv[k] == mv[0] && h.qv[k] == h.qv[0];
  }
  if (k5b_smem_bytes(h, ns) > 227 * 1024 || macro_smem_bytes(h.d, ns) > 227 * 1024) {
    set_error("projection with %d sample nodes per tile: per-tile staging exceeds shared memory", ns);
    return IGA_ELIMIT;
  }
  double x[3][IGA_MAXM], P[3][(IGA_MAXQ + 1) * IGA_MAXM];
  for (int k = 0; k < h.d; ++k) {
    const iga_status st = projection_1d(h.qv[k], mv[k], x[k], P[k]);
    if (st != IGA_OK) return st;
  }
  for (int k = 0; k < 3; ++k) {
    h.mv[k] = k < h.d ? mv[k] : 1;
    for (int i = 0; i < IGA_MAXM; ++i) h.interp_x[k][i] = (k < h.d && i < mv[k]) ? x[k][i] : 0.0;
    for (int i = 0; i < (IGA_MAXQ + 1) * IGA_MAXM; ++i)
      h.Pi1[k][i] = (k < h.d && i < (h.qv[k] + 1) * mv[k]) ? P[k][i] : (k >= h.d && i == 0 ? 1.0 : 0.0);
  }
  h.ns = ns;
  h.iso = iso;
  return IGA_OK;
}

// m = 0: interpolation at the q_k+1 Gauss nodes per direction (R1); else the L2 projection
// with an m-point rule in every direction (m >= max_k q_k + 1)
iga_status set_projection(Handle &h, int m) {
  int mv[3];
  for (int k = 0; k < h.d; ++k) mv[k] = m == 0 ? h.qv[k] + 1 : m;
  const iga_status st = set_projection_v(h, mv);
  if (st != IGA_OK) return st;
  bool iso_q = true;
  for (int k = 0; k < h.d; ++k) iso_q = iso_q && h.qv[k] == h.qv[0];
  h.m_proj = m == 0 ? (iso_q ? h.q + 1 : 0) : m;
  return IGA_OK;
}

}  // namespace iga
