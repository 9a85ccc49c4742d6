// iga_api.cu — the C ABI of libiga (include/iga.h): handle lifecycle, host/device
// pointer staging, the kernel sequence of each entry point, profiling events and
// the device degeneracy flag.
#include <cstdio>
#include <cstring>
#include <mutex>
#include "internal.h"

namespace iga {
const char *get_error();

Handle::~Handle() {
  void *bufs[] = {d_table, d_tabA, d_tabAT, d_coef, d_side, d_W, d_X, d_gpart, d_node_map, d_pairA, d_pairB,
                  d_row_ptr, d_col_idx, d_brow_ptr, d_bcol, d_rowinfo, d_emap, d_mblk, d_mslot0, d_mperm, d_slot_tr, d_k4d,
                  d_k5_pair, d_k5_col, d_tperm, d_cperm, d_rowdesc, d_g1len, d_g2len, d_g1slot, d_g2slot, d_sA_ptr, d_sA_slot,
                  d_inv_ptr, d_inv_ent, d_part, d_ug, d_k5_gphys, d_k5_mode, d_k5_extra, d_Wpart, d_F, d_th, d_det, d_Vt, d_mweights, d_patch_info, d_mknots, d_mspan, d_flag};
  for (void *b : bufs)
    if (b) cudaFree(b);
  for (int i = 0; i < N_STAGE; ++i)
    if (d_stage[i]) cudaFree(d_stage[i]);
  if (aux_stream) cudaStreamDestroy(aux_stream);
  if (ev_fork) cudaEventDestroy(ev_fork);
  if (ev_join) cudaEventDestroy(ev_join);
  for (auto e : ev_pool) cudaEventDestroy(e);
}

static std::mutex g_build_mutex;   // K1 uses __constant__ patch descriptors

static bool is_device_ptr(const void *p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

#define CU(x)                                                                            \
  do {                                                                                   \
    cudaError_t _e = (x);                                                                \
    if (_e != cudaSuccess) {                                                             \
      set_error("CUDA error %s at %s:%d (%s)", cudaGetErrorString(_e), __FILE__, __LINE__, #x); \
      return IGA_ECUDA;                                                                  \
    }                                                                                    \
  } while (0)

// Staging of [any] pointers: device pointers pass through; host pointers are copied
// through per-handle grow-only device buffers (one per argument slot), so repeated
// calls with host arguments cost only the copies.
struct Stager {
  Handle &h;
  cudaStream_t s;
  int slot = 0;
  std::vector<std::pair<double *, const double *>> pending_out;   // (device, host)
  std::vector<size_t> pending_bytes;
  Stager(Handle &hh, cudaStream_t ss, int first_slot = 0) : h(hh), s(ss), slot(first_slot) {}
  double *buffer(size_t n) {
    if (slot >= Handle::N_STAGE) return nullptr;
    const int i = slot++;
    const size_t bytes = std::max<size_t>(n, 1) * 8;
    if (h.stage_cap[i] < bytes) {
      if (h.d_stage[i]) {
        cudaStreamSynchronize(s);
        cudaFree(h.d_stage[i]);
        h.d_stage[i] = nullptr;
        h.stage_cap[i] = 0;
      }
      if (cudaMalloc((void **)&h.d_stage[i], bytes) != cudaSuccess) return nullptr;
      h.stage_cap[i] = bytes;
    }
    return h.d_stage[i];
  }
  bool in(const double *p, size_t n, const double **out) {
    if (!p || is_device_ptr(p)) { *out = p; return true; }
    double *d = buffer(n);
    if (!d) return false;
    if (cudaMemcpyAsync(d, p, n * 8, cudaMemcpyHostToDevice, s) != cudaSuccess) return false;
    *out = d;
    return true;
  }
  bool out(double *p, size_t n, double **dev) {
    if (!p || is_device_ptr(p)) { *dev = p; return true; }
    double *d = buffer(n);
    if (!d) return false;
    pending_out.push_back({d, p});
    pending_bytes.push_back(n * 8);
    *dev = d;
    return true;
  }
  bool flush() {
    for (size_t i = 0; i < pending_out.size(); ++i)
      if (cudaMemcpyAsync((void *)pending_out[i].second, pending_out[i].first, pending_bytes[i], cudaMemcpyDeviceToHost, s) != cudaSuccess)
        return false;
    return true;
  }
};

// profiling helper: record event pairs around launches
struct Prof {
  Handle &h;
  cudaStream_t s;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> marks;
  size_t next = 0;
  Prof(Handle &hh, cudaStream_t ss) : h(hh), s(ss) {}
  cudaEvent_t ev() {
    if (next >= h.ev_pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      h.ev_pool.push_back(e);
    }
    return h.ev_pool[next++];
  }
  int begin(int slot) {
    if (!h.profiling) return -1;
    cudaEvent_t a = ev(), b = ev();
    cudaEventRecord(a, s);
    marks.push_back({slot, {a, b}});
    return (int)marks.size() - 1;
  }
  void end(int id) {
    if (id >= 0) cudaEventRecord(marks[id].second.second, s);
  }
  void collect() {
    for (auto &m : marks) {
      float ms = 0;
      cudaEventElapsedTime(&ms, m.second.first, m.second.second);
      h.prof_ms[m.first] += ms;
      h.prof_launches[m.first] += 1;
    }
  }
};

// X̃ and W: the fused K5g (X̃ built in shared memory, profiling slot 3) when its staging fits,
// else K5x (slot 7) + K5a (slot 3)
static cudaError_t sens_xw(Handle &h, Prof &pf, const double *du, const double *dv, cudaStream_t s) {
#ifndef IGA_EXPERIMENT_NO_K5G
  if (sens_xw_fits(h)) {
    const int id = pf.begin(3);
    const cudaError_t e = launch_sens_XW(h, du, dv, h.d_W, s);
    pf.end(id);
    return e;
  }
#endif
  int id = pf.begin(7);
  cudaError_t e = launch_sens_X(h, du, dv, s);
  pf.end(id);
  if (e) return e;
  id = pf.begin(3);
  e = launch_sens_W(h, h.d_W, s);
  pf.end(id);
  return e;
}

static iga_status check_flag(Handle &h, cudaStream_t s) {
  int f[3];
  CU(cudaMemcpyAsync(f, h.d_flag, sizeof(f), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  if (f[0] == 1) {
    set_error("degenerate tile Jacobian (det J_T <= 0) in patch %d at quadrature point %d", f[1], f[2]);
    return IGA_EDEGENERATE;
  }
  if (f[0] == 2) {
    set_error("degenerate macro element: det grad F <= 0 in tile %d at interpolation node %d", f[1], f[2]);
    return IGA_EDEGENERATE;
  }
  return IGA_OK;
}

static iga_status check_material(const Handle &h, const double *young, double nu) {
  if (!young) { set_error("young is NULL"); return IGA_EINVAL; }
  if (!(nu > -1.0 && nu < 0.5)) { set_error("nu=%g outside (-1, 0.5)", nu); return IGA_EINVAL; }
  return IGA_OK;
}

}  // namespace iga

using namespace iga;

struct iga_handle {
  Handle h;
  std::mutex mu;   // serialises the calls that use the handle's workspace (include/iga.h, Concurrency)
};
// every workspace-using entry point holds the handle's lock until its device work is done
// (each call synchronises its stream before returning)
#define IGA_LOCK(HP) std::lock_guard<std::mutex> iga_lock_(const_cast<iga_handle *>(HP)->mu)

extern "C" {

const char *iga_last_error(void) { return get_error(); }
const char *iga_version(void) { return "libiga 0.1 (sm_100a, FP64 DMMA)"; }

iga_status iga_build_tables(const iga_spline *tile_patches, int32_t n_patches, const iga_interface *interfaces,
                            int32_t n_interfaces, const iga_spline *macro_topology, int32_t q, int32_t n_gauss,
                            const iga_shard *shard, void *stream, iga_handle **out) {
  const int32_t qv[3] = {q, q, q};
  return iga_build_tables_q(tile_patches, n_patches, interfaces, n_interfaces, macro_topology, qv, n_gauss, shard,
                            stream, out);
}

iga_status iga_build_tables_q(const iga_spline *tile_patches, int32_t n_patches, const iga_interface *interfaces,
                              int32_t n_interfaces, const iga_spline *macro_topology, const int32_t *q,
                              int32_t n_gauss, const iga_shard *shard, void *stream, iga_handle **out) {
  if (!out) { set_error("out is NULL"); return IGA_EINVAL; }
  *out = nullptr;
  if (n_patches > 64) { set_error("at most 64 tile patches"); return IGA_EINVAL; }
  std::lock_guard<std::mutex> lock(g_build_mutex);
  iga_handle *H = new (std::nothrow) iga_handle();
  if (!H) { set_error("out of host memory"); return IGA_ENOMEM; }
  Handle &h = H->h;
  cudaStream_t s = (cudaStream_t)stream;
  iga_status st;
  try {
    st = build_host(h, tile_patches, n_patches, interfaces, n_interfaces, macro_topology, q, n_gauss, shard);
  } catch (std::bad_alloc &) {
    set_error("out of host memory during the host build");
    st = IGA_ENOMEM;
  }
  if (st != IGA_OK) { delete H; return st; }
  auto fail = [&](iga_status e) { delete H; return e; };
#define CUB(x)                                                                                   \
  do {                                                                                           \
    cudaError_t _e = (x);                                                                        \
    if (_e != cudaSuccess) {                                                                     \
      set_error("CUDA error %s at %s:%d (%s)", cudaGetErrorString(_e), __FILE__, __LINE__, #x);  \
      return fail(_e == cudaErrorMemoryAllocation ? IGA_ENOMEM : IGA_ECUDA);                     \
    }                                                                                            \
  } while (0)
  st = upload_topology(h);
  if (st != IGA_OK) return fail(st);
  h.on_device = true;
  const int d = h.d;
  CUB(cudaMalloc((void **)&h.d_flag, 4 * sizeof(int)));
  CUB(cudaMemsetAsync(h.d_flag, 0, 4 * sizeof(int), s));
  CUB(cudaMalloc((void **)&h.d_table, sizeof(double) * h.M * h.kstride));
  CUB(cudaMemsetAsync(h.d_table, 0, sizeof(double) * h.M * h.kstride, s));
  // fragment-major operands; the zero padding (rows, κ >= n_k, patch columns) is never rewritten
  CUB(cudaMalloc((void **)&h.d_tabA, sizeof(double) * h.Mpad * h.ks3));
  CUB(cudaMemsetAsync(h.d_tabA, 0, sizeof(double) * h.Mpad * h.ks3, s));
  CUB(cudaMalloc((void **)&h.d_tabAT, sizeof(double) * h.k5_rows * h.Kp));
  CUB(cudaMemsetAsync(h.d_tabAT, 0, sizeof(double) * h.k5_rows * h.Kp, s));
  CUB(cudaMalloc((void **)&h.d_coef, sizeof(double) * h.Npad * h.ks3));
  CUB(cudaMemsetAsync(h.d_coef, 0, sizeof(double) * h.Npad * h.ks3, s));
  CUB(cudaMalloc((void **)&h.d_W, sizeof(double) * h.Npad * h.k5_rows));
  {   // K5a split-K: the segment count minimising waves-per-unit-of-work on this GPU's SMs
    int dev = 0, nsm = 148;
    CUB(cudaGetDevice(&dev));
    CUB(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    const int64_t nblk = (h.n_tiles_own + h.tpc - 1) / h.tpc, nkb = h.k5_rows / IGA_K5_BM;
    const double w1 = (double)((nblk * nkb + nsm - 1) / nsm);
    double best = w1;
    for (int S = 2; S <= 16 && S <= (int)(h.Kp / IGA_KCHUNK); ++S) {
      const double waves = (double)((nblk * nkb * S + nsm - 1) / nsm) / S;
      if (waves < best - 1e-9 && waves < 0.9 * w1) { best = waves; h.k5_nseg = S; }   // worth the partials
    }
    if (h.k5_nseg > 1) CUB(cudaMalloc((void **)&h.d_Wpart, sizeof(double) * h.k5_nseg * h.Npad * h.k5_rows));
  }
  CUB(cudaMalloc((void **)&h.d_F, sizeof(double) * h.n_local_ctrl * h.npi));
  CUB(cudaMalloc((void **)&h.d_th, sizeof(double) * h.npi));
  CUB(cudaMalloc((void **)&h.d_det, sizeof(double) * h.n_tiles * h.npi));
  CUB(cudaMalloc((void **)&h.d_Vt, sizeof(double) * (h.n_tiles + 1)));
  CUB(cudaMalloc((void **)&h.d_X, sizeof(double) * h.Npad * h.Kp));
  int nact_m = 1;
  for (int k = 0; k < d; ++k) nact_m *= h.pm[k] + 1;
  CUB(cudaMalloc((void **)&h.d_gpart, sizeof(double) * h.n_tiles * nact_m * d));
  CUB(cudaMalloc((void **)&h.d_row_ptr, sizeof(int64_t) * (h.n_nodes * d + 1)));
  CUB(cudaMalloc((void **)&h.d_col_idx, sizeof(int32_t) * std::max<int64_t>(h.nnz, 1)));
  // macro knots / element spans
  std::vector<double> mk;
  std::vector<int> ms;
  for (int k = 0; k < d; ++k) {
    mk.insert(mk.end(), h.mknots[k].begin(), h.mknots[k].end());
    ms.insert(ms.end(), h.mel_span[k].begin(), h.mel_span[k].end());
  }
  CUB(cudaMalloc((void **)&h.d_mknots, sizeof(double) * mk.size()));
  CUB(cudaMemcpy(h.d_mknots, mk.data(), sizeof(double) * mk.size(), cudaMemcpyHostToDevice));
  if (!h.mweights.empty()) {
    CUB(cudaMalloc((void **)&h.d_mweights, sizeof(double) * h.mweights.size()));
    CUB(cudaMemcpy(h.d_mweights, h.mweights.data(), sizeof(double) * h.mweights.size(), cudaMemcpyHostToDevice));
  }
  CUB(cudaMalloc((void **)&h.d_mspan, sizeof(int) * ms.size()));
  CUB(cudaMemcpy(h.d_mspan, ms.data(), sizeof(int) * ms.size(), cudaMemcpyHostToDevice));
  // tile data for K1
  std::vector<DevPatch> dp(n_patches);
  std::vector<double> tctrl, tknots;
  std::vector<int> tel;
  int pt_off = 0, ngd = 1;
  for (int k = 0; k < d; ++k) ngd *= h.n_g;
  for (int pi = 0; pi < n_patches; ++pi) {
    PatchInfo &P = h.patches[pi];
    DevPatch &D = dp[pi];
    memset(&D, 0, sizeof(D));
    D.deg = h.p;
    D.ctrl_off = P.ctrl_off;
    for (int k = 0; k < 3; ++k) {
      D.n[k] = P.n[k];
      D.n_span[k] = P.n_span[k];
      D.knot_off[k] = (int)tknots.size();
      D.elspan_off[k] = (int)tel.size();
      if (k < d) {
        tknots.insert(tknots.end(), P.knots[k].begin(), P.knots[k].end());
        tel.insert(tel.end(), P.el_span[k].begin(), P.el_span[k].end());
      }
    }
    D.n_spans = P.n_spans;
    D.pt_off = pt_off;
    P.pt_off = pt_off;
    pt_off += P.n_spans * ngd;
    tctrl.insert(tctrl.end(), P.ctrl.begin(), P.ctrl.end());
  }
  double *d_tctrl, *d_tknots;
  int *d_tel;
  CUB(cudaMalloc((void **)&d_tctrl, sizeof(double) * tctrl.size()));
  CUB(cudaMemcpy(d_tctrl, tctrl.data(), sizeof(double) * tctrl.size(), cudaMemcpyHostToDevice));
  CUB(cudaMalloc((void **)&d_tknots, sizeof(double) * tknots.size()));
  CUB(cudaMemcpy(d_tknots, tknots.data(), sizeof(double) * tknots.size(), cudaMemcpyHostToDevice));
  CUB(cudaMalloc((void **)&d_tel, sizeof(int) * tel.size()));
  CUB(cudaMemcpy(d_tel, tel.data(), sizeof(int) * tel.size(), cudaMemcpyHostToDevice));
  double gx[16], gw[16];
  gauss_legendre01(h.n_g, gx, gw);
  CUB(launch_tables(h, dp.data(), n_patches, d_tctrl, d_tknots, d_tel, gx, gw, pt_off, s));
  CUB(launch_pack_tables(h, s));
  CUB(launch_expand_pattern(h, s));
  CUB(cudaStreamSynchronize(s));
  cudaFree(d_tctrl);
  cudaFree(d_tknots);
  cudaFree(d_tel);
  st = check_flag(h, s);
  if (st != IGA_OK) return fail(st);
#undef CUB
  *out = H;
  return IGA_OK;
}

iga_status iga_build_topology(const iga_spline *tile_patches, int32_t n_patches, const iga_interface *interfaces,
                              int32_t n_interfaces, const iga_spline *macro_topology, int32_t q, int32_t n_gauss,
                              const iga_shard *shard, iga_handle **out) {
  const int32_t qv[3] = {q, q, q};
  return iga_build_topology_q(tile_patches, n_patches, interfaces, n_interfaces, macro_topology, qv, n_gauss, shard,
                              out);
}

iga_status iga_build_topology_q(const iga_spline *tile_patches, int32_t n_patches, const iga_interface *interfaces,
                                int32_t n_interfaces, const iga_spline *macro_topology, const int32_t *q,
                                int32_t n_gauss, const iga_shard *shard, iga_handle **out) {
  if (!out) { set_error("out is NULL"); return IGA_EINVAL; }
  *out = nullptr;
  iga_handle *H = new (std::nothrow) iga_handle();
  if (!H) { set_error("out of host memory"); return IGA_ENOMEM; }
  iga_status st;
  try {
    st = build_host(H->h, tile_patches, n_patches, interfaces, n_interfaces, macro_topology, q, n_gauss, shard);
  } catch (std::bad_alloc &) {
    set_error("out of host memory during the host build");
    st = IGA_ENOMEM;
  }
  if (st != IGA_OK) { delete H; return st; }
  *out = H;
  return IGA_OK;
}

void iga_free(iga_handle *H) { delete H; }

iga_status iga_get_sizes(const iga_handle *H, iga_sizes *o) {
  if (!H || !o) { set_error("NULL argument"); return IGA_EINVAL; }
  const Handle &h = H->h;
  memset(o, 0, sizeof(*o));
  o->dim = h.d;
  o->q = h.q;
  o->n_pi = h.npi;
  for (int k = 0; k < 3; ++k) {
    o->q_dir[k] = h.qv[k];
    o->m_dir[k] = h.mv[k];
  }
  o->n_k = h.nk;
  o->n_local_ctrl = h.n_local_ctrl;
  o->k_stride = h.kstride;
  o->n_patches = h.n_patches;
  o->n_gauss = h.n_g;
#ifndef IGA_EXPERIMENT_NO_K5G
  o->sens_path = (sens_xw_fits(h) ? 1 : 0) | (h.k5_nseg << 8);
#else
  o->sens_path = h.k5_nseg << 8;
#endif
  o->n_tiles = h.n_tiles_glob;
  o->n_local_rows = h.M;
  o->n_macro_cp = h.n_cp;
  o->n_nodes = h.n_nodes_glob;
  o->n_dof = h.n_dof;
  o->nnz = h.nnz;
  o->n_blocks = h.n_blocks;
  o->n_contrib = h.n_contrib;
  o->n_multi_blocks = h.n_multi;
  o->n_side_slots = h.n_slots;
  o->tile_begin = h.t_base;
  o->n_tiles_local = h.n_tiles;
  o->n_tiles_owned = h.n_tiles_own;
  o->row_begin = h.node_base * h.d;
  o->n_rows = h.n_nodes * h.d;
  return IGA_OK;
}

iga_status iga_assemble(const iga_handle *Hc, const double *macro_ctrl, const double *young, int32_t young_per_tile,
                        double nu, double *csr_values, double *local_values, void *stream) {
  if (!Hc || !macro_ctrl || (!csr_values && !local_values)) { set_error("NULL argument"); return IGA_EINVAL; }
  IGA_LOCK(Hc);
  Handle &h = const_cast<iga_handle *>(Hc)->h;
  if (!h.on_device) { set_error("topology-only handle (iga_build_topology) cannot run kernels"); return IGA_EINVAL; }
  iga_status st = check_material(h, young, nu);
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  Stager sg(h, s);
  Prof pf(h, s);
  int idst = pf.begin(6);
  CU(cudaMemsetAsync(h.d_flag, 0, 4 * sizeof(int), s));
  const double *dctrl, *dyoung;
  if (!sg.in(macro_ctrl, (size_t)h.n_cp * h.d, &dctrl) ||
      !sg.in(young, young_per_tile ? (size_t)h.n_tiles_glob : 1, &dyoung)) {
    set_error("staging of host inputs failed");
    return IGA_ENOMEM;
  }
  double *dvals, *dlocal_out;
  if (!sg.out(csr_values, (size_t)h.nnz, &dvals) ||
      !sg.out(local_values, (size_t)(h.M * h.n_tiles * h.d * h.d), &dlocal_out)) {
    set_error("staging of host outputs failed");
    return IGA_ENOMEM;
  }
  pf.end(idst);
  int id = pf.begin(0);
  CU(launch_interpolate(h, dctrl, dyoung, young_per_tile, nu, h.d_coef, true, s));
  pf.end(id);
  if (dvals) {   // csr_values NULL: the non-zero components only (K2 + K3 nzdata)
    id = pf.begin(1);
    CU(launch_contraction(h, dvals, nullptr, s));
    pf.end(id);
    id = pf.begin(2);
    CU(launch_scatter_multi(h, dvals, s));
    pf.end(id);
  }
  if (dlocal_out) {   // optional nzdata output (parity of the element matrices, R17): K3 again
    id = pf.begin(8);
    CU(launch_contraction(h, nullptr, dlocal_out, s));
    pf.end(id);
  }
  idst = pf.begin(6);
  if (!sg.flush()) { set_error("D2H copy of outputs failed"); return IGA_ECUDA; }
  pf.end(idst);
  st = check_flag(h, s);
  pf.collect();
  return st;
}

iga_status iga_apply(const iga_handle *Hc, const double *macro_ctrl, const double *young, int32_t young_per_tile,
                     double nu, const double *u, double *y, void *stream) {
  if (!Hc || !macro_ctrl || !u || !y) { set_error("NULL argument"); return IGA_EINVAL; }
  IGA_LOCK(Hc);
  Handle &h = const_cast<iga_handle *>(Hc)->h;
  if (!h.on_device) { set_error("topology-only handle (iga_build_topology) cannot run kernels"); return IGA_EINVAL; }
  iga_status st = check_material(h, young, nu);
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  if (!h.d_part) {   // partial slots: allocated on first use (assemble-only users never pay it)
    const size_t bytes = std::max<size_t>(8, sizeof(double) * (size_t)h.n_tiles * h.P * h.d);
    const size_t ubytes = std::max<size_t>(8, sizeof(double) * (size_t)h.n_tiles * h.n_local_ctrl * h.d);
    if (cudaMalloc((void **)&h.d_part, bytes) != cudaSuccess || cudaMalloc((void **)&h.d_ug, ubytes) != cudaSuccess) {
      cudaGetLastError();
      set_error("cudaMalloc of %zu + %zu bytes of apply buffers failed", bytes, ubytes);
      return IGA_ENOMEM;
    }
  }
  Stager sg(h, s);
  Prof pf(h, s);
  int idst = pf.begin(6);
  CU(cudaMemsetAsync(h.d_flag, 0, 4 * sizeof(int), s));
  const double *dctrl, *dyoung, *du;
  double *dy;
  if (!sg.in(macro_ctrl, (size_t)h.n_cp * h.d, &dctrl) ||
      !sg.in(young, young_per_tile ? (size_t)h.n_tiles_glob : 1, &dyoung) || !sg.in(u, (size_t)h.n_dof, &du) ||
      !sg.out(y, (size_t)(h.n_nodes * h.d), &dy)) {
    set_error("staging failed");
    return IGA_ENOMEM;
  }
  pf.end(idst);
  int id = pf.begin(0);
  CU(launch_interpolate(h, dctrl, dyoung, young_per_tile, nu, h.d_coef, true, s));
  pf.end(id);
  id = pf.begin(9);
  CU(launch_apply(h, du, dy, s));
  pf.end(id);
  idst = pf.begin(6);
  if (!sg.flush()) { set_error("D2H copy failed"); return IGA_ECUDA; }
  pf.end(idst);
  st = check_flag(h, s);
  pf.collect();
  return st;
}

iga_status iga_volume(const iga_handle *Hc, const double *macro_ctrl, double *volume, double *grad, void *stream) {
  if (!Hc || !macro_ctrl || !volume) { set_error("NULL argument"); return IGA_EINVAL; }
  IGA_LOCK(Hc);
  Handle &h = const_cast<iga_handle *>(Hc)->h;
  if (!h.on_device) { set_error("topology-only handle (iga_build_topology) cannot run kernels"); return IGA_EINVAL; }
  cudaStream_t s = (cudaStream_t)stream;
  Stager sg(h, s);
  Prof pf(h, s);
  CU(cudaMemsetAsync(h.d_flag, 0, 4 * sizeof(int), s));
  const double *dctrl;
  double *dgrad = nullptr;
  if (!sg.in(macro_ctrl, (size_t)h.n_cp * h.d, &dctrl) || (grad && !sg.out(grad, (size_t)(h.n_cp * h.d), &dgrad))) {
    set_error("staging failed");
    return IGA_ENOMEM;
  }
  CU(launch_volume(h, dctrl, h.d_Vt + h.n_tiles, dgrad ? h.d_gpart : nullptr, s));
  if (dgrad) {
    CU(launch_sens_reduce(h, h.d_gpart, dgrad, s));   // same per-tile partial layout as K5b
  }
  CU(cudaMemcpyAsync(volume, h.d_Vt + h.n_tiles, sizeof(double), cudaMemcpyDeviceToHost, s));
  if (!sg.flush()) { set_error("D2H copy failed"); return IGA_ECUDA; }
  iga_status st = check_flag(h, s);
  pf.collect();
  return st;
}

iga_status iga_load_vector(const iga_handle *Hc, const double *macro_ctrl, const double *body_force, double *f,
                           void *stream) {
  if (!Hc || !macro_ctrl || !body_force || !f) { set_error("NULL argument"); return IGA_EINVAL; }
  IGA_LOCK(Hc);
  Handle &h = const_cast<iga_handle *>(Hc)->h;
  if (!h.on_device) { set_error("topology-only handle (iga_build_topology) cannot run kernels"); return IGA_EINVAL; }
  cudaStream_t s = (cudaStream_t)stream;
  Stager sg(h, s);
  Prof pf(h, s);
  CU(cudaMemsetAsync(h.d_flag, 0, 4 * sizeof(int), s));
  const double *dctrl;
  double *df;
  if (!sg.in(macro_ctrl, (size_t)h.n_cp * h.d, &dctrl) || !sg.out(f, (size_t)(h.n_nodes * h.d), &df)) {
    set_error("staging failed");
    return IGA_ENOMEM;
  }
  CU(launch_volume(h, dctrl, nullptr, nullptr, s));   // d^(t) of every local tile
  CU(launch_load(h, body_force, df, s));
  if (!sg.flush()) { set_error("D2H copy failed"); return IGA_ECUDA; }
  iga_status st = check_flag(h, s);
  pf.collect();
  return st;
}

iga_status iga_interpolate(const iga_handle *Hc, const double *macro_ctrl, const double *young, int32_t young_per_tile,
                           double nu, double *coef, void *stream) {
  if (!Hc || !macro_ctrl || !coef) { set_error("NULL argument"); return IGA_EINVAL; }
  IGA_LOCK(Hc);
  Handle &h = const_cast<iga_handle *>(Hc)->h;
  if (!h.on_device) { set_error("topology-only handle (iga_build_topology) cannot run kernels"); return IGA_EINVAL; }
  iga_status st = check_material(h, young, nu);
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  Stager sg(h, s);
  Prof pf(h, s);
  CU(cudaMemsetAsync(h.d_flag, 0, 4 * sizeof(int), s));
  const double *dctrl, *dyoung;
  double *dcoef;
  const size_t ncoef = (size_t)h.n_tiles * h.d * h.d * h.kstride;
  if (!sg.in(macro_ctrl, (size_t)h.n_cp * h.d, &dctrl) ||
      !sg.in(young, young_per_tile ? (size_t)h.n_tiles_glob : 1, &dyoung) || !sg.out(coef, ncoef, &dcoef)) {
    set_error("staging failed");
    return IGA_ENOMEM;
  }
  CU(cudaMemsetAsync(dcoef, 0, ncoef * sizeof(double), s));
  int id = pf.begin(0);
  CU(launch_interpolate(h, dctrl, dyoung, young_per_tile, nu, dcoef, false, s));
  pf.end(id);
  if (!sg.flush()) { set_error("D2H copy failed"); return IGA_ECUDA; }
  st = check_flag(h, s);
  pf.collect();
  return st;
}

iga_status iga_sensitivity(const iga_handle *Hc, const double *macro_ctrl, const double *young,
                           int32_t young_per_tile, double nu, const double *u, const double *v, double *grad,
                           void *stream) {
  if (!Hc || !macro_ctrl || !u || !v || !grad) { set_error("NULL argument"); return IGA_EINVAL; }
  IGA_LOCK(Hc);
  Handle &h = const_cast<iga_handle *>(Hc)->h;
  if (!h.on_device) { set_error("topology-only handle (iga_build_topology) cannot run kernels"); return IGA_EINVAL; }
  iga_status st = check_material(h, young, nu);
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  Stager sg(h, s);
  Prof pf(h, s);
  int idst = pf.begin(6);
  CU(cudaMemsetAsync(h.d_flag, 0, 4 * sizeof(int), s));
  const double *dctrl, *dyoung, *du, *dv;
  double *dgrad;
  if (!sg.in(macro_ctrl, (size_t)h.n_cp * h.d, &dctrl) ||
      !sg.in(young, young_per_tile ? (size_t)h.n_tiles_glob : 1, &dyoung) || !sg.in(u, (size_t)h.n_dof, &du) ||
      !sg.in(v, (size_t)h.n_dof, &dv) || !sg.out(grad, (size_t)(h.n_cp * h.d), &dgrad)) {
    set_error("staging failed");
    return IGA_ENOMEM;
  }
  pf.end(idst);
  int id = 0;
  CU(sens_xw(h, pf, du, dv, s));
  id = pf.begin(4);
  CU(launch_sens_reverse(h, dctrl, dyoung, young_per_tile, nu, h.d_W, h.d_gpart, s));
  pf.end(id);
  id = pf.begin(5);
  CU(launch_sens_reduce(h, h.d_gpart, dgrad, s));
  pf.end(id);
  idst = pf.begin(6);
  if (!sg.flush()) { set_error("D2H copy failed"); return IGA_ECUDA; }
  pf.end(idst);
  st = check_flag(h, s);
  pf.collect();
  return st;
}

iga_status iga_assemble_sensitivity(const iga_handle *Hc, const double *macro_ctrl, const double *young,
                                    int32_t young_per_tile, double nu, const double *u, const double *v,
                                    double *csr_values, double *grad, void *stream) {
  if (!Hc || !macro_ctrl || !u || !v || !grad || !csr_values) { set_error("NULL argument"); return IGA_EINVAL; }
  IGA_LOCK(Hc);
  Handle &h = const_cast<iga_handle *>(Hc)->h;
  if (!h.on_device) { set_error("topology-only handle (iga_build_topology) cannot run kernels"); return IGA_EINVAL; }
  iga_status st = check_material(h, young, nu);
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  if (!h.aux_stream) {
    CU(cudaStreamCreateWithFlags(&h.aux_stream, cudaStreamNonBlocking));
    CU(cudaEventCreateWithFlags(&h.ev_fork, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&h.ev_join, cudaEventDisableTiming));
  }
  // u, v travel on the auxiliary stream while K2 -> K3 -> K4 form K on the caller's stream
  CU(cudaEventRecord(h.ev_fork, s));
  CU(cudaStreamWaitEvent(h.aux_stream, h.ev_fork, 0));
  Stager sg(h, s), sg2(h, h.aux_stream, 4);
  Prof pf(h, s);
  int idst = pf.begin(6);
  CU(cudaMemsetAsync(h.d_flag, 0, 4 * sizeof(int), s));
  const double *dctrl, *dyoung, *du, *dv;
  double *dvals, *dgrad;
  if (!sg.in(macro_ctrl, (size_t)h.n_cp * h.d, &dctrl) ||
      !sg.in(young, young_per_tile ? (size_t)h.n_tiles_glob : 1, &dyoung) ||
      !sg.out(csr_values, (size_t)h.nnz, &dvals) || !sg.out(grad, (size_t)(h.n_cp * h.d), &dgrad) ||
      !sg2.in(u, (size_t)h.n_dof, &du) || !sg2.in(v, (size_t)h.n_dof, &dv)) {
    set_error("staging failed");
    return IGA_ENOMEM;
  }
  CU(cudaEventRecord(h.ev_join, h.aux_stream));
  pf.end(idst);
  int id = pf.begin(0);
  CU(launch_interpolate(h, dctrl, dyoung, young_per_tile, nu, h.d_coef, true, s));
  pf.end(id);
  id = pf.begin(1);
  CU(launch_contraction(h, dvals, nullptr, s));
  pf.end(id);
  id = pf.begin(2);
  CU(launch_scatter_multi(h, dvals, s));
  pf.end(id);
  CU(cudaStreamWaitEvent(s, h.ev_join, 0));
  CU(sens_xw(h, pf, du, dv, s));
  id = pf.begin(4);
  CU(launch_sens_reverse(h, dctrl, dyoung, young_per_tile, nu, h.d_W, h.d_gpart, s));
  pf.end(id);
  id = pf.begin(5);
  CU(launch_sens_reduce(h, h.d_gpart, dgrad, s));
  pf.end(id);
  idst = pf.begin(6);
  if (!sg.flush()) { set_error("D2H copy failed"); return IGA_ECUDA; }
  pf.end(idst);
  st = check_flag(h, s);
  pf.collect();
  return st;
}

// ---- a-priori projection error and degree selection (Eqs. 59, 65) ----
namespace {
struct MacroOnly {   // the macro map on the device, no tile (iga_projection_error / iga_select_degree)
  Handle h;
  double *d_ctrl = nullptr, *d_e = nullptr;
  ~MacroOnly() {
    if (d_ctrl) cudaFree(d_ctrl);
    if (d_e) cudaFree(d_e);
  }
};

iga_status macro_only_setup(MacroOnly &mo, const iga_spline *macro, int32_t n_samples, cudaStream_t s) {
  if (!macro || !macro->ctrl) { set_error("macro spline with control points required"); return IGA_EINVAL; }
  if (macro->dim != 2 && macro->dim != 3) { set_error("dim must be 2 or 3"); return IGA_EINVAL; }
  if (n_samples < 2 || n_samples > IGA_MAXM) { set_error("n_samples=%d outside [2,%d]", n_samples, IGA_MAXM); return IGA_EINVAL; }
  Handle &h = mo.h;
  h.d = macro->dim;
  iga_status st = parse_macro(h, macro, h.d);
  if (st != IGA_OK) return st;
  h.n_tiles_glob = h.n_tiles;
  h.n_tiles_own = h.n_tiles;
  std::vector<double> mk;
  std::vector<int> ms;
  for (int k = 0; k < h.d; ++k) {
    mk.insert(mk.end(), h.mknots[k].begin(), h.mknots[k].end());
    ms.insert(ms.end(), h.mel_span[k].begin(), h.mel_span[k].end());
  }
  if (cudaMalloc((void **)&h.d_mknots, sizeof(double) * mk.size()) || cudaMalloc((void **)&h.d_mspan, sizeof(int) * ms.size()) ||
      cudaMalloc((void **)&h.d_flag, 4 * sizeof(int)) || cudaMalloc((void **)&mo.d_ctrl, sizeof(double) * h.n_cp * h.d) ||
      cudaMalloc((void **)&mo.d_e, sizeof(double) * h.n_tiles)) {
    set_error("device allocation failed");
    return IGA_ENOMEM;
  }
  if (!h.mweights.empty()) {
    if (cudaMalloc((void **)&h.d_mweights, sizeof(double) * h.mweights.size())) { set_error("device allocation failed"); return IGA_ENOMEM; }
    CU(cudaMemcpyAsync(h.d_mweights, h.mweights.data(), sizeof(double) * h.mweights.size(), cudaMemcpyHostToDevice, s));
  }
  CU(cudaMemcpyAsync(h.d_mknots, mk.data(), sizeof(double) * mk.size(), cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync(h.d_mspan, ms.data(), sizeof(int) * ms.size(), cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync(mo.d_ctrl, macro->ctrl, sizeof(double) * h.n_cp * h.d, cudaMemcpyHostToDevice, s));
  CU(cudaStreamSynchronize(s));
  return IGA_OK;
}

// E_proj for degrees q (d values) with q_k + 1 + m_extra projection points per direction
iga_status macro_only_error(MacroOnly &mo, const int32_t *q, int32_t m_extra, double nu, int32_t n_samples,
                            double *e_max, std::vector<double> *e_host, cudaStream_t s) {
  Handle &h = mo.h;
  iga_status st = set_degrees(h, q);
  if (st != IGA_OK) return st;
  int mv[3] = {1, 1, 1};
  for (int k = 0; k < h.d; ++k) mv[k] = h.qv[k] + 1 + m_extra;
  st = set_projection_v(h, mv);
  if (st != IGA_OK) return st;
  if (projection_error_smem_bytes(h.d, h.ns, n_samples, h.npi) > 227 * 1024) {
    set_error("projection error: per-tile staging exceeds shared memory (reduce n_samples or m_extra)");
    return IGA_ELIMIT;
  }
  CU(cudaMemsetAsync(h.d_flag, 0, 4 * sizeof(int), s));
  CU(launch_projection_error(h, mo.d_ctrl, nu, n_samples, mo.d_e, s));
  std::vector<double> e((size_t)h.n_tiles);
  CU(cudaMemcpyAsync(e.data(), mo.d_e, sizeof(double) * e.size(), cudaMemcpyDeviceToHost, s));
  st = check_flag(h, s);
  if (st != IGA_OK) return st;
  double mx = 0.0;
  for (double x : e) mx = std::max(mx, x);
  *e_max = mx;
  if (e_host) e_host->swap(e);
  return IGA_OK;
}
}  // namespace

iga_status iga_projection_error(const iga_spline *macro, const int32_t *q, int32_t m_extra, double nu,
                                int32_t n_samples, double *e_max, double *e_tile, void *stream) {
  if (!q || !e_max) { set_error("NULL argument"); return IGA_EINVAL; }
  if (m_extra < 0) { set_error("m_extra < 0"); return IGA_EINVAL; }
  if (!(nu > -1.0 && nu < 0.5)) { set_error("nu=%g outside (-1, 0.5)", nu); return IGA_EINVAL; }
  cudaStream_t s = (cudaStream_t)stream;
  MacroOnly mo;
  iga_status st = macro_only_setup(mo, macro, n_samples ? n_samples : 8, s);
  if (st != IGA_OK) return st;
  std::vector<double> e;
  st = macro_only_error(mo, q, m_extra, nu, n_samples ? n_samples : 8, e_max, &e, s);
  if (st != IGA_OK) return st;
  if (e_tile) CU(cudaMemcpy(e_tile, e.data(), sizeof(double) * e.size(), cudaMemcpyDefault));
  return IGA_OK;
}

iga_status iga_select_degree(const iga_spline *macro, double nu, double tol, int32_t m_extra, int32_t n_samples,
                             int32_t q_max, int32_t *q_out, double *e_out, void *stream) {
  if (!q_out || !(tol > 0.0)) { set_error("NULL q_out or tol <= 0"); return IGA_EINVAL; }
  if (!(nu > -1.0 && nu < 0.5)) { set_error("nu=%g outside (-1, 0.5)", nu); return IGA_EINVAL; }
  if (q_max <= 0 || q_max > IGA_MAXQ) q_max = IGA_MAXQ;
  cudaStream_t s = (cudaStream_t)stream;
  const int ns_ = n_samples ? n_samples : 8;
  MacroOnly mo;
  iga_status st = macro_only_setup(mo, macro, ns_, s);
  if (st != IGA_OK) return st;
  const int d = mo.h.d;
  // reading R19: q(s) = max(p_M,k + s, 0), uniform enrichment / coarsening from the macro degrees
  auto q_of = [&](int sh, int32_t *q) {
    int mx = 0;
    for (int k = 0; k < d; ++k) {
      q[k] = std::max(mo.h.pm[k] + sh, 0);
      mx = std::max(mx, q[k]);
    }
    return mx;
  };
  int32_t q[3] = {0, 0, 0};
  int sh = 0;
  if (q_of(0, q) > q_max) { set_error("macro degree exceeds q_max=%d", q_max); return IGA_EINVAL; }
  double e = 0.0;
  st = macro_only_error(mo, q, m_extra, nu, ns_, &e, nullptr, s);
  if (st != IGA_OK) return st;
  if (e <= tol) {
    while (q_of(sh, q) > 0) {
      double e_down = 0.0;
      q_of(sh - 1, q);
      st = macro_only_error(mo, q, m_extra, nu, ns_, &e_down, nullptr, s);
      if (st != IGA_OK) return st;
      if (e_down > tol) break;
      --sh;
      e = e_down;
    }
  } else {
    for (;;) {
      if (q_of(sh + 1, q) > q_max) {
        q_of(sh, q);
        for (int k = 0; k < d; ++k) q_out[k] = q[k];
        if (e_out) *e_out = e;
        set_error("E_proj = %.3e > tol = %.1e at the largest admissible degree (q_max = %d)", e, tol, q_max);
        return IGA_ELIMIT;
      }
      ++sh;
      st = macro_only_error(mo, q, m_extra, nu, ns_, &e, nullptr, s);
      if (st != IGA_OK) return st;
      if (e <= tol) break;
    }
  }
  q_of(sh, q);
  for (int k = 0; k < d; ++k) q_out[k] = q[k];
  if (e_out) *e_out = e;
  return IGA_OK;
}

iga_status iga_get_pattern(const iga_handle *Hc, int64_t *row_ptr, int32_t *col_idx) {
  if (!Hc) { set_error("NULL handle"); return IGA_EINVAL; }
  IGA_LOCK(Hc);
  const Handle &h = Hc->h;
  if (h.on_device) {
    if (row_ptr) CU(cudaMemcpy(row_ptr, h.d_row_ptr, sizeof(int64_t) * (h.n_nodes * h.d + 1), cudaMemcpyDefault));
    if (col_idx) CU(cudaMemcpy(col_idx, h.d_col_idx, sizeof(int32_t) * h.nnz, cudaMemcpyDefault));
    return IGA_OK;
  }
  // topology-only handle: expand the block CSR on the host (host pointers only)
  const int d = h.d;
  for (int64_t I = 0; I < h.n_nodes; ++I) {
    int64_t b0 = h.brow_ptr[I], nb = h.brow_ptr[I + 1] - b0;
    for (int a = 0; a < d; ++a) {
      int64_t base = (int64_t)d * d * b0 + a * d * nb;
      if (row_ptr) row_ptr[I * d + a] = base;
      if (col_idx)
        for (int64_t j = 0; j < nb; ++j)
          for (int b = 0; b < d; ++b) col_idx[base + d * j + b] = h.bcol[b0 + j] * d + b;
    }
  }
  if (row_ptr) row_ptr[h.n_nodes * d] = h.nnz;
  return IGA_OK;
}

iga_status iga_get_block_map(const iga_handle *Hc, int64_t t_begin, int64_t t_end, int64_t *out) {
  if (!Hc || !out) { set_error("NULL argument"); return IGA_EINVAL; }
  IGA_LOCK(Hc);
  const Handle &h = Hc->h;
  if (t_begin < 0 || t_end > h.n_tiles || t_begin > t_end) { set_error("bad tile range"); return IGA_EINVAL; }
  const int d = h.d;
  const int64_t nl = h.n_local_ctrl;
  auto pos = [&](int64_t I, int64_t J) -> int64_t {
    const int64_t i = I - h.node_base;
    if (i < 0 || i >= h.n_nodes) return -1;   // row of another shard
    const int32_t *b = h.bcol.data() + h.brow_ptr[i], *e = h.bcol.data() + h.brow_ptr[i + 1];
    const int32_t *f = std::lower_bound(b, e, (int32_t)J);
    return (int64_t)d * d * h.brow_ptr[i] + (int64_t)d * (f - b);
  };
#pragma omp parallel for schedule(static)
  for (int64_t t = t_begin; t < t_end; ++t)
    for (int64_t r = 0; r < h.M; ++r) {
      int64_t I = h.node_map[t * nl + h.pairA[r]], J = h.node_map[t * nl + h.pairB[r]];
      int64_t o = ((t - t_begin) * h.M + r) * 2;
      out[o] = pos(I, J);
      out[o + 1] = pos(J, I);
    }
  return IGA_OK;
}

iga_status iga_get_node_map(const iga_handle *Hc, int32_t *out) {
  if (!Hc || !out) { set_error("NULL argument"); return IGA_EINVAL; }
  memcpy(out, Hc->h.node_map.data(), Hc->h.node_map.size() * sizeof(int32_t));
  return IGA_OK;
}

iga_status iga_get_tables(const iga_handle *Hc, double *out) {
  if (!Hc || !out) { set_error("NULL argument"); return IGA_EINVAL; }
  IGA_LOCK(Hc);
  const Handle &h = Hc->h;
  if (!h.on_device) { set_error("topology-only handle has no tables"); return IGA_EINVAL; }
  CU(cudaMemcpy2D(out, sizeof(double) * h.nk, h.d_table, sizeof(double) * h.kstride, sizeof(double) * h.nk, h.M,
                  cudaMemcpyDefault));
  return IGA_OK;
}

iga_status iga_get_pairs(const iga_handle *Hc, int32_t *out) {
  if (!Hc || !out) { set_error("NULL argument"); return IGA_EINVAL; }
  IGA_LOCK(Hc);
  const Handle &h = Hc->h;
  for (int64_t r = 0; r < h.M; ++r) {
    int pa = h.pairA[r], pb = h.pairB[r];
    int pi = 0;
    while (pi + 1 < h.n_patches && pa >= h.patches[pi + 1].ctrl_off) ++pi;
    out[2 * r] = pa - h.patches[pi].ctrl_off;
    out[2 * r + 1] = pb - h.patches[pi].ctrl_off;
  }
  return IGA_OK;
}

iga_status iga_set_projection(iga_handle *H, int32_t m) {
  if (!H) { set_error("NULL handle"); return IGA_EINVAL; }
  IGA_LOCK(H);
  return set_projection(H->h, m);
}

iga_status iga_get_projection(const iga_handle *H, int32_t *m) {
  if (!H || !m) { set_error("NULL argument"); return IGA_EINVAL; }
  IGA_LOCK(H);
  *m = H->h.m_proj;
  return IGA_OK;
}

iga_status iga_set_profiling(iga_handle *H, int32_t enable) {
  if (!H) { set_error("NULL handle"); return IGA_EINVAL; }
  IGA_LOCK(H);
  H->h.profiling = enable != 0;
  if (enable)
    for (int i = 0; i < IGA_N_PROF; ++i) { H->h.prof_ms[i] = 0; H->h.prof_launches[i] = 0; }
  return IGA_OK;
}

iga_status iga_get_kernel_times(const iga_handle *H, double *ms_out, int64_t *launches_out) {
  if (!H) { set_error("NULL handle"); return IGA_EINVAL; }
  IGA_LOCK(H);
  for (int i = 0; i < IGA_N_PROF; ++i) {
    if (ms_out) ms_out[i] = H->h.prof_ms[i];
    if (launches_out) launches_out[i] = H->h.prof_launches[i];
  }
  return IGA_OK;
}

}  // extern "C"
