"""Thin ctypes binding of libiga (include/iga.h): argument marshalling only.

Every step of the hot path runs in the CUDA kernels behind the C ABI; there is no
Python or CPU fallback.  If libiga.so is missing this module raises at import of
`load()` — build it with `python -m paper_2107_09568_b200.build` (or
`__graft_entry__.build()`).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("IGA_LIB") or os.path.join(HERE, "libiga.so")   # IGA_LIB: experiment builds only

IGA_STATUS = {0: "IGA_OK", 1: "IGA_EINVAL", 2: "IGA_EDEGENERATE", 3: "IGA_ENONCONFORMING", 4: "IGA_ENOMEM",
              5: "IGA_ECUDA", 6: "IGA_ELIMIT"}


class IgaError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{IGA_STATUS.get(status, status)}: {msg}")
        self.status = status


class iga_spline(C.Structure):
    _fields_ = [("dim", C.c_int32), ("degree", C.c_int32 * 3), ("n_knots", C.c_int32 * 3),
                ("knots", C.POINTER(C.c_double) * 3), ("ctrl", C.POINTER(C.c_double)),
                ("weights", C.POINTER(C.c_double))]


class iga_interface(C.Structure):
    _fields_ = [("patch_a", C.c_int32), ("dir_a", C.c_int32), ("side_a", C.c_int32),
                ("patch_b", C.c_int32), ("dir_b", C.c_int32), ("side_b", C.c_int32)]


class iga_sizes(C.Structure):
    _fields_ = [("dim", C.c_int32), ("q", C.c_int32), ("n_pi", C.c_int32), ("n_k", C.c_int32),
                ("k_stride", C.c_int32), ("n_patches", C.c_int32), ("n_gauss", C.c_int32), ("sens_path", C.c_int32),
                ("n_tiles", C.c_int64), ("n_local_rows", C.c_int64), ("n_macro_cp", C.c_int64),
                ("n_nodes", C.c_int64), ("n_dof", C.c_int64), ("nnz", C.c_int64), ("n_blocks", C.c_int64),
                ("n_contrib", C.c_int64), ("n_multi_blocks", C.c_int64), ("n_side_slots", C.c_int64),
                ("tile_begin", C.c_int64), ("n_tiles_local", C.c_int64), ("n_tiles_owned", C.c_int64),
                ("row_begin", C.c_int64), ("n_rows", C.c_int64), ("q_dir", C.c_int32 * 3), ("m_dir", C.c_int32 * 3),
                ("n_local_ctrl", C.c_int32)]


class iga_shard(C.Structure):
    _fields_ = [("n_shards", C.c_int32), ("shard", C.c_int32)]


N_PROF = 10   # IGA_N_PROF: 0 K2, 1 K3(+scatter), 2 K4, 3 K5a, 4 K5b, 5 K5c, 6 staging, 7 K5x, 8 K3 nzdata, 9 apply
EXPORTS = ["iga_build_tables", "iga_build_tables_q", "iga_build_topology", "iga_build_topology_q",
           "iga_projection_error", "iga_select_degree", "iga_assemble", "iga_sensitivity", "iga_assemble_sensitivity",
           "iga_apply", "iga_volume", "iga_load_vector", "iga_interpolate",
           "iga_get_sizes",
           "iga_get_pattern", "iga_get_block_map", "iga_get_node_map", "iga_get_tables", "iga_get_pairs",
           "iga_set_projection", "iga_get_projection", "iga_set_profiling", "iga_get_kernel_times", "iga_free",
           "iga_last_error", "iga_version"]

_lib = None


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libiga.so not built at {LIB_PATH}; run __graft_entry__.build()")
    lib = C.CDLL(LIB_PATH)
    vp, i32, i64, d = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    lib.iga_build_tables.argtypes = [C.POINTER(iga_spline), i32, C.POINTER(iga_interface), i32,
                                     C.POINTER(iga_spline), i32, i32, C.POINTER(iga_shard), vp, C.POINTER(vp)]
    lib.iga_build_topology.argtypes = [C.POINTER(iga_spline), i32, C.POINTER(iga_interface), i32,
                                       C.POINTER(iga_spline), i32, i32, C.POINTER(iga_shard), C.POINTER(vp)]
    lib.iga_build_tables_q.argtypes = [C.POINTER(iga_spline), i32, C.POINTER(iga_interface), i32,
                                       C.POINTER(iga_spline), C.POINTER(i32), i32, C.POINTER(iga_shard), vp,
                                       C.POINTER(vp)]
    lib.iga_build_topology_q.argtypes = [C.POINTER(iga_spline), i32, C.POINTER(iga_interface), i32,
                                         C.POINTER(iga_spline), C.POINTER(i32), i32, C.POINTER(iga_shard),
                                         C.POINTER(vp)]
    lib.iga_projection_error.argtypes = [C.POINTER(iga_spline), C.POINTER(i32), i32, d, i32, C.POINTER(d), vp, vp]
    lib.iga_select_degree.argtypes = [C.POINTER(iga_spline), d, d, i32, i32, i32, C.POINTER(i32), C.POINTER(d), vp]
    lib.iga_assemble.argtypes = [vp, vp, vp, i32, d, vp, vp, vp]
    lib.iga_sensitivity.argtypes = [vp, vp, vp, i32, d, vp, vp, vp, vp]
    lib.iga_interpolate.argtypes = [vp, vp, vp, i32, d, vp, vp]
    lib.iga_apply.argtypes = [vp, vp, vp, i32, d, vp, vp, vp]
    lib.iga_assemble_sensitivity.argtypes = [vp, vp, vp, i32, d, vp, vp, vp, vp, vp]
    lib.iga_volume.argtypes = [vp, vp, vp, vp, vp]
    lib.iga_load_vector.argtypes = [vp, vp, vp, vp, vp]
    lib.iga_get_sizes.argtypes = [vp, C.POINTER(iga_sizes)]
    lib.iga_get_pattern.argtypes = [vp, vp, vp]
    lib.iga_get_block_map.argtypes = [vp, i64, i64, vp]
    lib.iga_get_node_map.argtypes = [vp, vp]
    lib.iga_get_tables.argtypes = [vp, vp]
    lib.iga_get_pairs.argtypes = [vp, vp]
    lib.iga_set_profiling.argtypes = [vp, i32]
    lib.iga_set_projection.argtypes = [vp, i32]
    lib.iga_get_projection.argtypes = [vp, C.POINTER(i32)]
    lib.iga_get_kernel_times.argtypes = [vp, vp, vp]
    lib.iga_free.argtypes = [vp]
    lib.iga_free.restype = None
    lib.iga_last_error.restype = C.c_char_p
    lib.iga_version.restype = C.c_char_p
    for name in EXPORTS:
        if name not in ("iga_free", "iga_last_error", "iga_version"):
            getattr(lib, name).restype = C.c_int
    _lib = lib
    return lib


def _check(status):
    if status != 0:
        raise IgaError(status, load().iga_last_error().decode())


_NP_OF_TORCH = {"torch.float64": np.float64, "torch.int64": np.int64, "torch.int32": np.int32}


def _ptr(x, n=None, dtype=np.float64, name="argument"):
    """Raw pointer of a torch tensor (host or CUDA) or a numpy array, after checking what
    the C ABI will read or write through it: C-contiguous, of `dtype`, with at least `n`
    elements (None: no size check), on the current CUDA device if it is a CUDA tensor.
    Raises ValueError (never an assert: the ABI trusts these n·sizeof bytes)."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError(f"{name}: numpy array must be C-contiguous")
        if x.dtype != np.dtype(dtype):
            raise ValueError(f"{name}: dtype {x.dtype}, expected {np.dtype(dtype)}")
        if n is not None and x.size < n:
            raise ValueError(f"{name}: {x.size} elements, needs {n}")
        return x.ctypes.data
    if not hasattr(x, "data_ptr"):
        raise ValueError(f"{name}: expected a numpy array or a torch tensor, got {type(x).__name__}")
    if not x.is_contiguous():
        raise ValueError(f"{name}: tensor must be contiguous")
    if _NP_OF_TORCH.get(str(x.dtype)) is not np.dtype(dtype).type:
        raise ValueError(f"{name}: dtype {x.dtype}, expected {np.dtype(dtype)}")
    if n is not None and x.numel() < n:
        raise ValueError(f"{name}: {x.numel()} elements, needs {n}")
    if x.is_cuda:
        import torch
        if x.device.index != torch.cuda.current_device():
            raise ValueError(f"{name}: on {x.device}, the handle works on cuda:{torch.cuda.current_device()}")
    return x.data_ptr()


def _stream_ptr(stream):
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream
        except ImportError:
            pass
        return None
    return getattr(stream, "cuda_stream", stream)


def _spline(s, keep):
    sp = iga_spline()
    sp.dim = s.dim
    for k in range(3):
        if k < s.dim:
            U = np.ascontiguousarray(s.knots[k], dtype=np.float64)
            keep.append(U)
            sp.degree[k] = s.degree[k]
            sp.n_knots[k] = len(U)
            sp.knots[k] = U.ctypes.data_as(C.POINTER(C.c_double))
    if s.ctrl is not None:
        P = np.ascontiguousarray(s.ctrl, dtype=np.float64)
        keep.append(P)
        sp.ctrl = P.ctypes.data_as(C.POINTER(C.c_double))
    if getattr(s, "weights", None) is not None:
        w = np.ascontiguousarray(s.weights, dtype=np.float64)
        keep.append(w)
        sp.weights = w.ctypes.data_as(C.POINTER(C.c_double))
    return sp


def _qvec(q, d):
    qs = [int(q)] * d if np.ndim(q) == 0 else [int(x) for x in q]
    if len(qs) != d:
        raise ValueError(f"q has {len(qs)} entries for d = {d}")
    return (C.c_int32 * 3)(*(qs + [0] * (3 - d)))


def projection_error(macro, q, nu, n_samples=8, m_extra=0, e_tile=None, stream=None):
    """iga_projection_error: E_proj (Eq. 59) of the macro spline for degree(s) q; e_tile
    (optional, n_tiles doubles, host or device) receives the per-tile maxima."""
    keep = []
    mac = _spline(macro, keep)
    e = C.c_double()
    _check(load().iga_projection_error(C.byref(mac), _qvec(q, macro.dim), int(m_extra), float(nu), int(n_samples),
                                       C.byref(e), _ptr(e_tile, name="e_tile"), _stream_ptr(stream)))
    return e.value


def select_degree(macro, nu, tol, n_samples=8, m_extra=0, q_max=0, stream=None):
    """iga_select_degree (Eq. 65, reading R19): (q per direction, E_proj(q))."""
    keep = []
    mac = _spline(macro, keep)
    q = (C.c_int32 * 3)()
    e = C.c_double()
    _check(load().iga_select_degree(C.byref(mac), float(nu), float(tol), int(m_extra), int(n_samples), int(q_max),
                                    q, C.byref(e), _stream_ptr(stream)))
    return tuple(q[k] for k in range(macro.dim)), e.value


class Assembler:
    """Handle around iga_build_tables for a problem description (synth.Problem-like:
    .tile (patches), .interfaces, .macro (degree/knots), .q, .n_gauss).
    shard=(n_shards, shard): form only that slab of the problem (iga_shard)."""

    def __init__(self, prob, n_gauss=0, stream=None, topology_only=False, shard=None):
        lib = load()
        keep = []
        arr = (iga_spline * len(prob.tile))(*[_spline(s, keep) for s in prob.tile])
        ifs = (iga_interface * max(1, len(prob.interfaces)))()
        for n, f in enumerate(prob.interfaces):
            ifs[n] = iga_interface(f.patch_a, f.dir_a, f.side_a, f.patch_b, f.dir_b, f.side_b)
        mac = _spline(prob.macro, keep)
        sh = C.byref(iga_shard(int(shard[0]), int(shard[1]))) if shard is not None else None
        h = C.c_void_p()
        qv = _qvec(prob.q, prob.macro.dim)   # one projection degree per direction (iga_build_tables_q)
        if topology_only:
            _check(lib.iga_build_topology_q(arr, len(prob.tile), ifs, len(prob.interfaces), C.byref(mac), qv,
                                            n_gauss, sh, C.byref(h)))
        else:
            _check(lib.iga_build_tables_q(arr, len(prob.tile), ifs, len(prob.interfaces), C.byref(mac), qv,
                                          n_gauss, sh, _stream_ptr(stream), C.byref(h)))
        self._h = h
        self.sizes = iga_sizes()
        _check(lib.iga_get_sizes(h, C.byref(self.sizes)))

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.iga_free(self._h)
            self._h = None

    # --- hot path -----------------------------------------------------------
    # required lengths of the [any] arguments (include/iga.h)
    def _ctrl(self, ctrl):
        return _ptr(ctrl, self.sizes.n_macro_cp * self.sizes.dim, name="macro_ctrl")

    def _young(self, young):
        n = _numel(young)
        if n not in (1, self.sizes.n_tiles):
            raise ValueError(f"young: {n} values, expected 1 or n_tiles = {self.sizes.n_tiles}")
        return _ptr(young, n, name="young"), int(n > 1)

    def _nloc(self):
        s = self.sizes
        return s.n_local_rows * s.n_tiles_local * s.dim * s.dim

    def assemble(self, ctrl, young, nu, values, local=None, stream=None):
        yp, per_tile = self._young(young)
        _check(load().iga_assemble(self._h, self._ctrl(ctrl), yp, per_tile, float(nu),
                                   _ptr(values, self.sizes.nnz, name="csr_values"),
                                   _ptr(local, self._nloc(), name="local_values"), _stream_ptr(stream)))

    def sensitivity(self, ctrl, young, nu, u, v, grad, stream=None):
        s = self.sizes
        yp, per_tile = self._young(young)
        _check(load().iga_sensitivity(self._h, self._ctrl(ctrl), yp, per_tile, float(nu),
                                      _ptr(u, s.n_dof, name="u"), _ptr(v, s.n_dof, name="v"),
                                      _ptr(grad, s.n_macro_cp * s.dim, name="grad"), _stream_ptr(stream)))

    def assemble_sensitivity(self, ctrl, young, nu, u, v, values, grad, stream=None):
        """K (CSR values) and g = uᵀ(∂K/∂P)v in one call (iga_assemble_sensitivity)."""
        s = self.sizes
        yp, per_tile = self._young(young)
        _check(load().iga_assemble_sensitivity(self._h, self._ctrl(ctrl), yp, per_tile, float(nu),
                                               _ptr(u, s.n_dof, name="u"), _ptr(v, s.n_dof, name="v"),
                                               _ptr(values, s.nnz, name="csr_values"),
                                               _ptr(grad, s.n_macro_cp * s.dim, name="grad"), _stream_ptr(stream)))

    def volume(self, ctrl, grad=None, stream=None):
        """V^π (float) and optionally dV^π/dP into grad (iga_volume)."""
        out = np.zeros(1)
        _check(load().iga_volume(self._h, self._ctrl(ctrl), out.ctypes.data,
                                 _ptr(grad, self.sizes.n_macro_cp * self.sizes.dim, name="grad"), _stream_ptr(stream)))
        return float(out[0])

    def load_vector(self, ctrl, body_force, f, stream=None):
        """Body-force load vector for a constant b (iga_load_vector)."""
        b = np.ascontiguousarray(body_force, dtype=np.float64)
        if b.size != self.sizes.dim:
            raise ValueError(f"body_force: {b.size} values, expected d = {self.sizes.dim}")
        _check(load().iga_load_vector(self._h, self._ctrl(ctrl), b.ctypes.data, _ptr(f, self.sizes.n_rows, name="f"),
                                      _stream_ptr(stream)))

    def apply(self, ctrl, young, nu, u, y, stream=None):
        """Matrix-free y = K^π u (iga_apply)."""
        yp, per_tile = self._young(young)
        _check(load().iga_apply(self._h, self._ctrl(ctrl), yp, per_tile, float(nu), _ptr(u, self.sizes.n_dof, name="u"),
                                _ptr(y, self.sizes.n_rows, name="y"), _stream_ptr(stream)))

    def interpolate(self, ctrl, young, nu, coef, stream=None):
        s = self.sizes
        yp, per_tile = self._young(young)
        _check(load().iga_interpolate(self._h, self._ctrl(ctrl), yp, per_tile, float(nu),
                                      _ptr(coef, s.n_tiles_local * s.dim * s.dim * s.k_stride, name="coef"),
                                      _stream_ptr(stream)))

    # --- accessors ----------------------------------------------------------
    def pattern(self, row_ptr=None, col_idx=None):
        _check(load().iga_get_pattern(self._h, _ptr(row_ptr, self.sizes.n_rows + 1, np.int64, "row_ptr"),
                                      _ptr(col_idx, self.sizes.nnz, np.int32, "col_idx")))

    def block_map(self, t_begin=0, t_end=None):
        t_end = self.sizes.n_tiles_local if t_end is None else t_end
        out = np.empty(((t_end - t_begin) * self.sizes.n_local_rows, 2), dtype=np.int64)
        _check(load().iga_get_block_map(self._h, t_begin, t_end, out.ctypes.data))
        return out

    def node_map_for(self, n_local_ctrl=None):
        nl = self.sizes.n_local_ctrl
        if n_local_ctrl is not None and int(n_local_ctrl) != nl:
            raise ValueError(f"n_local_ctrl={n_local_ctrl}: the handle's tiles have {nl} local control points")
        n_local_ctrl = nl
        out = np.empty(self.sizes.n_tiles_local * n_local_ctrl, dtype=np.int32)
        _check(load().iga_get_node_map(self._h, out.ctypes.data))
        return out.reshape(self.sizes.n_tiles_local, n_local_ctrl)

    def tables(self):
        out = np.empty((self.sizes.n_local_rows, self.sizes.n_k), dtype=np.float64)
        _check(load().iga_get_tables(self._h, out.ctypes.data))
        return out

    def pairs(self):
        out = np.empty((self.sizes.n_local_rows, 2), dtype=np.int32)
        _check(load().iga_get_pairs(self._h, out.ctypes.data))
        return out

    def set_projection(self, m):
        """L2 projection with an m-point Gauss rule per direction (m = 0, or q+1 when
        isotropic: interpolation at the q_k+1 Gauss nodes)."""
        _check(load().iga_set_projection(self._h, int(m)))
        _check(load().iga_get_sizes(self._h, C.byref(self.sizes)))   # m_dir

    def projection(self):
        m = C.c_int32()
        _check(load().iga_get_projection(self._h, C.byref(m)))
        return m.value

    def set_profiling(self, enable=True):
        _check(load().iga_set_profiling(self._h, int(enable)))

    def kernel_times(self):
        ms = np.zeros(N_PROF, dtype=np.float64)
        n = np.zeros(N_PROF, dtype=np.int64)
        _check(load().iga_get_kernel_times(self._h, ms.ctypes.data, n.ctypes.data))
        return ms, n


def _numel(x):
    return x.size if isinstance(x, np.ndarray) else x.numel()
