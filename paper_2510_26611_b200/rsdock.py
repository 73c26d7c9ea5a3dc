"""Thin Python binding of librsdock (include/rs_dock.h) -- argument marshalling only.

Every step of the scoring path runs in the library's CUDA kernels; there is no Python or CPU
fallback: if librsdock.so is missing or was built without a usable device, the calls raise.
PyTorch is used only for device memory and streams (tensors' data_ptr / current stream).

Same names as the C ABI: rs_params_default, rs_build_protein, rs_score_poses,
rs_score_poses_async, rs_get_info, rs_export_tables, rs_export_setup, rs_last_error, rs_free.
`Protein` is a small RAII wrapper over the opaque handle.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RSDOCK_LIB") or os.path.join(_PKG, "librsdock.so")

RS_E_INVALID_ARG, RS_E_CUDA, RS_E_NOMEM, RS_E_NO_DEVICE = -1, -2, -3, -4
RS_FLAG_HOST_ONLY = 1
RS_FLAG_F32_FACTORS = 2
RS_FLAG_BOX_SCHEME_B = 4
RS_FLAG_DEVICE_FFT = 8
RS_FLAG_HOST_FFT = 16
RS_FLAG_TUCKER_EVAL = 32
RS_PATH_WINDOW, RS_PATH_L2, RS_PATH_L2_RUNTIME, RS_PATH_TUCKER = 1, 2, 3, 4

EXPORTED = ["rs_params_default", "rs_build_protein", "rs_combine_proteins", "rs_restrict_box", "rs_score_poses", "rs_score_poses_async",
            "rs_score_forces", "rs_ppiem_scan", "rs_landscape_minima",
            "rs_score_path", "rs_export_tucker", "rs_save_handle", "rs_load_handle", "rs_get_info", "rs_export_tables", "rs_export_setup", "rs_last_error", "rs_free"]


class rs_params(ctypes.Structure):
    _fields_ = [("grid_n", ctypes.c_int32), ("rank_R", ctypes.c_int32),
                ("eps_compress", ctypes.c_double), ("eps_quad", ctypes.c_double),
                ("sigma_split", ctypes.c_double), ("eps_split", ctypes.c_double),
                ("sigma_vdw", ctypes.c_double), ("dmin_cap", ctypes.c_double),
                ("tucker_rank_max", ctypes.c_int32), ("als_sweeps", ctypes.c_int32),
                ("device", ctypes.c_int32), ("n_threads", ctypes.c_int32),
                ("seed", ctypes.c_uint64), ("flags", ctypes.c_uint32),
                ("nbr_cell", ctypes.c_double)]


class rs_info(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("b", ctypes.c_double), ("h", ctypes.c_double),
                ("inv_h", ctypes.c_double), ("R", ctypes.c_int32), ("R_exact", ctypes.c_int32),
                ("tucker_r", ctypes.c_int32 * 3), ("quad_K", ctypes.c_int32),
                ("quad_s", ctypes.c_double), ("quad_Ls", ctypes.c_double),
                ("quad_err", ctypes.c_double), ("R_long_ref", ctypes.c_int32),
                ("R_short", ctypes.c_int32), ("n_sigma", ctypes.c_int32),
                ("n_atoms", ctypes.c_int64), ("tucker_err", ctypes.c_double),
                ("cp_core_err", ctypes.c_double), ("sampled_max_err", ctypes.c_double),
                ("sampled_rms_err", ctypes.c_double), ("n_err_samples", ctypes.c_int32),
                ("sigma_vdw", ctypes.c_double), ("dmin_cap", ctypes.c_double),
                ("nbr_cells", ctypes.c_int64), ("nbr_entries", ctypes.c_int64),
                ("nbr_shift", ctypes.c_int32), ("device_bytes", ctypes.c_int64),
                ("setup_seconds", ctypes.c_double), ("on_device", ctypes.c_int32),
                ("factor_bits", ctypes.c_int32), ("box_lo", ctypes.c_int32 * 3),
                ("box_hi", ctypes.c_int32 * 3)]


_lib = None
_dp = ctypes.POINTER(ctypes.c_double)
_vp = ctypes.c_void_p


def load():
    """Load librsdock.so (raises if absent: build it with __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} not built; run __graft_entry__.build() -- there is no "
                           "CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    L.rs_params_default.argtypes = [ctypes.POINTER(rs_params)]
    L.rs_build_protein.argtypes = [_vp, _vp, ctypes.c_int64, ctypes.c_double,
                                   ctypes.POINTER(rs_params)]
    L.rs_build_protein.restype = _vp
    L.rs_combine_proteins.argtypes = [_vp, ctypes.c_int32, ctypes.c_int32]
    L.rs_combine_proteins.restype = _vp
    L.rs_restrict_box.argtypes = [_vp, _vp, _vp, ctypes.c_int32, ctypes.c_int32]
    L.rs_restrict_box.restype = _vp
    L.rs_score_poses.argtypes = [_vp, _vp, _vp, ctypes.c_int64, _vp, ctypes.c_int64, _vp, _vp]
    L.rs_score_poses.restype = ctypes.c_int64
    L.rs_score_poses_async.argtypes = [_vp, _vp, _vp, ctypes.c_int64, _vp, ctypes.c_int64, _vp,
                                       _vp, _vp, _vp]
    L.rs_score_poses_async.restype = ctypes.c_int64
    L.rs_score_forces.argtypes = [_vp, _vp, _vp, ctypes.c_int64, _vp, ctypes.c_int64, _vp, _vp, _vp]
    L.rs_score_forces.restype = ctypes.c_int64
    L.rs_ppiem_scan.argtypes = [_vp, _vp, _vp, ctypes.c_int64, _vp, _vp, ctypes.c_int32, _vp,
                                ctypes.c_int32, ctypes.c_double, ctypes.c_double, ctypes.c_int32,
                                _vp, _vp, _vp]
    L.rs_ppiem_scan.restype = ctypes.c_int64
    L.rs_landscape_minima.argtypes = [_vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _vp]
    L.rs_landscape_minima.restype = ctypes.c_int32
    L.rs_export_tucker.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp]
    L.rs_export_tucker.restype = ctypes.c_int
    L.rs_save_handle.argtypes = [_vp, ctypes.c_char_p]
    L.rs_save_handle.restype = ctypes.c_int
    L.rs_load_handle.argtypes = [ctypes.c_char_p, ctypes.c_int32, ctypes.c_int32]
    L.rs_load_handle.restype = _vp
    L.rs_score_path.argtypes = [_vp, _vp, ctypes.c_int64]
    L.rs_score_path.restype = ctypes.c_int
    L.rs_get_info.argtypes = [_vp, ctypes.POINTER(rs_info)]
    L.rs_get_info.restype = ctypes.c_int
    L.rs_export_tables.argtypes = [_vp] + [_vp] * 6
    L.rs_export_tables.restype = ctypes.c_int
    L.rs_export_setup.argtypes = [_vp, _vp, _vp, _vp, _vp]
    L.rs_export_setup.restype = ctypes.c_int
    L.rs_last_error.restype = ctypes.c_char_p
    L.rs_free.argtypes = [_vp]
    _lib = L
    return L


# ---------------------------------------------------------------------------- raw C names

def rs_params_default(**overrides) -> rs_params:
    p = rs_params()
    load().rs_params_default(ctypes.byref(p))
    for k, v in overrides.items():
        setattr(p, k, v)
    return p


def rs_last_error() -> str:
    return load().rs_last_error().decode()


def _ptr(x, name="array", count=None, dtype="float64", cuda=None):
    """Data pointer of a numpy array or torch tensor after checking what the C ABI reads from
    it: the element type, C-contiguity, at least `count` elements and (cuda=True/False) where
    it lives.  Marshalling only: nothing is converted or copied; a mismatch raises."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        if x.dtype != np.dtype(dtype):
            raise TypeError(f"{name}: expected {dtype}, got {x.dtype}")
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError(f"{name}: must be C-contiguous")
        if cuda:
            raise ValueError(f"{name}: must be a CUDA tensor (a numpy array is host memory)")
        n, ptr = x.size, x.ctypes.data
    else:
        import torch
        want = {"float64": torch.float64, "int32": torch.int32, "int64": torch.int64}[dtype]
        if x.dtype != want:
            raise TypeError(f"{name}: expected torch.{dtype}, got {x.dtype}")
        if not x.is_contiguous():
            raise ValueError(f"{name}: must be contiguous")
        if cuda is not None and bool(x.is_cuda) != bool(cuda):
            raise ValueError(f"{name}: must be a {'CUDA' if cuda else 'host'} tensor")
        n, ptr = x.numel(), x.data_ptr()
    if count is not None and n < count:
        raise ValueError(f"{name}: needs at least {count} elements, has {n}")
    return ptr


def rs_build_protein(q, xyz, box_half_width, params: rs_params | None = None):
    q = np.ascontiguousarray(q, dtype=np.float64)
    xyz = np.ascontiguousarray(xyz, dtype=np.float64).reshape(-1, 3)
    h = load().rs_build_protein(q.ctypes.data, xyz.ctypes.data, q.shape[0], float(box_half_width),
                                ctypes.byref(params) if params is not None else None)
    if not h:
        raise RuntimeError("rs_build_protein: " + rs_last_error())
    return h


def rs_combine_proteins(parts, flags=0):
    """parts: sequence of rs_handle pointers (Eq. (23) complex; see include/rs_dock.h)."""
    arr = (ctypes.c_void_p * len(parts))(*parts)
    h = load().rs_combine_proteins(ctypes.cast(arr, ctypes.c_void_p), len(parts), int(flags))
    if not h:
        raise RuntimeError("rs_combine_proteins: " + rs_last_error())
    return h


def rs_restrict_box(h, lo, hi, rank, flags=0):
    """Box-restricted recompression (N3, scheme (C)); lo, hi: 3 cell indices each."""
    lo = np.ascontiguousarray(lo, dtype=np.int32)
    hi = np.ascontiguousarray(hi, dtype=np.int32)
    r = load().rs_restrict_box(h, lo.ctypes.data, hi.ctypes.data, int(rank), int(flags))
    if not r:
        raise RuntimeError("rs_restrict_box: " + rs_last_error())
    return r


def rs_score_poses(h, q_lig, xyz_lig, n_lig, poses, P, energies_out, mindist_out) -> int:
    n_lig, P = int(n_lig), int(P)
    r = load().rs_score_poses(h, _ptr(q_lig, "q_lig", n_lig), _ptr(xyz_lig, "xyz_lig", 3 * n_lig),
                              n_lig, _ptr(poses, "poses", 7 * P), P,
                              _ptr(energies_out, "energies_out", P), _ptr(mindist_out, "mindist_out", P))
    if r < 0:
        raise RuntimeError(f"rs_score_poses ({r}): " + rs_last_error())
    return int(r)


def rs_score_poses_async(h, q_lig, xyz_lig, n_lig, poses, P, energies_out, mindist_out,
                         invalid_count=None, stream=None) -> int:
    n_lig, P = int(n_lig), int(P)
    r = load().rs_score_poses_async(h, _ptr(q_lig, "q_lig", n_lig, cuda=True),
                                    _ptr(xyz_lig, "xyz_lig", 3 * n_lig, cuda=True), n_lig,
                                    _ptr(poses, "poses", 7 * P, cuda=True), P,
                                    _ptr(energies_out, "energies_out", P, cuda=True),
                                    _ptr(mindist_out, "mindist_out", P, cuda=True),
                                    _ptr(invalid_count, "invalid_count", 1, "int64", cuda=True),
                                    stream)
    if r < 0:
        raise RuntimeError(f"rs_score_poses_async ({r}): " + rs_last_error())
    return int(r)


def rs_score_forces(h, q_lig, xyz_lig, n_lig, poses, P, forces_out, invalid_count=None,
                    stream=None) -> int:
    n_lig, P = int(n_lig), int(P)
    r = load().rs_score_forces(h, _ptr(q_lig, "q_lig", n_lig, cuda=True),
                               _ptr(xyz_lig, "xyz_lig", 3 * n_lig, cuda=True), n_lig,
                               _ptr(poses, "poses", 7 * P, cuda=True), P,
                               _ptr(forces_out, "forces_out", 9 * P, cuda=True),
                               _ptr(invalid_count, "invalid_count", 1, "int64", cuda=True), stream)
    if r < 0:
        raise RuntimeError(f"rs_score_forces ({r}): " + rs_last_error())
    return int(r)


def rs_ppiem_scan(h, q_lig, xyz_lig, centre, dirs, quats, s_start, tol=1e-3, max_iter=64):
    """PPIEM scan (NEXT row N2): returns (energies, s, status), each m_P x m_L (numpy)."""
    q_lig = np.ascontiguousarray(q_lig, dtype=np.float64) if isinstance(q_lig, np.ndarray) else q_lig
    xyz_lig = np.ascontiguousarray(xyz_lig, dtype=np.float64) if isinstance(xyz_lig, np.ndarray) else xyz_lig
    centre = np.ascontiguousarray(centre, dtype=np.float64)
    dirs = np.ascontiguousarray(dirs, dtype=np.float64)
    quats = np.ascontiguousarray(quats, dtype=np.float64)
    m_P, m_L = dirs.shape[0], quats.shape[0]
    E = np.empty((m_P, m_L))
    s = np.empty((m_P, m_L))
    st = np.empty((m_P, m_L), dtype=np.int32)
    n_lig = int(q_lig.shape[0])
    r = load().rs_ppiem_scan(h, _ptr(q_lig, "q_lig", n_lig), _ptr(xyz_lig, "xyz_lig", 3 * n_lig),
                             n_lig, _ptr(centre, "centre", 3), _ptr(dirs, "dirs", 3 * m_P), m_P,
                             _ptr(quats, "quats", 4 * m_L), m_L, float(s_start), float(tol),
                             int(max_iter), _ptr(E), _ptr(s), _ptr(st, "status", dtype="int32"))
    if r < 0:
        raise RuntimeError(f"rs_ppiem_scan ({r}): " + rs_last_error())
    return E, s, st


def rs_landscape_minima(E, top_k):
    """PPIEM step A6: flat indices j*m_L + k of up to top_k local minima, by energy."""
    E = np.ascontiguousarray(E, dtype=np.float64)
    out = np.empty(max(int(top_k), 1), dtype=np.int32)
    r = load().rs_landscape_minima(_ptr(E), E.shape[0], E.shape[1], int(top_k),
                                   _ptr(out, "idx_out", dtype="int32"))
    if r < 0:
        raise RuntimeError("rs_landscape_minima: " + rs_last_error())
    return out[:r].copy()


def rs_score_path(h, xyz_lig) -> int:
    """Kernel variant rs_score_poses runs for this ligand (RS_PATH_WINDOW / _L2 / _L2_RUNTIME)."""
    if isinstance(xyz_lig, np.ndarray):
        xyz_lig = np.ascontiguousarray(xyz_lig, dtype=np.float64).reshape(-1, 3)
    n = xyz_lig.shape[0] if xyz_lig.ndim == 2 else xyz_lig.shape[0] // 3
    r = load().rs_score_path(h, _ptr(xyz_lig, "xyz_lig", count=3 * n, cuda=False), n)
    if r < 0:
        raise RuntimeError("rs_score_path: " + rs_last_error())
    return int(r)


def rs_get_info(h) -> dict:
    info = rs_info()
    if load().rs_get_info(h, ctypes.byref(info)) != 0:
        raise RuntimeError(rs_last_error())
    out = {}
    for name, _ in rs_info._fields_:
        v = getattr(info, name)
        out[name] = list(v) if name in ("tucker_r", "box_lo", "box_hi") else v
    return out


def rs_export_tables(h) -> dict:
    info = rs_get_info(h)
    n, R, ns, Rs = info["n"], info["R"], info["n_sigma"], info["R_short"]
    F = [np.empty((n, R)) for _ in range(3)]
    S = [np.empty((2 * ns + 1, Rs)) for _ in range(3)]
    rc = load().rs_export_tables(h, *[a.ctypes.data for a in F], *[a.ctypes.data for a in S])
    if rc != 0:
        raise RuntimeError(rs_last_error())
    return dict(n=n, b=info["b"], R=R, n_sigma=ns, Rs=Rs, F1=F[0], F2=F[1], F3=F[2], S1=S[0],
                S2=S[1], S3=S[2])


def rs_export_setup(h) -> dict:
    info = rs_get_info(h)
    K1 = info["quad_K"] + 1
    t, a = np.empty(K1), np.empty(K1)
    is_long = np.empty(K1, dtype=np.int32)
    cells = np.empty((info["n_atoms"], 3), dtype=np.int32)
    rc = load().rs_export_setup(h, t.ctypes.data, a.ctypes.data, is_long.ctypes.data,
                                cells.ctypes.data)
    if rc != 0:
        raise RuntimeError(rs_last_error())
    return dict(t=t, a=a, is_long=is_long.astype(bool), cells=cells, s=info["quad_s"],
                K=info["quad_K"], Ls=info["quad_Ls"])


def rs_export_tucker(h) -> dict:
    """The handle's Tucker form (N5): U0, U1, U2 (n x r_l, row i = U_l[i, :]) and G."""
    r = np.zeros(3, dtype=np.int32)
    if load().rs_export_tucker(h, r.ctypes.data, None, None, None, None) != 0:
        raise RuntimeError("rs_export_tucker: " + rs_last_error())
    n = rs_get_info(h)["n"]
    U = [np.empty((n, int(r[l]))) for l in range(3)]
    G = np.empty(tuple(int(x) for x in r))
    if load().rs_export_tucker(h, r.ctypes.data, U[0].ctypes.data, U[1].ctypes.data,
                               U[2].ctypes.data, G.ctypes.data) != 0:
        raise RuntimeError("rs_export_tucker: " + rs_last_error())
    return {"U0": U[0], "U1": U[1], "U2": U[2], "G": G}


def rs_save_handle(h, path) -> None:
    if load().rs_save_handle(h, os.fsencode(path)) != 0:
        raise RuntimeError("rs_save_handle: " + rs_last_error())


def rs_load_handle(path, device=-1, flags=0):
    h = load().rs_load_handle(os.fsencode(path), int(device), int(flags))
    if not h:
        raise RuntimeError("rs_load_handle: " + rs_last_error())
    return h


def rs_free(h) -> None:
    if h:
        load().rs_free(h)


# ---------------------------------------------------------------------------- wrapper

class Protein:
    """Owns one rs_handle (the protein's RS tensor, resident on the device)."""

    def __init__(self, q, xyz, box_half_width, **params):
        self._h = None
        self.params = rs_params_default(**params)
        self._h = rs_build_protein(q, xyz, box_half_width, self.params)
        self.info = rs_get_info(self._h)

    def restrict_box(self, lo, hi, rank, flags=0):
        """A new Protein whose long-range factors are recompressed inside the cell box
        [lo, hi] (N3, scheme (C)); NaN rows outside it."""
        new = type(self).__new__(type(self))
        new._h = None
        new.params = self.params
        new._h = rs_restrict_box(self._h, lo, hi, rank, flags)
        new.info = rs_get_info(new._h)
        return new

    @classmethod
    def combine(cls, parts, flags=0):
        """The complex of several proteins on one grid (Eq. (23)): rank-concatenated factors,
        union of the atoms.  The parts stay valid and owned by their objects."""
        self = cls.__new__(cls)
        self._h = None
        self.params = parts[0].params
        self._h = rs_combine_proteins([p.handle for p in parts], flags)
        self.info = rs_get_info(self._h)
        return self

    def export_tucker(self) -> dict:
        return rs_export_tucker(self._h)

    def save(self, path):
        """Write the handle's tables to `path` (rs_save_handle: SPEC's kernel cache)."""
        rs_save_handle(self._h, path)

    @classmethod
    def load(cls, path, device=-1, flags=0):
        """A Protein from a file written by save(), uploaded to `device` without a setup."""
        self = cls.__new__(cls)
        self._h = None
        self._h = rs_load_handle(path, device, flags)
        self.info = rs_get_info(self._h)
        self.params = None
        return self

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            rs_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def export_tables(self) -> dict:
        return rs_export_tables(self._h)

    def export_setup(self) -> dict:
        return rs_export_setup(self._h)

    def score(self, q_lig, xyz_lig, poses, energies_out=None, mindist_out=None):
        """Synchronous scoring.  Inputs may be numpy arrays (host) or torch tensors (host or
        device).  Returns (energies, mindist, n_invalid); outputs live where the poses live
        unless given."""
        P = int(poses.shape[0])
        L = int(q_lig.shape[0])
        if isinstance(poses, np.ndarray):
            poses = np.ascontiguousarray(poses, dtype=np.float64)
            q_lig = np.ascontiguousarray(q_lig, dtype=np.float64)
            xyz_lig = np.ascontiguousarray(xyz_lig, dtype=np.float64)
            if energies_out is None:
                energies_out = np.empty(P)
            if mindist_out is None:
                mindist_out = np.empty(P)
        else:
            import torch
            if energies_out is None:
                energies_out = torch.empty(P, dtype=torch.float64, device=poses.device)
            if mindist_out is None:
                mindist_out = torch.empty(P, dtype=torch.float64, device=poses.device)
        inv = rs_score_poses(self._h, q_lig, xyz_lig, L, poses, P, energies_out, mindist_out)
        return energies_out, mindist_out, inv

    def forces_async(self, q_lig, xyz_lig, poses, forces_out, invalid_count=None, stream=None):
        """Enqueue the rigid-ligand forces (P x 9 device tensor: net force, torque about the
        centre, Eq. (24) radial resultant) on `stream` (default: torch's current stream)."""
        import torch
        if stream is None:
            stream = torch.cuda.current_stream(poses.device)
        s = stream.cuda_stream if hasattr(stream, "cuda_stream") else stream
        return rs_score_forces(self._h, q_lig, xyz_lig, int(q_lig.shape[0]), poses,
                               int(poses.shape[0]), forces_out, invalid_count, s)

    def score_async(self, q_lig, xyz_lig, poses, energies_out, mindist_out, invalid_count=None,
                    stream=None):
        """Enqueue scoring of device tensors on `stream` (default: torch's current stream)."""
        import torch
        if stream is None:
            stream = torch.cuda.current_stream(poses.device)
        s = stream.cuda_stream if hasattr(stream, "cuda_stream") else stream
        return rs_score_poses_async(self._h, q_lig, xyz_lig, int(q_lig.shape[0]), poses,
                                    int(poses.shape[0]), energies_out, mindist_out, invalid_count,
                                    s)
