"""Thin ctypes binding of libhbpdc.so (include/hbpdc.h).

Argument marshalling only: every step of the hot path runs in the library's
CUDA kernels.  Device arrays are torch float64 CUDA tensors (PyTorch provides
device memory and the stream); there is no CPU fallback -- if the extension is
missing or no GPU is present, the calls raise.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HBPDC_LIB", os.path.join(_HERE, "libhbpdc.so"))

ADVECTION, EULER, NAVIER_STOKES = 0, 1, 2
GLL, GL = 0, 1
PC_NONE, PC_BJEXT, PC_BJEXT_H = 0, 1, 2
PC_PER_STEP_PER_ALPHA, PC_PER_NEWTON = 0, 1
JVP_AUTO, JVP_FD, JVP_EXACT, JVP_LINEAR = 0, 1, 2, 3
_EQ = {"advection": ADVECTION, "euler": EULER, "navier_stokes": NAVIER_STOKES}
_PC = {"none": PC_NONE, "bjext": PC_BJEXT, "bjext_h": PC_BJEXT_H}
_JVP = {"auto": JVP_AUTO, "fd": JVP_FD, "exact": JVP_EXACT, "linear": JVP_LINEAR}

STATUS = {0: "OK", 1: "E_ARG", 2: "E_CUDA", 3: "E_NCCL", 4: "E_OOM", 5: "E_NONFINITE",
          6: "E_NEG_PRESSURE", 7: "E_LU_SINGULAR", 8: "E_NEWTON", 9: "E_GMRES"}

EXPORTS = ["hbpdc_init", "hbpdc_local_shape", "hbpdc_node_coords", "hbpdc_node_coords_z", "hbpdc_rhs", "hbpdc_residual",
           "hbpdc_jvp", "hbpdc_precond_build", "hbpdc_precond_set", "hbpdc_precond_export",
           "hbpdc_precond_apply", "hbpdc_step", "hbpdc_step_host", "hbpdc_reset", "hbpdc_profile",
           "hbpdc_profile_read", "hbpdc_launch_count", "hbpdc_last_error", "hbpdc_finalize",
           "hbpdc_partition", "hbpdc_nccl_unique_id", "hbpdc_loopback_group_create",
           "hbpdc_loopback_group_destroy"]
COMM_AUTO, COMM_NCCL, COMM_LOOPBACK = 0, 1, 2
_COMM = {"auto": COMM_AUTO, "nccl": COMM_NCCL, "loopback": COMM_LOOPBACK}


class Problem(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int), ("equation", ctypes.c_int), ("a", ctypes.c_double * 2),
                ("gamma", ctypes.c_double), ("mach_eps", ctypes.c_double), ("mu", ctypes.c_double),
                ("prandtl", ctypes.c_double), ("N", ctypes.c_int), ("nodes", ctypes.c_int),
                ("nx", ctypes.c_int), ("ny", ctypes.c_int), ("xmin", ctypes.c_double),
                ("xmax", ctypes.c_double), ("ymin", ctypes.c_double), ("ymax", ctypes.c_double),
                ("flux", ctypes.c_int), ("lifting", ctypes.c_int), ("q", ctypes.c_int),
                ("kmax", ctypes.c_int), ("eta_br2", ctypes.c_double), ("nz", ctypes.c_int),
                ("zmin", ctypes.c_double), ("zmax", ctypes.c_double), ("az", ctypes.c_double)]


class SolverOpts(ctypes.Structure):
    _fields_ = [("newton_rtol", ctypes.c_double), ("newton_atol_dw", ctypes.c_double),
                ("newton_floor", ctypes.c_double), ("newton_max", ctypes.c_int),
                ("gmres_rtol", ctypes.c_double), ("gmres_restart", ctypes.c_int),
                ("krylov_max_per_newton", ctypes.c_int), ("precond", ctypes.c_int),
                ("precond_policy", ctypes.c_int), ("jvp_mode", ctypes.c_int), ("batch_stages", ctypes.c_int),
                ("gmres_sstep", ctypes.c_int), ("schur", ctypes.c_int)]


class Dist(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int), ("nranks", ctypes.c_int), ("px", ctypes.c_int),
                ("py", ctypes.c_int), ("nccl_unique_id", ctypes.c_void_p),
                ("cuda_stream", ctypes.c_void_p), ("device", ctypes.c_int), ("own_stream", ctypes.c_int),
                ("comm", ctypes.c_int), ("loopback_group", ctypes.c_void_p), ("force_halo", ctypes.c_int)]


class StepStats(ctypes.Structure):
    _fields_ = [("stage_solves", ctypes.c_int), ("newton_its", ctypes.c_int),
                ("gmres_its", ctypes.c_int), ("precond_builds", ctypes.c_int),
                ("max_krylov_j", ctypes.c_int), ("jvp_calls", ctypes.c_int),
                ("precond_applies", ctypes.c_int), ("precond_k_reused", ctypes.c_int),
                ("final_newton_rel", ctypes.c_double),
                ("wall_s", ctypes.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def load():
    """Load libhbpdc.so; raise if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} not built: run __graft_entry__.build() "
                           "(make -C paper_2109_04804_b200/csrc)")
    lib = ctypes.CDLL(LIB_PATH)
    P, D, I, V = ctypes.c_void_p, ctypes.c_double, ctypes.c_int, None
    sig = {
        "hbpdc_init": (I, [ctypes.POINTER(Problem), ctypes.POINTER(SolverOpts), ctypes.POINTER(Dist),
                           ctypes.POINTER(P)]),
        "hbpdc_local_shape": (I, [P] + [ctypes.POINTER(ctypes.c_int)] * 6),
        "hbpdc_node_coords": (I, [P, P, P]),
        "hbpdc_node_coords_z": (I, [P, P]),
        "hbpdc_rhs": (I, [P, P, P, P]),
        "hbpdc_residual": (I, [P, D, D, D, P, P, P, P, P, ctypes.POINTER(D)]),
        "hbpdc_jvp": (I, [P, D, D, D, P, P, P, P, P, P, I, P]),
        "hbpdc_precond_build": (I, [P, D, D, D, P]),
        "hbpdc_precond_set": (I, [P, D, D, D, P, P, I]),
        "hbpdc_precond_export": (I, [P, P, ctypes.c_size_t, ctypes.POINTER(I)]),
        "hbpdc_precond_apply": (I, [P, P, P, P, P]),
        "hbpdc_step": (I, [P, D, P, ctypes.POINTER(StepStats)]),
        "hbpdc_step_host": (I, [P, D, P, ctypes.POINTER(StepStats)]),
        "hbpdc_reset": (I, [P]),
        "hbpdc_profile": (I, [P, I]),
        "hbpdc_profile_read": (I, [P, I, ctypes.POINTER(ctypes.c_longlong), ctypes.POINTER(D),
                                   ctypes.POINTER(D)]),
        "hbpdc_launch_count": (I, [ctypes.POINTER(ctypes.c_longlong)]),
        "hbpdc_last_error": (ctypes.c_char_p, [P]),
        "hbpdc_finalize": (V, [P]),
        "hbpdc_partition": (I, [I, I, I, I, I, I] + [ctypes.POINTER(ctypes.c_int)] * 5),
        "hbpdc_nccl_unique_id": (I, [P]),
        "hbpdc_loopback_group_create": (I, [I, ctypes.POINTER(P)]),
        "hbpdc_loopback_group_destroy": (V, [P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def partition(dim, nx, ny, px, py, rank):
    """Host-only partition arithmetic of the library: (ex0, ey0, nx_local,
    ny_local, [nbr -x, +x, -y, +y])."""
    v = [ctypes.c_int() for _ in range(4)]
    nb = (ctypes.c_int * 4)()
    st = load().hbpdc_partition(dim, nx, ny, px, py, rank, *[ctypes.byref(x) for x in v], nb)
    if st != 0:
        raise HbpdcError(st, "invalid partition")
    return tuple(x.value for x in v) + (list(nb),)


def nccl_unique_id():
    """128-byte NCCL unique id (rank 0 creates it, torch.distributed distributes it)."""
    buf = ctypes.create_string_buffer(128)
    st = load().hbpdc_nccl_unique_id(buf)
    if st != 0:
        raise HbpdcError(st, "ncclGetUniqueId failed")
    return buf.raw


class LoopbackGroup:
    """Ranks living as host threads of this process (COMM_LOOPBACK)."""

    def __init__(self, nranks):
        self.h = ctypes.c_void_p()
        st = load().hbpdc_loopback_group_create(nranks, ctypes.byref(self.h))
        if st != 0:
            raise HbpdcError(st, "loopback group")

    def close(self):
        if self.h and self.h.value:
            load().hbpdc_loopback_group_destroy(self.h)
            self.h = ctypes.c_void_p()


def launch_count():
    """Kernels launched by the library in this process so far."""
    n = ctypes.c_longlong()
    load().hbpdc_launch_count(ctypes.byref(n))
    return n.value


class HbpdcError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"hbpdc {STATUS.get(status, status)}: {msg}")
        self.status = status


def _ptr(t, n=None):
    """Device pointer of a contiguous float64 CUDA tensor holding at least n doubles."""
    if t is None:
        return None
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous():
        raise TypeError("expected a contiguous float64 CUDA tensor")
    if n is not None and t.numel() < n:
        raise ValueError(f"tensor holds {t.numel()} doubles, the call needs {n}")
    return ctypes.c_void_p(t.data_ptr())


class Context:
    """One rank's view of an HBPC/DGSEM problem (hbpdc_ctx)."""

    def __init__(self, *, dim, equation, N, nx, ny=1, bounds=(0.0, 1.0, 0.0, 1.0), a=(1.0, 1.0),
                 gamma=1.4, mu=0.0, prandtl=0.72, q=4, kmax=0, newton_rtol=1e-10,
                 newton_atol_dw=1e-12, newton_floor=64.0, newton_max=50, gmres_rtol=1e-6,
                 restart=700, max_krylov=7000, precond="bjext", precond_policy="per_step_per_alpha",
                 jvp_mode="auto", batch_stages=True, gmres_sstep=1, rank=0, nranks=1, px=1, py=1, nccl_id=None, stream=None, device=0,
                 comm="auto", loopback=None, force_halo=False, flux="llf", mach=1.0, schur=False,
                 nodes="gll", lifting="br1", eta_br2=2.0, nz=1):
        import torch
        self.lib = load()
        if not torch.cuda.is_available():
            raise RuntimeError("hbpdc needs a CUDA device (no CPU fallback)")
        pb = Problem(dim=dim, equation=_EQ[equation], gamma=gamma, mach_eps=mach, mu=mu, prandtl=prandtl,
                     N=N, nodes={"gll": GLL, "gl": GL}[nodes], nx=nx, ny=ny, xmin=bounds[0], xmax=bounds[1], ymin=bounds[2],
                     ymax=bounds[3], flux={"llf": 0, "glf": 1}[flux], lifting={"br1": 0, "br2": 1}[lifting],
                     q=q, kmax=kmax, eta_br2=eta_br2, nz=nz,
                     zmin=bounds[4] if len(bounds) > 4 else 0.0, zmax=bounds[5] if len(bounds) > 5 else 1.0,
                     az=a[2] if len(a) > 2 else 0.0)
        pb.a[0], pb.a[1] = a[0], a[1]
        op = SolverOpts(newton_rtol=newton_rtol, newton_atol_dw=newton_atol_dw, newton_floor=newton_floor,
                        newton_max=newton_max, gmres_rtol=gmres_rtol, gmres_restart=restart,
                        krylov_max_per_newton=max_krylov, precond=_PC[precond],
                        precond_policy=0 if precond_policy == "per_step_per_alpha" else 1,
                        jvp_mode=_JVP[jvp_mode], batch_stages=int(batch_stages),
                        gmres_sstep=int(gmres_sstep), schur=int(schur))
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.stream = stream
        self._nccl_id = nccl_id
        ds = Dist(rank=rank, nranks=nranks, px=px, py=py,
                  nccl_unique_id=ctypes.cast(ctypes.c_char_p(nccl_id), ctypes.c_void_p) if nccl_id else None,
                  cuda_stream=ctypes.c_void_p(stream.cuda_stream), device=device, own_stream=0,
                  comm=_COMM[comm], loopback_group=loopback.h if loopback is not None else None,
                  force_halo=int(force_halo))
        self._ds = ds
        h = ctypes.c_void_p()
        st = self.lib.hbpdc_init(ctypes.byref(pb), ctypes.byref(op), ctypes.byref(ds), ctypes.byref(h))
        self.h = h
        if st != 0:
            msg = self.lib.hbpdc_last_error(h).decode() if h.value else "init failed"
            if h.value:
                self.lib.hbpdc_finalize(h)
                self.h = ctypes.c_void_p()
            raise HbpdcError(st, msg)
        vals = [ctypes.c_int() for _ in range(6)]
        self._check(self.lib.hbpdc_local_shape(self.h, *[ctypes.byref(v) for v in vals]))
        self.n_elem, self.m, self.ex0, self.ey0, self.nx_local, self.ny_local = [v.value for v in vals]
        self.n = self.n_elem * self.m
        self.dim, self.N = dim, N
        self.nz_local = nz if dim == 3 else 1
        self.device = device
        self.rank, self.nranks, self.px, self.py = rank, nranks, px, py

    # -- helpers ---------------------------------------------------------------------
    def _check(self, st):
        if st != 0:
            raise HbpdcError(st, self.lib.hbpdc_last_error(self.h).decode())

    def empty(self, n=None):
        import torch
        return torch.empty(self.n if n is None else n, dtype=torch.float64, device=f"cuda:{self.device}")

    def node_coords(self):
        nodes = (self.N + 1) ** self.dim
        x = np.zeros(self.n_elem * nodes)
        y = np.zeros(self.n_elem * nodes)
        self._check(self.lib.hbpdc_node_coords(self.h, x.ctypes.data_as(ctypes.c_void_p),
                                               y.ctypes.data_as(ctypes.c_void_p)))
        p = self.N + 1
        if self.dim == 1:
            return (x.reshape(self.nx_local, p),)
        if self.dim == 3:
            z = np.zeros(self.n_elem * nodes)
            self._check(self.lib.hbpdc_node_coords_z(self.h, z.ctypes.data_as(ctypes.c_void_p)))
            sh = (self.nz_local, self.ny_local, self.nx_local, p, p, p)
            return (x.reshape(sh), y.reshape(sh), z.reshape(sh))
        sh = (self.ny_local, self.nx_local, p, p)
        return (x.reshape(sh), y.reshape(sh))

    # -- operators -------------------------------------------------------------------
    def rhs(self, W, sigma=None, out=None):
        out = self.empty() if out is None else out
        self._check(self.lib.hbpdc_rhs(self.h, _ptr(W, self.n), _ptr(sigma, self.n), _ptr(out, self.n)))
        return out

    def residual(self, a1, a2, dt, b, W, sigma, G1=None, G2=None, norm=False):
        G1 = self.empty() if G1 is None else G1
        G2 = self.empty() if G2 is None else G2
        nrm = ctypes.c_double()
        self._check(self.lib.hbpdc_residual(self.h, a1, a2, dt, _ptr(b, self.n), _ptr(W, self.n), _ptr(sigma, self.n), _ptr(G1, self.n),
                                            _ptr(G2, self.n), ctypes.byref(nrm) if norm else None))
        return (G1, G2, nrm.value) if norm else (G1, G2)

    def jvp(self, a1, a2, dt, W, sigma, dW, dsigma, mode="auto", eps_override=None, out1=None, out2=None):
        out1 = self.empty() if out1 is None else out1
        out2 = self.empty() if out2 is None else out2
        eo = None
        if eps_override is not None:
            arr = (ctypes.c_double * 2)(*[(-1.0 if e is None else e) for e in eps_override])
            eo = ctypes.cast(arr, ctypes.c_void_p)
        self._check(self.lib.hbpdc_jvp(self.h, a1, a2, dt, _ptr(W, self.n), _ptr(sigma, self.n), _ptr(dW, self.n), _ptr(dsigma, self.n),
                                       _ptr(out1, self.n), _ptr(out2, self.n), _JVP[mode], eo))
        return out1, out2

    def precond_build(self, a1, a2, dt, W):
        self._check(self.lib.hbpdc_precond_build(self.h, a1, a2, dt, _ptr(W, self.n)))

    def precond_set(self, a1, a2, dt, W, S, shared):
        self._check(self.lib.hbpdc_precond_set(self.h, a1, a2, dt, _ptr(W, self.n),
                                               _ptr(S, self.m * self.m * (1 if shared else self.n_elem)), int(shared)))

    def precond_export(self, shared_hint=None):
        """(S blocks as a device tensor, shared flag); the size comes from the library
        (shared_hint is accepted for compatibility and ignored)."""
        import torch
        flag = ctypes.c_int()
        self._check(self.lib.hbpdc_precond_export(self.h, None, 0, ctypes.byref(flag)))
        nblk = 1 if flag.value else self.n_elem
        S = torch.empty(nblk * self.m * self.m, dtype=torch.float64, device=f"cuda:{self.device}")
        self._check(self.lib.hbpdc_precond_export(self.h, _ptr(S), S.numel(), ctypes.byref(flag)))
        return S, bool(flag.value)

    def precond_apply(self, inW, insig, outW=None, outsig=None):
        outW = self.empty() if outW is None else outW
        outsig = self.empty() if outsig is None else outsig
        self._check(self.lib.hbpdc_precond_apply(self.h, _ptr(inW, self.n), _ptr(insig, self.n), _ptr(outW, self.n), _ptr(outsig, self.n)))
        return outW, outsig

    def step(self, dt, W):
        st = StepStats()
        self._check(self.lib.hbpdc_step(self.h, dt, _ptr(W, self.n), ctypes.byref(st)))
        return st.as_dict()

    def step_host(self, dt, W_host):
        """W_host: a C-contiguous float64 numpy array or pinned CPU torch tensor."""
        st = StepStats()
        if isinstance(W_host, np.ndarray):
            if W_host.dtype != np.float64 or not W_host.flags.c_contiguous or W_host.size < self.n:
                raise ValueError("step_host: expected a C-contiguous float64 array of n doubles")
            p = W_host.ctypes.data_as(ctypes.c_void_p)
        else:
            if W_host.numel() < self.n:
                raise ValueError("step_host: host tensor too small")
            p = ctypes.c_void_p(W_host.data_ptr())
        self._check(self.lib.hbpdc_step_host(self.h, dt, p, ctypes.byref(st)))
        return st.as_dict()

    def reset(self):
        self._check(self.lib.hbpdc_reset(self.h))

    def profile(self, enable):
        self._check(self.lib.hbpdc_profile(self.h, int(enable)))

    PROFILE_IDS = {"gemv": 0, "jvp": 1, "residual": 2, "arnoldi_dots": 3, "arnoldi_update": 4,
                   "kapply": 5, "build": 6, "arnoldi_fused": 7}

    def profile_read(self, kernel_id):
        """(launches, total_ms, algorithmic_bytes) of a profiled kernel id."""
        n = ctypes.c_longlong()
        ms = ctypes.c_double()
        by = ctypes.c_double()
        self._check(self.lib.hbpdc_profile_read(self.h, kernel_id, ctypes.byref(n), ctypes.byref(ms),
                                                ctypes.byref(by)))
        return n.value, ms.value, by.value

    def close(self):
        if self.h and self.h.value:
            self.lib.hbpdc_finalize(self.h)
            self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def context_for(cfg, **overrides):
    """Context for a configs.Config (BASELINE.json config restated)."""
    kw = dict(dim=cfg.dim, equation=cfg.equation, N=cfg.N, nx=cfg.nx, ny=cfg.ny, bounds=cfg.bounds,
              a=cfg.a, gamma=cfg.gamma, mu=cfg.mu, prandtl=cfg.prandtl, q=cfg.q, kmax=cfg.kmax,
              newton_rtol=cfg.newton_rtol, newton_atol_dw=cfg.newton_atol_dw, gmres_rtol=cfg.gmres_rtol,
              restart=cfg.restart, max_krylov=cfg.max_krylov, precond=cfg.precond)
    if cfg.dim == 3:
        kw["nz"] = cfg.nz
    kw.update(overrides)
    return Context(**kw)
