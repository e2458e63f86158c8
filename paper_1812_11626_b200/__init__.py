"""B200-native SU(N) unfold of the GKSL master equation (arXiv:1812.11626).

Thin Python binding of the C-ABI in include/sunfold.h (argument marshalling only; every
step of the path runs in the sm_100a kernels of libsunfold.so).  PyTorch provides device
memory and streams.  There is no CPU fallback: if the CUDA library cannot be loaded the
import of the ops raises.

    plan = Plan(H0, H1, Ls, gammas)      # sun_plan_create (validation + pattern analysis)
    Q0, Q1, K = plan.run()               # sun_run (count+scan+fill) -> sun_plan_nnz
    Q0, Q1, K = plan.run_two_pass()      # sun_count -> sun_plan_nnz -> sun_unfold
    dvdt = apply(Q0, Q1, eps, K, v)      # sun_apply

Operators are `DeviceZCSR` (torch CUDA tensors) or any object with `n, row_ptr, col, val`
host arrays (e.g. workloads.ZCSR), which are copied to the device.
Outputs are `CSR(row_ptr int64[M+1], col int32[nnz], val float64[nnz])` CUDA tensors and
K float64[M].  Generator order and the stored-pattern rule are those of include/sunfold.h.
"""
from __future__ import annotations

import ctypes
import contextlib
from typing import NamedTuple, Optional, Sequence

import numpy as np
import torch

from . import _lib

__all__ = ["CSR", "DeviceZCSR", "Plan", "unfold", "unfold_split", "apply", "rk4", "expand_state", "state_diag",
           "gen_index", "lib", "SunError"]


class SunError(RuntimeError):
    pass


class CSR(NamedTuple):
    row_ptr: torch.Tensor  # int64 [m+1]
    col: torch.Tensor  # int32 [nnz]
    val: torch.Tensor  # float64 [nnz]

    @property
    def m(self) -> int:
        return int(self.row_ptr.shape[0] - 1)

    @property
    def nnz(self) -> int:
        return int(self.col.shape[0])

    def to_torch(self) -> torch.Tensor:
        """A torch.sparse_csr_tensor of this matrix (column indices widened to int64: a copy)."""
        return torch.sparse_csr_tensor(self.row_ptr, self.col.to(torch.int64), self.val, size=(self.m, self.m),
                                       check_invariants=False)


class DeviceZCSR(NamedTuple):
    n: int
    row_ptr: torch.Tensor  # int64 [n+1] cuda
    col: torch.Tensor  # int32 [nnz] cuda
    val: torch.Tensor  # complex128 [nnz] cuda

    @staticmethod
    def from_host(A, device="cuda", non_blocking: bool = False) -> "DeviceZCSR":
        def t(x, dt):
            x = torch.as_tensor(np.ascontiguousarray(x))
            if x.dtype != dt:
                x = x.to(dt)
            return x.to(device, non_blocking=non_blocking)

        return DeviceZCSR(int(A.n), t(A.row_ptr, torch.int64), t(A.col, torch.int32), t(A.val, torch.complex128))


def lib():
    return _lib.load()


def _check(status: int, what: str):
    if status != 0:
        raise SunError(f"{what}: {lib().sun_status_string(status).decode()} (status {status})")


def _stream_handle(stream) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


@contextlib.contextmanager
def _on(stream):
    """Run a call's marshalling and allocations on `stream`: the stream first waits for the
    caller's current stream (inputs made there are ordered before the kernels), and every
    tensor allocated inside (workspace, outputs, scratch) belongs to `stream`, so the caching
    allocator never hands its memory to another stream while the kernels still use it."""
    if stream is None:
        yield
        return
    cur = torch.cuda.current_stream(stream.device)
    if stream == cur:
        yield
        return
    stream.wait_stream(cur)
    with torch.cuda.stream(stream):
        yield


def _to_device(A) -> DeviceZCSR:
    """Operator marshalling: DeviceZCSR as is; host ZCSR (workloads); a torch sparse-CSR tensor;
    a dense N x N torch tensor or numpy array (its nonzero entries, row-major)."""
    if isinstance(A, DeviceZCSR):
        return A
    if isinstance(A, np.ndarray):
        A = torch.as_tensor(A)
    if isinstance(A, torch.Tensor):
        dev = A.device if A.is_cuda else torch.device("cuda")
        if A.layout == torch.sparse_csr:
            return DeviceZCSR(int(A.shape[0]), A.crow_indices().to(dev, torch.int64),
                              A.col_indices().to(dev, torch.int32), A.values().to(dev, torch.complex128))
        assert A.dim() == 2 and A.shape[0] == A.shape[1], "operators are N x N"
        D = A.to(dev, torch.complex128)
        nzr, nzc = torch.nonzero(D, as_tuple=True)  # row-major order, columns ascending
        counts = torch.bincount(nzr, minlength=D.shape[0])
        rp = torch.zeros(D.shape[0] + 1, dtype=torch.int64, device=dev)
        rp[1:] = torch.cumsum(counts, 0)
        return DeviceZCSR(int(D.shape[0]), rp, nzc.to(torch.int32), D[nzr, nzc].contiguous())
    return DeviceZCSR.from_host(A)


def _zcsr_struct(A: DeviceZCSR) -> _lib.SunZCSR:
    assert A.row_ptr.is_cuda and A.col.is_cuda and A.val.is_cuda
    assert A.row_ptr.dtype == torch.int64 and A.col.dtype == torch.int32 and A.val.dtype == torch.complex128
    return _lib.SunZCSR(int(A.n), int(A.col.shape[0]), A.row_ptr.data_ptr(), A.col.data_ptr(), A.val.data_ptr())


def _dcsr_struct(Q: CSR) -> _lib.SunDCSR:
    return _lib.SunDCSR(Q.m, Q.nnz, Q.row_ptr.data_ptr(), Q.col.data_ptr(), Q.val.data_ptr())


def gen_index(n: int, kind: str, a: int, b: int = -1) -> int:
    """Canonical generator index (R5): kind 'S', 'J' (a < b) or 'D' (a = l)."""
    return int(lib().sun_gen_index(n, {"S": 0, "J": 1, "D": 2}[kind], a, b))


class Plan:
    """A validated, analysed unfold problem bound to a device workspace (sun_plan_create)."""

    def __init__(self, H0, H1=None, Ls: Sequence = (), gammas: Sequence[float] = (), stream=None,
                 guard_bytes: int = 0, general: bool = False, small_cap: bool = False):
        """guard_bytes > 0 (tests): the workspace gets a tail of that many 0xA5 bytes beyond the
        size the library is told; workspace_guard_intact() checks it (out-of-bounds writes).
        general=True: the general-pattern mode even for banded operators (SUN_PLAN_GENERAL);
        operators of any other pattern take it anyway.  small_cap=True (tests): general mode with a
        16-candidate merge buffer (SUN_PLAN_SMALLCAP)."""
        with _on(stream):
            self._init(H0, H1, Ls, gammas, stream, guard_bytes, (1 if general else 0) | (2 if small_cap else 0))

    def _init(self, H0, H1, Ls, gammas, stream, guard_bytes, flags=0):
        L = lib()
        self.stream = stream
        self.H0 = _to_device(H0)
        self.H1 = _to_device(H1) if H1 is not None else None
        self.Ls = [_to_device(x) for x in Ls]
        self.gammas = np.ascontiguousarray(np.asarray(list(gammas), dtype=np.float64))
        if len(self.Ls) != len(self.gammas):
            raise ValueError("len(Ls) != len(gammas)")
        self.n = self.H0.n
        self.m = self.n * self.n - 1
        self.P = len(self.Ls)
        self._s_h0 = _zcsr_struct(self.H0)
        self._s_h1 = _zcsr_struct(self.H1) if self.H1 is not None else None
        self._s_ls = [_zcsr_struct(x) for x in self.Ls]
        arr = (ctypes.c_void_p * max(self.P, 1))()
        for i, s in enumerate(self._s_ls):
            arr[i] = ctypes.addressof(s)
        self._arr = arr
        s_h1 = ctypes.addressof(self._s_h1) if self._s_h1 is not None else None
        s_ls = ctypes.addressof(arr) if self.P else None
        nbytes = int(L.sun_workspace_bytes_ops(ctypes.addressof(self._s_h0), s_h1, s_ls, self.P))
        if nbytes == 0:
            _check(2, "sun_workspace_bytes_ops")
        self.workspace = torch.empty(nbytes + guard_bytes, dtype=torch.uint8, device="cuda")
        self._guard = guard_bytes
        if guard_bytes:
            self.workspace[nbytes:].fill_(0xA5)
        plan = ctypes.c_void_p()
        st = L.sun_plan_create_ex(
            ctypes.addressof(plan), ctypes.addressof(self._s_h0), s_h1, s_ls,
            self.gammas.ctypes.data_as(ctypes.c_void_p) if self.P else None,
            self.P, flags, ctypes.c_void_p(self.workspace.data_ptr()), ctypes.c_size_t(nbytes),
            ctypes.c_void_p(_stream_handle(stream)))
        _check(st, "sun_plan_create")
        self._plan = plan
        self._caps = None  # output capacities for run(): previous nnz
        self._banded = self.info()["mode_q0"] != 3
        self.stash = None
        if not self._banded:
            self.set_stash(True)

    def workspace_guard_intact(self) -> bool:
        if not self._guard:
            return True
        return bool((self.workspace[-self._guard:] == 0xA5).all().item())

    # -- the three phases ----------------------------------------------------------------
    def count(self):
        with _on(self.stream):
            _check(lib().sun_count(self._plan, _stream_handle(self.stream)), "sun_count")

    def nnz(self):
        a, b = ctypes.c_int64(), ctypes.c_int64()
        _check(lib().sun_plan_nnz(self._plan, ctypes.addressof(a), ctypes.addressof(b)), "sun_plan_nnz")
        return int(a.value), int(b.value)

    def _alloc(self, cap0: int, cap1: int):
        """Output buffers of the given capacities (three allocations; Q0/Q1/K are views)."""
        dev = self.workspace.device
        m1 = self.m + 1
        has1 = self.H1 is not None
        rp = torch.empty(2 * m1 if has1 else m1, dtype=torch.int64, device=dev)
        cols = torch.empty(cap0 + cap1, dtype=torch.int32, device=dev)
        vals = torch.empty(cap0 + cap1 + self.m, dtype=torch.float64, device=dev)
        Q0 = CSR(rp[:m1], cols[:cap0], vals[:cap0])
        Q1 = CSR(rp[m1:], cols[cap0:], vals[cap0:cap0 + cap1]) if has1 else None
        K = vals[cap0 + cap1:]
        return Q0, Q1, K

    @staticmethod
    def _trim(bufs, nnz0, nnz1):
        Q0, Q1, K = bufs
        if Q0.col.numel() == nnz0 and (Q1 is None or Q1.col.numel() == nnz1):
            return bufs  # exact capacities: no views to make
        Q0 = CSR(Q0.row_ptr, Q0.col[:nnz0], Q0.val[:nnz0])
        if Q1 is not None:
            Q1 = CSR(Q1.row_ptr, Q1.col[:nnz1], Q1.val[:nnz1])
        return Q0, Q1, K

    @staticmethod
    def _structs(bufs):
        Q0, Q1, _ = bufs
        return _dcsr_struct(Q0), (_dcsr_struct(Q1) if Q1 is not None else None)

    def fill(self, nnz0: int, nnz1: int, out=None):
        """Allocate (unless `out` is given) and fill Q0, Q1 and K (sun_unfold, after count/nnz)."""
        with _on(self.stream):
            bufs = out if out is not None else self._alloc(nnz0, nnz1)
            s0, s1 = self._structs(bufs)
            _check(lib().sun_unfold(self._plan, ctypes.addressof(s0),
                                    ctypes.addressof(s1) if s1 is not None else None,
                                    bufs[2].data_ptr(), _stream_handle(self.stream)), "sun_unfold")
            return self._trim(bufs, nnz0, nnz1)

    def nnz_bound(self):
        b0 = int(lib().sun_nnz_bound(self._plan, 0))
        b1 = int(lib().sun_nnz_bound(self._plan, 1)) if self.H1 is not None else 0
        return b0, b1

    def run(self, out=None):
        """Whole unfold with no host round trip between the passes (sun_run), then the nnz
        readback.  Output capacity: `out`, else the previous call's nnz (the first call of a
        banded plan uses the structural bound sun_nnz_bound -- the returned tensors are views of
        those buffers -- and that of a general-pattern plan the exact two-step path).
        Returns (Q0, Q1 or None, K) trimmed to the produced nnz."""
        with _on(self.stream):
            return self._run(out)

    def _run(self, out):
        L = lib()
        if out is None:
            if self._caps is None:
                if not self._banded:  # first call, general mode: exact sizes from the two-step path
                    res = self.run_two_pass()
                    self._caps = (res[0].nnz, res[1].nnz if res[1] is not None else 0)
                    return res
                bufs = self._alloc(*self.nnz_bound())  # banded: the structural bound, one pass
            else:
                bufs = self._alloc(*self._caps)
        else:
            bufs = out
        s0, s1 = self._structs(bufs)
        _check(L.sun_run(self._plan, ctypes.addressof(s0), ctypes.addressof(s1) if s1 is not None else None,
                         bufs[2].data_ptr(), _stream_handle(self.stream)), "sun_run")
        a, b = ctypes.c_int64(), ctypes.c_int64()
        st = L.sun_plan_nnz(self._plan, ctypes.addressof(a), ctypes.addressof(b))
        nnz0, nnz1 = int(a.value), int(b.value)
        if st == 5:  # SUN_ERR_CAPACITY: new values need more entries; refill with exact sizes
            self._caps = (nnz0, nnz1)
            return self.fill(nnz0, nnz1)
        _check(st, "sun_run/sun_plan_nnz")
        self._caps = (nnz0, nnz1)
        return self._trim(bufs, nnz0, nnz1)

    def run_two_pass(self, out=None):
        """The paper's two-step CRS fill through the C-ABI: sun_count ->
        sun_plan_nnz -> allocate exactly -> sun_unfold."""
        self.count()
        nnz0, nnz1 = self.nnz()
        return self.fill(nnz0, nnz1, out)

    def rk4(self, v: torch.Tensor, h: float, nsteps: int, t0: float = 0.0, eps0: float = 0.0, eps1: float = 0.0,
            omega: float = 1.0, work=None) -> torch.Tensor:
        """Matrix-free RK4 of this plan's system in place on v (sun_rk4_plan; F1): Q0 / Q1 are
        regenerated in every stage instead of read.  Needs a counted plan (after run())."""
        with _on(self.stream):
            return self._rk4(v, h, nsteps, t0, eps0, eps1, omega, work)

    def _rk4(self, v, h, nsteps, t0, eps0, eps1, omega, work):
        L = lib()
        nb = int(L.sun_rk4_plan_work_bytes(self._plan))
        w = work if work is not None else torch.empty((nb + 7) // 8, dtype=torch.float64, device=v.device)
        wb = w.numel() * w.element_size()
        _check(L.sun_rk4_plan(self._plan, ctypes.c_double(eps0), ctypes.c_double(eps1), ctypes.c_double(omega),
                              ctypes.c_double(t0), ctypes.c_double(h), ctypes.c_int64(nsteps),
                              ctypes.c_void_p(v.data_ptr()), ctypes.c_void_p(w.data_ptr()), ctypes.c_size_t(wb),
                              ctypes.c_void_p(_stream_handle(self.stream))), "sun_rk4_plan")
        return v

    def apply(self, v: torch.Tensor, eps: float = 0.0, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """dv/dt = (Q0 + eps Q1) v + K without reading Q (sun_apply_plan); needs a counted plan."""
        with _on(self.stream):
            y = out if out is not None else torch.empty_like(v)
            w = torch.empty(self.n, dtype=torch.float64, device=v.device)
            self._apply(v, eps, y, w)
            return y

    def _apply(self, v, eps, y, w):
        _check(lib().sun_apply_plan(self._plan, ctypes.c_double(eps), ctypes.c_void_p(v.data_ptr()),
                                    ctypes.c_void_p(y.data_ptr()), ctypes.c_void_p(w.data_ptr()),
                                    ctypes.c_size_t(w.numel() * 8), ctypes.c_void_p(_stream_handle(self.stream))),
               "sun_apply_plan")

    def launches_per_run(self) -> int:
        """Kernels of this library launched by one run() (sun_run: count + fill)."""
        inf = self.info()
        return int(inf["launches_count"] + inf["launches_fill"])

    #: largest light-row stash set_stash(True) allocates (and at most a quarter of free memory)
    STASH_MAX_BYTES = 8 << 30

    def set_stash(self, enable: bool) -> bool:
        """General-pattern plans: a device buffer in which the count pass keeps the assembled light
        rows, so the fill copies them (sun_plan_set_stash; bit-identical output).  Enabled at plan
        creation when it fits STASH_MAX_BYTES and a quarter of the free device memory.  Returns
        whether a stash is set.  A new count pass is needed before the next fill."""
        L = lib()
        nb = int(L.sun_plan_stash_bytes(self._plan))
        buf = None
        if enable and nb > 0:
            free = torch.cuda.mem_get_info()[0]
            if nb <= min(self.STASH_MAX_BYTES, free // 4):
                with _on(self.stream):
                    buf = torch.empty(nb, dtype=torch.uint8, device="cuda")
        _check(L.sun_plan_set_stash(self._plan, ctypes.c_void_p(buf.data_ptr() if buf is not None else 0),
                                    ctypes.c_size_t(nb if buf is not None else 0)), "sun_plan_set_stash")
        self.stash = buf
        return buf is not None

    def set_graphs(self, enable: bool):
        """CUDA-graph replay of the enqueue sequences on (default) or off (sun_plan_set_graphs)."""
        _check(lib().sun_plan_set_graphs(self._plan, 1 if enable else 0), "sun_plan_set_graphs")

    def set_timing(self, enable: bool):
        """Phase timing on/off (sun_plan_set_timing): event records around the count and fill
        passes inside each sequence (graph event-record nodes)."""
        _check(lib().sun_plan_set_timing(self._plan, 1 if enable else 0), "sun_plan_set_timing")

    def phase_ms(self):
        """(count_ms, fill_ms) device time of the last timed sequence (sun_plan_phase_ms; -1 for
        a phase it did not run).  Waits for that sequence."""
        c, f = ctypes.c_float(), ctypes.c_float()
        _check(lib().sun_plan_phase_ms(self._plan, ctypes.addressof(c), ctypes.addressof(f)), "sun_plan_phase_ms")
        return float(c.value), float(f.value)

    def info(self) -> dict:
        inf = _lib.SunPlanInfo()
        _check(lib().sun_plan_info(self._plan, ctypes.addressof(inf)), "sun_plan_info")
        return {f: getattr(inf, f) for f, _ in _lib.SunPlanInfo._fields_}

    def close(self):
        if getattr(self, "_plan", None):
            lib().sun_plan_destroy(self._plan)
            self._plan = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def unfold(H0, H1=None, Ls: Sequence = (), gammas: Sequence[float] = (), stream=None):
    """expand(H, {L_p, gamma_p}) -> (Q0 CSR, Q1 CSR or None, K), all on the GPU.  With `stream`,
    the work (and every allocation) is on that stream, after the caller's current stream; the
    outputs belong to `stream` (synchronise with it before using them elsewhere)."""
    with _on(stream):
        plan = Plan(H0, H1, Ls, gammas, stream)
        try:
            return plan.run()
        finally:
            plan.close()


def unfold_split(H0, H1=None, Ls: Sequence = (), gammas: Sequence[float] = (), stream=None):
    """The paper's split (Eq. 9): dv/dt = [Q(t) + R] v + K with Q = Q_H[H0] (Eq. 6)
    and R, K from the dissipators (Eqs. 10-11), as separate CSR matrices.
    Two unfolds through the same C-ABI: (H0, no dissipators) and (0, {L_p, gamma_p}); a trace of
    L_p contributes its unitary part to R (reading R3).  Returns (QH, R, Q1 or None, K)."""
    with _on(stream):
        return _unfold_split(H0, H1, Ls, gammas, stream)


def _unfold_split(H0, H1, Ls, gammas, stream):
    H0d = _to_device(H0)
    zero = DeviceZCSR(H0d.n, torch.zeros(H0d.n + 1, dtype=torch.int64, device=H0d.row_ptr.device),
                      torch.zeros(0, dtype=torch.int32, device=H0d.row_ptr.device),
                      torch.zeros(0, dtype=torch.complex128, device=H0d.row_ptr.device))
    QH, Q1, _ = unfold(H0d, H1, (), (), stream)
    if len(Ls):
        R, _, K = unfold(zero, None, Ls, gammas, stream)
    else:
        R, _, K = unfold(zero, None, (), (), stream)
    return QH, R, Q1, K


def expand_state(rho, stream=None) -> torch.Tensor:
    """v = Re Tr(F_s rho) (Eq. 5; sun_expand_state).  rho: DeviceZCSR or host CSR object."""
    with _on(stream):
        R = _to_device(rho)
        s = _zcsr_struct(R)
        v = torch.empty(R.n * R.n - 1, dtype=torch.float64, device=R.row_ptr.device)
        _check(lib().sun_expand_state(ctypes.addressof(s), ctypes.c_void_p(v.data_ptr()),
                                      ctypes.c_void_p(_stream_handle(stream))), "sun_expand_state")
        return v


def state_diag(v: torch.Tensor, n: int, stream=None) -> torch.Tensor:
    """Populations <a|rho|a> of the state with coherence vector v (sun_state_diag)."""
    assert v.is_cuda and v.dtype == torch.float64 and v.shape[0] == n * n - 1
    with _on(stream):
        d = torch.empty(n, dtype=torch.float64, device=v.device)
        _check(lib().sun_state_diag(ctypes.c_void_p(v.data_ptr()), n, ctypes.c_void_p(d.data_ptr()),
                                    ctypes.c_void_p(_stream_handle(stream))), "sun_state_diag")
        return d


def rk4(Q0: CSR, Q1: Optional[CSR], K: Optional[torch.Tensor], v: torch.Tensor, h: float, nsteps: int,
        t0: float = 0.0, eps0: float = 0.0, eps1: float = 0.0, omega: float = 1.0, work=None,
        stream=None) -> torch.Tensor:
    """Fixed-step RK4 of dv/dt = (Q0 + eps(t) Q1) v + K in place on v (sun_rk4, Step 3.1)."""
    assert v.is_cuda and v.dtype == torch.float64 and v.shape[0] == Q0.m
    with _on(stream):
        return _rk4_csr(Q0, Q1, K, v, h, nsteps, t0, eps0, eps1, omega, work, stream)


def _rk4_csr(Q0, Q1, K, v, h, nsteps, t0, eps0, eps1, omega, work, stream):
    nb = int(lib().sun_rk4_work_bytes(Q0.m))
    w = work if work is not None else torch.empty((nb + 7) // 8, dtype=torch.float64, device=v.device)
    assert w.numel() * w.element_size() >= nb
    s0 = _dcsr_struct(Q0)
    s1 = _dcsr_struct(Q1) if Q1 is not None else None
    _check(lib().sun_rk4(ctypes.addressof(s0), ctypes.addressof(s1) if s1 is not None else None,
                         ctypes.c_void_p(K.data_ptr()) if K is not None else None, ctypes.c_double(eps0),
                         ctypes.c_double(eps1), ctypes.c_double(omega), ctypes.c_double(t0), ctypes.c_double(h),
                         ctypes.c_int64(nsteps), ctypes.c_void_p(v.data_ptr()), ctypes.c_void_p(w.data_ptr()),
                         ctypes.c_void_p(_stream_handle(stream))), "sun_rk4")
    return v


def state_reconstruct(v: torch.Tensor, n: int, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """rho = I/N + sum_j v_j F_j as a dense complex128 N x N tensor (Step 3.2; sun_state_reconstruct)."""
    assert v.is_cuda and v.dtype == torch.float64 and v.numel() == n * n - 1
    with _on(stream):
        rho = out if out is not None else torch.empty((n, n), dtype=torch.complex128, device=v.device)
        assert rho.dtype == torch.complex128 and rho.is_contiguous() and rho.numel() == n * n
        _check(lib().sun_state_reconstruct(ctypes.c_void_p(v.data_ptr()), n, ctypes.c_void_p(rho.data_ptr()),
                                           ctypes.c_void_p(_stream_handle(stream))), "sun_state_reconstruct")
        return rho


def structure_constants(n: int, which: str = "f", count_only: bool = False, stream=None):
    """Nonzero f_mns ('f') or d_mns ('d') of SU(N), every ordered triple, generated on the GPU from
    index arithmetic (sun_structure_constants; Step 2.2).  Returns (idx int32 (nnz, 3),
    val float64 (nnz,)) on the device, or the count only."""
    with _on(stream):
        return _structure_constants(n, which, count_only, stream)


def _structure_constants(n, which, count_only, stream):
    w = {"f": 0, "d": 1}[which]
    dev = torch.device("cuda")
    nb = int(lib().sun_sc_work_bytes(n))
    if nb == 0:
        raise SunError(f"sun_sc_work_bytes: N = {n} out of range")
    work = torch.empty((nb + 7) // 8, dtype=torch.int64, device=dev)
    cnt = ctypes.c_int64()
    h = ctypes.c_void_p(_stream_handle(stream))
    _check(lib().sun_structure_constants(n, w, None, None, 0, ctypes.addressof(cnt), ctypes.c_void_p(work.data_ptr()),
                                         nb, h), "sun_structure_constants")
    if count_only:
        return int(cnt.value)
    nnz = int(cnt.value)
    idx = torch.empty((max(nnz, 1), 3), dtype=torch.int32, device=dev)
    val = torch.empty(max(nnz, 1), dtype=torch.float64, device=dev)
    _check(lib().sun_structure_constants(n, w, ctypes.c_void_p(idx.data_ptr()), ctypes.c_void_p(val.data_ptr()), nnz,
                                         ctypes.addressof(cnt), ctypes.c_void_p(work.data_ptr()), nb, h),
           "sun_structure_constants")
    return idx[:nnz], val[:nnz]


def dense_work_bytes(n: int, chunk: int = 1) -> int:
    """Scratch bytes of unfold_dense for `chunk` realisations at once (sun_dense_work_bytes)."""
    return int(lib().sun_dense_work_bytes(n, chunk))


def unfold_dense(H: torch.Tensor, A: Optional[torch.Tensor] = None, Q: Optional[torch.Tensor] = None,
                 K: Optional[torch.Tensor] = None, work: Optional[torch.Tensor] = None, chunk: int = 1,
                 stream=None):
    """Dense unfold of L = -i[H, .] + L_D[A] (Eq. 7) for a batch of realisations
    (sun_unfold_dense).

    H: complex128 (B, N, N) or (N, N) on the GPU; A: complex128 (B, M, M) / (M, M) rate
    matrix over the basis (generator order R5), or None.  Returns (Q (B, M, M) float64,
    K (B, M) float64), squeezed like H.  `work` (any dtype, >= dense_work_bytes(N, 1)
    bytes) may be passed to reuse scratch; else `chunk` realisations' worth is allocated.
    """
    with _on(stream):
        return _unfold_dense(H, A, Q, K, work, chunk, stream)


def _unfold_dense(H, A, Q, K, work, chunk, stream):
    squeeze = H.dim() == 2
    Hb = H.unsqueeze(0) if squeeze else H
    assert Hb.is_cuda and Hb.dtype == torch.complex128 and Hb.dim() == 3 and Hb.shape[1] == Hb.shape[2]
    B, n = int(Hb.shape[0]), int(Hb.shape[1])
    m = n * n - 1
    Hb = Hb.contiguous()
    Ab = None
    if A is not None:
        Ab = (A.unsqueeze(0) if A.dim() == 2 else A).contiguous()
        assert Ab.dtype == torch.complex128 and tuple(Ab.shape) == (B, m, m) and Ab.device == Hb.device
    if Q is None:
        Q = torch.empty((B, m, m), dtype=torch.float64, device=Hb.device)
    if K is None:
        K = torch.empty((B, m), dtype=torch.float64, device=Hb.device)
    assert Q.is_contiguous() and Q.numel() == B * m * m and K.is_contiguous() and K.numel() == B * m
    if work is None:
        nb = dense_work_bytes(n, max(1, min(chunk, B)))
        if nb == 0:
            raise SunError(f"sun_dense_work_bytes: N = {n} out of range")
        work = torch.empty((nb + 15) // 16, dtype=torch.complex128, device=Hb.device)
    wb = work.numel() * work.element_size()
    _check(lib().sun_unfold_dense(n, B, ctypes.c_void_p(Hb.data_ptr()),
                                  ctypes.c_void_p(Ab.data_ptr()) if Ab is not None else None,
                                  ctypes.c_void_p(Q.data_ptr()), ctypes.c_void_p(K.data_ptr()),
                                  ctypes.c_void_p(work.data_ptr()), ctypes.c_size_t(wb),
                                  ctypes.c_void_p(_stream_handle(stream))), "sun_unfold_dense")
    if squeeze:
        return Q.view(m, m), K.view(m)
    return Q.view(B, m, m), K.view(B, m)


def apply(Q0: CSR, Q1: Optional[CSR], eps: float, K: Optional[torch.Tensor], v: torch.Tensor,
          out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """dv/dt = Q0 v + eps Q1 v + K (Eq. 9) via sun_apply."""
    assert v.is_cuda and v.dtype == torch.float64 and v.shape[0] == Q0.m
    with _on(stream):
        y = out if out is not None else torch.empty_like(v)
        _apply_csr(Q0, Q1, eps, K, v, y, stream)
        return y


def _apply_csr(Q0, Q1, eps, K, v, y, stream):
    s0 = _dcsr_struct(Q0)
    s1 = _dcsr_struct(Q1) if Q1 is not None else None
    _check(lib().sun_apply(ctypes.addressof(s0), ctypes.addressof(s1) if s1 is not None else None, ctypes.c_double(eps),
                           ctypes.c_void_p(K.data_ptr()) if K is not None else None,
                           ctypes.c_void_p(v.data_ptr()), ctypes.c_void_p(y.data_ptr()),
                           ctypes.c_void_p(_stream_handle(stream))), "sun_apply")
