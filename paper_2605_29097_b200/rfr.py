"""Thin ctypes binding of librfr (include/librfr.h): argument marshalling only.

Every step of the renderer runs in librfr's sm_100a kernels; this module only turns torch CUDA
tensors into the C structs of the ABI and checks the returned status.  PyTorch supplies device
memory and the current stream.  There is no CPU fallback: if librfr.so is missing or no CUDA device
is present, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from typing import Optional

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librfr.so")

RFR_NO_GAIN = 1
RFR_CHECK_FINITE = 2
RFR_REUSE_BLEND = 4
RFR_DIRECT = 8          # direct kernels instead of the Chebyshev-moment path (A/B)
RFR_R1 = 16             # the r1 kernels instead of the r2 tiled engine (A/B)
RFR_FLAG_DOMAIN = 1
RFR_FLAG_NUMERIC = 2

_P = C.POINTER(C.c_float)


class rfr_freq_grid(C.Structure):
    _fields_ = [("f0_hz", C.c_double), ("df_hz", C.c_double), ("n_freq", C.c_int32)]


class rfr_samples(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in
                ("x", "y", "z", "sdf", "refl", "nx", "ny", "nz", "power", "phi_origin")] + \
               [("n_rays", C.c_int64), ("n_per_ray", C.c_int32)]


class rfr_antennas(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in
                ("tx_x", "tx_y", "tx_z", "rx_x", "rx_y", "rx_z", "phi_tx", "phi_rx")] + \
               [("n_ant", C.c_int64)]


class rfr_sample_grads(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("sdf", "refl", "nx", "ny", "nz", "power", "sharpness")]


class rfr_opts(C.Structure):
    _fields_ = [("flags", C.c_uint32)]


class rfr_workspace(C.Structure):
    _fields_ = [("ptr", C.c_void_p), ("bytes", C.c_size_t), ("n_samples", C.c_int64),
                ("n_ant", C.c_int64), ("n_freq", C.c_int32), ("n_query", C.c_int64)]


class rfr_plan_info(C.Structure):
    _fields_ = [("applied", C.c_int32), ("tiles", C.c_int32), ("lx", C.c_int32), ("ly", C.c_int32),
                ("lz", C.c_int32), ("P", C.c_int32), ("Pg", C.c_int32), ("n_points", C.c_int32),
                ("delta_t", C.c_double), ("delta_g", C.c_double)]


SWEEPS = {"plan": 0, "sort": 1, "prep": 2, "filter": 3, "backward": 4, "forward": 5,
          "forward_out": 6}

STATUS = {0: "ok", 1: "invalid argument", 2: "shape mismatch or workspace too small",
          3: "domain", 4: "numeric", 5: "CUDA launch failure", 6: "unsupported", 7: "NCCL failure"}

EXPORTS = ("rfr_workspace_size", "rfr_forward", "rfr_loss", "rfr_filter", "rfr_filter_partial",
           "rfr_filter_power", "rfr_backward", "rfr_backward_partial", "rfr_backward_finish",
           "rfr_backward_filter", "rfr_backward_filter_partial", "rfr_filter_backward", "rfr_heatmap_loss",
           "rfr_comm_unique_id", "rfr_comm_init", "rfr_comm_destroy",
           "rfr_poll_flags", "rfr_status_string", "rfr_abi_version", "rfr_launch_count",
           "rfr_plan_state", "rfr_profile_enable", "rfr_profile_read", "rfr_filter_gather")


class RfrError(RuntimeError):
    pass


_lib = None


def load(path: str = LIB_PATH):
    """Load librfr.so (built in-tree by __graft_entry__.build()).  Raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"librfr.so not built at {path}: run __graft_entry__.build()")
    lib = C.CDLL(path)
    vp, i64, i32, u32, f = C.c_void_p, C.c_int64, C.c_int32, C.c_uint32, C.c_float
    S, A, G, O, R = (C.POINTER(rfr_samples), C.POINTER(rfr_antennas), C.POINTER(rfr_freq_grid),
                     C.POINTER(rfr_opts), C.POINTER(rfr_sample_grads))
    W = C.POINTER(rfr_workspace)
    sig = {
        "rfr_workspace_size": [i64, i64, i32, i64, C.POINTER(C.c_size_t)],
        "rfr_forward": [S, f, A, G, O, vp, W, vp],
        "rfr_loss": [vp, vp, i64, vp, vp, W, vp],
        "rfr_filter": [vp, A, G, vp, vp, vp, i64, vp, vp, vp, W, vp],
        "rfr_filter_partial": [vp, A, G, vp, vp, vp, i64, vp, W, vp],
        "rfr_filter_power": [vp, i64, vp, vp],
        "rfr_backward": [vp, S, f, A, G, O, R, vp, W, vp],
        "rfr_backward_partial": [vp, S, f, A, G, O, vp, W, vp],
        "rfr_backward_finish": [vp, S, f, O, R, W, vp],
        "rfr_backward_filter": [vp, vp, S, f, A, G, O, R, vp, vp, vp, W, vp],
        "rfr_backward_filter_partial": [vp, vp, S, f, A, G, O, vp, vp, W, vp],
        "rfr_filter_backward": [vp, vp, vp, f, A, G, vp, vp, vp, i64, vp, W, vp],
        "rfr_heatmap_loss": [vp, vp, i64, vp, vp, f, f, vp, vp, vp, W, vp],
        "rfr_poll_flags": [W, C.POINTER(u32), C.c_void_p],
        "rfr_plan_state": [W, C.POINTER(rfr_plan_info), C.c_void_p],
        "rfr_filter_gather": [vp, A, i64, G, vp, vp, vp, i64, vp, vp, vp, W, vp],
        "rfr_profile_enable": [C.c_int],
        "rfr_profile_read": [C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_uint64)],
        "rfr_comm_unique_id": [vp],
        "rfr_comm_init": [vp, C.c_int, C.c_int, C.POINTER(vp)],
        "rfr_comm_destroy": [vp],
    }
    for name, args in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int
    lib.rfr_status_string.argtypes = [C.c_int]
    lib.rfr_status_string.restype = C.c_char_p
    lib.rfr_abi_version.restype = C.c_int
    lib.rfr_launch_count.restype = C.c_uint64
    _lib = lib
    return lib


def _check(rc: int, what: str):
    if rc != 0:
        raise RfrError(f"{what}: {STATUS.get(rc, rc)}")


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    if not t.is_cuda:
        raise RfrError("librfr takes CUDA tensors only (no CPU fallback)")
    if not t.is_contiguous():
        raise RfrError("tensor must be contiguous")
    return t.data_ptr()


def _stream(stream: Optional[torch.cuda.Stream] = None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


# ------------------------------------------------------------------------------ device inputs
@dataclasses.dataclass
class DeviceSamples:
    x: torch.Tensor
    y: torch.Tensor
    z: torch.Tensor
    sdf: torch.Tensor
    refl: torch.Tensor
    nx: torch.Tensor
    ny: torch.Tensor
    nz: torch.Tensor
    power: torch.Tensor
    n_rays: int
    n_per_ray: int
    phi_origin: Optional[torch.Tensor] = None

    FIELDS = ("x", "y", "z", "sdf", "refl", "nx", "ny", "nz", "power")

    @property
    def n(self) -> int:
        return self.n_rays * self.n_per_ray

    @classmethod
    def from_host(cls, S, device="cuda") -> "DeviceSamples":
        t = lambda a: None if a is None else torch.as_tensor(np.ascontiguousarray(a, np.float32)).to(device)
        return cls(*(t(getattr(S, f)) for f in cls.FIELDS), n_rays=int(S.n_rays),
                   n_per_ray=int(S.n_per_ray), phi_origin=t(S.phi_origin))

    def struct(self) -> rfr_samples:
        return rfr_samples(*(_ptr(getattr(self, f)) for f in self.FIELDS), _ptr(self.phi_origin),
                           self.n_rays, self.n_per_ray)


@dataclasses.dataclass
class DeviceAntennas:
    tx_x: torch.Tensor
    tx_y: torch.Tensor
    tx_z: torch.Tensor
    rx_x: Optional[torch.Tensor] = None
    rx_y: Optional[torch.Tensor] = None
    rx_z: Optional[torch.Tensor] = None
    phi_tx: Optional[torch.Tensor] = None
    phi_rx: Optional[torch.Tensor] = None

    NAMES = ("tx_x", "tx_y", "tx_z", "rx_x", "rx_y", "rx_z", "phi_tx", "phi_rx")

    @property
    def n(self) -> int:
        return int(self.tx_x.shape[0])

    @classmethod
    def from_host(cls, A, device="cuda") -> "DeviceAntennas":
        t = lambda a: None if a is None else torch.as_tensor(np.ascontiguousarray(a, np.float32)).to(device)
        return cls(*(t(getattr(A, f)) for f in cls.NAMES))

    def slice(self, lo: int, hi: int) -> "DeviceAntennas":
        """A shard is a pointer offset plus a count (views of the same storage)."""
        return DeviceAntennas(*(None if getattr(self, f) is None else getattr(self, f)[lo:hi]
                                for f in self.NAMES))

    def struct(self) -> rfr_antennas:
        return rfr_antennas(*(_ptr(getattr(self, f)) for f in self.NAMES), self.n)


def grid_struct(grid) -> rfr_freq_grid:
    return rfr_freq_grid(float(grid.f0), float(grid.df), int(grid.n_freq))


# ------------------------------------------------------------------------------ ABI wrappers
def rfr_workspace_size(n_samples: int, n_ant: int, n_freq: int, n_query: int = 0) -> int:
    out = C.c_size_t()
    _check(load().rfr_workspace_size(n_samples, n_ant, n_freq, n_query, C.byref(out)),
           "rfr_workspace_size")
    return out.value


class Workspace:
    """Device scratch of librfr (rfr_workspace): a uint8 tensor plus its planning dimensions, the
    upper bounds of every call that uses it (include/librfr.h)."""

    def __init__(self, n_samples: int, n_ant: int, n_freq: int, n_query: int = 0, device="cuda",
                 nbytes: Optional[int] = None):
        self.dims = (int(n_samples), int(n_ant), int(n_freq), int(n_query))
        need = rfr_workspace_size(*self.dims)
        self.tensor = torch.zeros(max(need if nbytes is None else nbytes, 256), dtype=torch.uint8,
                                  device=device)

    def numel(self) -> int:
        return self.tensor.numel()

    def struct(self) -> rfr_workspace:
        return rfr_workspace(_ptr(self.tensor), self.tensor.numel(), *self.dims)

    def truncated(self, nbytes: int) -> "Workspace":
        """A view of the first nbytes with the same planning dims (for argument-error tests)."""
        w = Workspace.__new__(Workspace)
        w.dims, w.tensor = self.dims, self.tensor[:nbytes]
        return w


def cheb_state(ws: Workspace) -> dict:
    """Diagnostic (synchronous): the Chebyshev-moment choice the LAST call on this workspace took,
    read from the workspace header (librfr.cu kChebHdrOff): sel (0 = direct kernels), P, delta, and
    the empty-space-skipping counts of the last forward / backward (samples that carry work)."""
    import struct as _st
    raw = bytes(ws.tensor[64:148].cpu().numpy().tobytes())
    sel, P, delta, inv = _st.unpack("<Iidd", raw[:24])
    n_fwd, n_bwd = _st.unpack("<qq", raw[64:80])      # compacted active counts (offsets 128, 136)
    (p_tile,) = _st.unpack("<i", raw[80:84])           # moments of the last tiled filter (144)
    return {"sel": sel, "P": P, "delta": delta, "n_active_fwd": n_fwd, "n_active_bwd": n_bwd,
            "P_tiled_filter": p_tile}


def workspace(n_samples: int, n_ant: int, n_freq: int, n_query: int = 0, device="cuda") -> Workspace:
    return Workspace(n_samples, n_ant, n_freq, n_query, device)


def _ws(ws: Workspace):
    if not isinstance(ws, Workspace):
        raise RfrError("expected an rfr.Workspace")
    return C.byref(ws.struct())


def rfr_forward(samples: DeviceSamples, sharpness: float, ants: DeviceAntennas, grid,
                signal: torch.Tensor, ws: torch.Tensor, flags: int = 0, stream=None):
    s, a, g, o = samples.struct(), ants.struct(), grid_struct(grid), rfr_opts(flags)
    _check(load().rfr_forward(C.byref(s), float(sharpness), C.byref(a), C.byref(g), C.byref(o),
                              _ptr(signal), _ws(ws), _stream(stream)), "rfr_forward")
    return signal


def rfr_loss(signal: torch.Tensor, target: torch.Tensor, grad: torch.Tensor, loss: torch.Tensor,
             ws: torch.Tensor, stream=None):
    n = signal.numel() // 2
    _check(load().rfr_loss(_ptr(signal), _ptr(target), n, _ptr(grad), _ptr(loss), _ws(ws),
                           _stream(stream)), "rfr_loss")
    return loss, grad


def rfr_filter(signal: torch.Tensor, ants: DeviceAntennas, grid, qx, qy, qz, power: torch.Tensor,
               ws: torch.Tensor, mf: Optional[torch.Tensor] = None, comm: "Comm" = None,
               stream=None):
    a, g = ants.struct(), grid_struct(grid)
    _check(load().rfr_filter(_ptr(signal), C.byref(a), C.byref(g), _ptr(qx), _ptr(qy), _ptr(qz),
                             int(qx.numel()), _ptr(power), _ptr(mf), _comm(comm), _ws(ws),
                             _stream(stream)), "rfr_filter")
    return power


def rfr_filter_partial(signal, ants: DeviceAntennas, grid, qx, qy, qz, mf: torch.Tensor,
                       ws: torch.Tensor, stream=None):
    a, g = ants.struct(), grid_struct(grid)
    _check(load().rfr_filter_partial(_ptr(signal), C.byref(a), C.byref(g), _ptr(qx), _ptr(qy),
                                     _ptr(qz), int(qx.numel()), _ptr(mf), _ws(ws),
                                     _stream(stream)), "rfr_filter_partial")
    return mf


def rfr_filter_gather(signal: torch.Tensor, ants: DeviceAntennas, grid, qx, qy, qz,
                      power: torch.Tensor, ws: torch.Tensor, comm: Optional["Comm"] = None,
                      n_ant_total: Optional[int] = None, mf: Optional[torch.Tensor] = None,
                      stream=None):
    """Query-sharded filter (see include/librfr.h): power / mf hold this rank's query slice
    shard_range(len(qx), rank, world)."""
    a, g = ants.struct(), grid_struct(grid)
    n_tot = ants.n * (comm.nranks if comm else 1) if n_ant_total is None else n_ant_total
    _check(load().rfr_filter_gather(_ptr(signal), C.byref(a), int(n_tot), C.byref(g), _ptr(qx),
                                    _ptr(qy), _ptr(qz), int(qx.numel()), _ptr(power), _ptr(mf),
                                    _comm(comm), _ws(ws), _stream(stream)), "rfr_filter_gather")
    return power


def rfr_filter_power(mf: torch.Tensor, power: torch.Tensor, stream=None):
    _check(load().rfr_filter_power(_ptr(mf), int(power.numel()), _ptr(power), _stream(stream)),
           "rfr_filter_power")
    return power


def rfr_filter_backward(grad_power: torch.Tensor, mf: torch.Tensor, ants: DeviceAntennas, grid,
                        qx, qy, qz, grad_signal: torch.Tensor, ws: torch.Tensor,
                        power: Optional[torch.Tensor] = None, eps: float = 0.0, stream=None):
    """K5: dL/ds for a loss of the filter power (see include/librfr.h)."""
    a, g = ants.struct(), grid_struct(grid)
    _check(load().rfr_filter_backward(_ptr(grad_power), _ptr(mf), _ptr(power), float(eps),
                                      C.byref(a), C.byref(g), _ptr(qx), _ptr(qy), _ptr(qz),
                                      int(qx.numel()), _ptr(grad_signal), _ws(ws),
                                      _stream(stream)), "rfr_filter_backward")
    return grad_signal


def rfr_heatmap_loss(power: torch.Tensor, power_gt: torch.Tensor, grad_power: torch.Tensor,
                     loss: torch.Tensor, ws: torch.Tensor, cell: Optional[torch.Tensor] = None,
                     history: Optional[torch.Tensor] = None, thr_hi: float = 0.0,
                     ratio: float = 0.0, mask: Optional[torch.Tensor] = None, stream=None):
    """K7: masked heatmap L2 (see include/librfr.h).  cell: int32, history: float32, mask: uint8."""
    if cell is not None and cell.dtype != torch.int32:
        raise RfrError("cell must be int32")
    if mask is not None and mask.dtype != torch.uint8:
        raise RfrError("mask must be uint8")
    _check(load().rfr_heatmap_loss(_ptr(power), _ptr(power_gt), int(power.numel()), _ptr(cell),
                                   _ptr(history), float(thr_hi), float(ratio), _ptr(grad_power),
                                   _ptr(mask), _ptr(loss), _ws(ws), _stream(stream)),
           "rfr_heatmap_loss")
    return loss, grad_power


@dataclasses.dataclass
class Grads:
    sdf: torch.Tensor
    refl: torch.Tensor
    nx: torch.Tensor
    ny: torch.Tensor
    nz: torch.Tensor
    power: torch.Tensor
    sharpness: torch.Tensor

    NAMES = ("sdf", "refl", "nx", "ny", "nz", "power", "sharpness")

    @classmethod
    def empty(cls, n: int, device="cuda") -> "Grads":
        return cls(*(torch.empty(n, dtype=torch.float32, device=device) for _ in range(6)),
                   torch.empty(1, dtype=torch.float32, device=device))

    def struct(self) -> rfr_sample_grads:
        return rfr_sample_grads(*(_ptr(getattr(self, f)) for f in self.NAMES))


def rfr_backward(grad_signal: torch.Tensor, samples: DeviceSamples, sharpness: float,
                 ants: DeviceAntennas, grid, out: Grads, ws: torch.Tensor, flags: int = 0,
                 comm: "Comm" = None, stream=None):
    s, a, g, o, r = samples.struct(), ants.struct(), grid_struct(grid), rfr_opts(flags), out.struct()
    _check(load().rfr_backward(_ptr(grad_signal), C.byref(s), float(sharpness), C.byref(a),
                               C.byref(g), C.byref(o), C.byref(r), _comm(comm), _ws(ws),
                               _stream(stream)), "rfr_backward")
    return out


def rfr_backward_filter(grad_signal: torch.Tensor, signal: torch.Tensor, samples: DeviceSamples,
                        sharpness: float, ants: DeviceAntennas, grid, out: Grads,
                        power: torch.Tensor, ws: torch.Tensor, mf: Optional[torch.Tensor] = None,
                        flags: int = 0, comm: "Comm" = None, stream=None):
    """K3 + K4 in one sweep: rfr_backward from grad_signal and rfr_filter of signal at the sample
    points (see include/librfr.h)."""
    s, a, g, o, r = samples.struct(), ants.struct(), grid_struct(grid), rfr_opts(flags), out.struct()
    _check(load().rfr_backward_filter(_ptr(grad_signal), _ptr(signal), C.byref(s), float(sharpness),
                                      C.byref(a), C.byref(g), C.byref(o), C.byref(r), _ptr(power),
                                      _ptr(mf), _comm(comm), _ws(ws), _stream(stream)),
           "rfr_backward_filter")
    return out, power


def rfr_backward_filter_partial(grad_signal, signal, samples: DeviceSamples, sharpness: float,
                                ants: DeviceAntennas, grid, partials: torch.Tensor,
                                mf: torch.Tensor, ws: torch.Tensor, flags: int = 0, stream=None):
    """The fused sweep for one antenna shard: partials [5][n_s] and partial complex M [n_s]."""
    s, a, g, o = samples.struct(), ants.struct(), grid_struct(grid), rfr_opts(flags)
    _check(load().rfr_backward_filter_partial(_ptr(grad_signal), _ptr(signal), C.byref(s),
                                              float(sharpness), C.byref(a), C.byref(g), C.byref(o),
                                              _ptr(partials), _ptr(mf), _ws(ws), _stream(stream)),
           "rfr_backward_filter_partial")
    return partials, mf


def rfr_backward_partial(grad_signal, samples: DeviceSamples, sharpness: float,
                         ants: DeviceAntennas, grid, partials: torch.Tensor, ws: torch.Tensor,
                         flags: int = 0, stream=None):
    s, a, g, o = samples.struct(), ants.struct(), grid_struct(grid), rfr_opts(flags)
    _check(load().rfr_backward_partial(_ptr(grad_signal), C.byref(s), float(sharpness), C.byref(a),
                                       C.byref(g), C.byref(o), _ptr(partials), _ws(ws),
                                       _stream(stream)), "rfr_backward_partial")
    return partials


def rfr_backward_finish(partials: torch.Tensor, samples: DeviceSamples, sharpness: float,
                        out: Grads, ws: torch.Tensor, flags: int = 0, stream=None):
    s, o, r = samples.struct(), rfr_opts(flags), out.struct()
    _check(load().rfr_backward_finish(_ptr(partials), C.byref(s), float(sharpness), C.byref(o),
                                      C.byref(r), _ws(ws), _stream(stream)),
           "rfr_backward_finish")
    return out


def rfr_launch_count() -> int:
    return int(load().rfr_launch_count())


def rfr_plan_state(ws: torch.Tensor, stream=None) -> dict:
    """Plan of the last r2-engine call on ws (diagnostic, host-synchronous)."""
    v = rfr_plan_info()
    _check(load().rfr_plan_state(_ws(ws), C.byref(v), _stream(stream)), "rfr_plan_state")
    return {f: getattr(v, f) for f, _ in rfr_plan_info._fields_}


def rfr_profile_enable(on: bool = True):
    _check(load().rfr_profile_enable(1 if on else 0), "rfr_profile_enable")


def rfr_profile_read(sweep: str):
    """(milliseconds, launches) accumulated for one sweep since rfr_profile_enable(True)."""
    ms, n = C.c_double(), C.c_uint64()
    _check(load().rfr_profile_read(SWEEPS[sweep], C.byref(ms), C.byref(n)), "rfr_profile_read")
    return ms.value, n.value


def rfr_poll_flags(ws: torch.Tensor, stream=None) -> int:
    v = C.c_uint32()
    _check(load().rfr_poll_flags(_ws(ws), C.byref(v), _stream(stream)), "rfr_poll_flags")
    return v.value


# ------------------------------------------------------------------------------ multi-GPU host logic
class Comm:
    """librfr's NCCL communicator for this rank (rfr_comm_*).  The 128-byte unique id is created by
    rank 0 and broadcast with the caller's torch.distributed process group (plumbing only)."""

    def __init__(self, handle: int, nranks: int, rank: int):
        self.handle, self.nranks, self.rank = handle, nranks, rank

    @staticmethod
    def unique_id(group=None) -> bytes:
        """Rank 0's NCCL unique id (rfr_comm_unique_id), broadcast to every rank of the group
        (torch.distributed: plumbing only).  Host logic, no device needed."""
        import torch.distributed as dist
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        uid = (C.c_char * 128)()
        if rank == 0:
            _check(load().rfr_comm_unique_id(uid), "rfr_comm_unique_id")
        if world > 1:
            obj = [bytes(uid)]
            dist.broadcast_object_list(obj, src=0, group=group)
            return obj[0]
        return bytes(uid)

    @classmethod
    def create(cls, group=None) -> "Comm":
        import torch.distributed as dist
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        uid = (C.c_char * 128)()
        C.memmove(uid, cls.unique_id(group), 128)
        h = C.c_void_p()
        _check(load().rfr_comm_init(uid, world, rank, C.byref(h)), "rfr_comm_init")
        return cls(h.value, world, rank)

    def close(self):
        if self.handle:
            _check(load().rfr_comm_destroy(self.handle), "rfr_comm_destroy")
            self.handle = None


def _comm(c: Optional[Comm]):
    return None if c is None else c.handle



def shard_range(n: int, rank: int, world: int):
    """Contiguous antenna slice [lo, hi) of rank `rank` out of `world` (balanced to +-1)."""
    if world <= 0 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, rem = divmod(n, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def c64_view(t: torch.Tensor) -> torch.Tensor:
    """float32 [..., 2] interleaved view <-> complex64 helper for callers."""
    return torch.view_as_complex(t)
