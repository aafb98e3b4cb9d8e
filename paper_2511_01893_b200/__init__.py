"""B200-native memoized ADMM-FFT laminography (arXiv 2511.01893, "mLR").

Python face of ``lib/libmlr.so``: the drop-in ``mlr.h`` C ABI (host arrays,
same names and error model as the reference's capi.cpp) and the device
``mlrg.h`` C ABI (device pointers, e.g. torch tensors). The library is the
product; this module only binds it with ctypes. There is no CPU fallback:
every call fails loudly when the CUDA library is missing.
"""
from __future__ import annotations

import ctypes as C
import os
import tempfile

import numpy as np

__all__ = ["lib", "LIB_PATH", "MlrError", "Config", "Array", "Result", "make_phantom", "project",
           "reconstruct", "array_from_numpy", "Context", "DeviceRecon", "reconstruct_device", "Solver",
           "Memo", "projection_matrix", "slot_mix"]

LIB_PATH = os.environ.get("MLRG_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libmlr.so")
_LIB = None

MLR_OK, MLR_ERR_CONFIG, MLR_ERR_IO, MLR_ERR_RUNTIME, MLR_ERR_ABORTED = range(5)
COUNTER_NAMES = ["lookups", "cache_hits", "remote_hits", "misses", "cache_comparisons", "cache_probes",
                 "timeouts", "batches_sent", "inserts_enqueued", "inserts_sent", "inserts_dropped"]
OPS = {"fu1d": 0, "fu2d": 1, "fu1d_adj": 2, "fu2d_adj": 3, "f2d": 4, "f2d_adj": 5}


class MlrError(RuntimeError):
    """An MLR_* error code with the library's thread-local message."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


_P, _I64, _U64, _I32, _D = C.c_void_p, C.c_int64, C.c_uint64, C.c_int32, C.c_double
_SIGS = {
    # mlr.h
    "mlr_last_error": (C.c_char_p, []),
    "mlr_free": (None, [_P]),
    "mlr_config_new": (_P, []),
    "mlr_config_from_file": (_P, [C.c_char_p]),
    "mlr_config_set": (C.c_int, [_P, C.c_char_p, C.c_char_p]),
    "mlr_config_dump": (_P, [_P]),
    "mlr_config_free": (None, [_P]),
    "mlr_array_load": (_P, [C.c_char_p]),
    "mlr_array_save": (C.c_int, [_P, C.c_char_p]),
    "mlr_array_shape": (C.c_int, [_P, C.POINTER(_I64)]),
    "mlr_array_data": (C.POINTER(_D), [_P]),
    "mlr_array_free": (None, [_P]),
    "mlr_make_phantom": (_P, [C.c_char_p, _I64, _I64, _I64, _U64]),
    "mlr_project": (_P, [_P, _P]),
    "mlr_reconstruct": (_P, [_P, _P, _P]),
    "mlr_result_volume": (_P, [_P]),
    "mlr_result_csv": (_P, [_P]),
    "mlr_result_aborted": (C.c_int, [_P]),
    "mlr_result_abort_reason": (_P, [_P]),
    "mlr_result_free": (None, [_P]),
    "mlr_server_start": (_P, [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int]),
    "mlr_server_port": (C.c_int, [_P]),
    "mlr_server_stop": (None, [_P]),
    "mlr_plan_offload": (_P, [C.c_char_p, _D, C.c_char_p]),
    "mlr_lru_baseline": (_P, [C.c_char_p, _D, _U64]),
    "mlr_train_encoder": (_P, [_P, C.c_char_p, _U64, C.c_char_p]),
    "mlr_bench": (_P, [_P]),
    # mlrg.h
    "mlrg_last_error": (C.c_char_p, []),
    "mlrg_free": (None, [_P]),
    "mlrg_version": (C.c_int, []),
    "mlrg_ctx_create": (_P, [_I64, _I64, _I64, _I64, _I64, _I64, _D, _P]),
    "mlrg_ctx_create_kernel": (_P, [_I64, _I64, _I64, _I64, _I64, _I64, _D, _P, C.c_int]),
    "mlrg_ctx_destroy": (None, [_P]),
    "mlrg_sync": (C.c_int, [_P]),
    "mlrg_fu1d": (C.c_int, [_P, _P, _P, _I64]),
    "mlrg_fu1d_adj": (C.c_int, [_P, _P, _P, _I64]),
    "mlrg_fu2d": (C.c_int, [_P, _P, _P, _P, _I64]),
    "mlrg_fu2d_adj": (C.c_int, [_P, _P, _P, _I64]),
    "mlrg_f2d": (C.c_int, [_P, _P, _P, _I64, C.c_int]),
    "mlrg_forward_L": (C.c_int, [_P, _P, _P]),
    "mlrg_adjoint_L": (C.c_int, [_P, _P, _P]),
    "mlrg_grad": (C.c_int, [_P, _P, _P, _P, _P]),
    "mlrg_div": (C.c_int, [_P, _P, _P, _P, _P]),
    "mlrg_encode": (C.c_int, [_P, C.c_int, _P, _I64, C.c_int, _U64, _P, _P, _I64]),
    "mlrg_encode_cnn": (C.c_int, [_P, C.c_int, _P, _I64, C.c_int, _U64, _P, _P, _I64]),
    "mlrg_cnn_weights": (C.c_int, [C.c_int, _U64, _P, _P, _P]),
    "mlrg_reconstruct": (_P, [C.c_char_p, _P, _P, _P, _P]),
    "mlrg_recon_csv": (_P, [_P]),
    "mlrg_recon_aborted": (C.c_int, [_P]),
    "mlrg_recon_abort_reason": (_P, [_P]),
    "mlrg_recon_audit": (_I64, [_P, _P, _P, _I64]),
    "mlrg_recon_counters": (C.c_int, [_P, _P]),
    "mlrg_recon_tiers": (C.c_int, [_P, _P]),
    "mlrg_recon_free": (None, [_P]),
    "mlrg_solver_new": (_P, [C.c_char_p, _P, _P, _P]),
    "mlrg_solver_step": (C.c_int, [_P, _P]),
    "mlrg_solver_volume": (C.c_int, [_P, _P]),
    "mlrg_solver_csv": (_P, [_P]),
    "mlrg_solver_counters": (C.c_int, [_P, _P]),
    "mlrg_solver_tiers": (C.c_int, [_P, _P]),
    "mlrg_solver_audit": (_I64, [_P, _P, _P, _I64]),
    "mlrg_solver_free": (None, [_P]),
    "mlrg_solver_new_sharded": (_P, [C.c_char_p, _P, _P, _P, _P]),
    "mlrg_solver_shard": (C.c_int, [_P, _P]),
    "mlrg_comm_create": (_P, [C.c_char_p, C.c_int, C.c_int, _D]),
    "mlrg_comm_free": (None, [_P]),
    "mlrg_comm_barrier": (C.c_int, [_P]),
    "mlrg_comm_abort": (C.c_int, [_P]),
    "mlrg_comm_allreduce": (C.c_int, [_P, _P, C.c_int]),
    "mlrg_comm_allgather": (C.c_int, [_P, _P, _U64, _P]),
    "mlrg_partition": (C.c_int, [_I64, _I64, _I64, C.c_int, _P]),
    "mlrg_memo_new": (_P, [C.c_float, C.c_int, _U64, _U64, C.c_int, C.c_int, C.c_int]),
    "mlrg_memo_free": (None, [_P]),
    "mlrg_memo_lookup": (C.c_int, [_P, _I64, C.c_int, _P, _P, _P, _P, _P, _P, _P]),
    "mlrg_memo_insert": (C.c_int, [_P, C.c_int, _P, _U64]),
    "mlrg_memo_flush": (C.c_int, [_P]),
    "mlrg_memo_counters": (C.c_int, [_P, _P]),
    "mlrg_ctx_stats": (C.c_int, [_P, _P]),
    "mlrg_kmeans": (C.c_int, [_P, C.c_int64, C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int, _P, _P]),
    "mlrg_projection_matrix": (C.c_int, [_I64, _I64, _I64, C.c_int, _U64, _P, _I64]),
    "mlrg_slot_mix": (C.c_int, [_P, C.c_int, _U64, _I64, C.c_int]),
    "mlrg_result_audit": (_I64, [_P, _P, _P, _I64]),
    "mlrg_launch_count": (_U64, []),
    "mlrg_prof_enable": (None, [C.c_int]),
    "mlrg_prof_reset": (None, []),
    "mlrg_prof_query": (C.c_int, [C.c_char_p, _P, _P]),
    "mlrg_prof_dump": (C.c_int, [C.c_char_p]),
}
EXPORTS = tuple(_SIGS)


def lib():
    """Loads lib/libmlr.so once (RuntimeError if it was never built)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                               "(make -C paper_2511_01893_b200/csrc); there is no CPU fallback")
        handle = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(handle, name)
            fn.restype, fn.argtypes = res, args
        _LIB = handle
    return _LIB


def _err() -> str:
    return (lib().mlr_last_error() or b"").decode()


def _check(code: int):
    if code != MLR_OK:
        raise MlrError(code, _err())


def _ptr(p, what="call"):
    if not p:
        raise MlrError(MLR_ERR_RUNTIME, f"{what}: {_err()}")
    return p


def _take_text(p) -> str:
    if not p:
        raise MlrError(MLR_ERR_RUNTIME, _err())
    s = C.cast(p, C.c_char_p).value.decode()
    lib().mlr_free(p)
    return s


# ---------------------------------------------------------------------------------------------
# drop-in mlr.h surface
# ---------------------------------------------------------------------------------------------
class Config:
    """mlr_config: the reference's flat key=value configuration (config.hpp:16-46)."""

    def __init__(self, path: str | None = None, **keys):
        L = lib()
        self._h = _ptr(L.mlr_config_from_file(path.encode()) if path else L.mlr_config_new(), "config")
        for k, v in keys.items():
            self.set(k, v)

    def set(self, key: str, value) -> "Config":
        if isinstance(value, bool):
            value = "true" if value else "false"
        _check(lib().mlr_config_set(self._h, key.encode(), str(value).encode()))
        return self

    def dump(self) -> str:
        return _take_text(lib().mlr_config_dump(self._h))

    def __del__(self):
        if getattr(self, "_h", None) and _LIB is not None:
            _LIB.mlr_config_free(self._h)
            self._h = None


class Array:
    """mlr_array: a host complex128 array owned by the library."""

    def __init__(self, handle, owner=None):
        self._h, self._owner = _ptr(handle, "array"), owner

    @property
    def shape(self):
        s = (_I64 * 3)()
        _check(lib().mlr_array_shape(self._h, s))
        return tuple(int(x) for x in s)

    def numpy(self) -> np.ndarray:
        shape = self.shape
        n = int(np.prod(shape))
        ptr = lib().mlr_array_data(self._h)
        flat = np.ctypeslib.as_array(ptr, shape=(2 * n,)) if n else np.zeros(0)
        return flat.view(np.complex128).reshape(shape).copy()

    def view(self) -> np.ndarray:
        """Zero-copy read-only complex128 view of the data (mlr_array_data); the
        view keeps this Array (and a result's owner) alive."""
        shape = self.shape
        n = int(np.prod(shape))
        if n == 0:
            return np.zeros(shape, dtype=np.complex128)
        buf = (C.c_double * (2 * n)).from_address(C.cast(lib().mlr_array_data(self._h), C.c_void_p).value)
        buf._owner = self
        out = np.frombuffer(buf, dtype=np.complex128).reshape(shape)
        out.flags.writeable = False
        return out

    def save(self, path: str):
        _check(lib().mlr_array_save(self._h, path.encode()))

    @staticmethod
    def load(path: str) -> "Array":
        return Array(lib().mlr_array_load(path.encode()))

    def __del__(self):
        if getattr(self, "_h", None) and self._owner is None and _LIB is not None:
            _LIB.mlr_array_free(self._h)
            self._h = None


def array_from_numpy(a: np.ndarray, domain: int = 0) -> Array:
    """Builds an mlr_array through the public API only (an LVOL file, volume_io.cpp:16-35)."""
    a = np.ascontiguousarray(a, dtype=np.complex128)
    header = b"LVOL" + bytes([3, domain]) + bytes(10) + np.asarray(a.shape, "<u8").tobytes()
    with tempfile.NamedTemporaryFile(suffix=".lvol", delete=False) as f:
        f.write(header + a.astype("<c16").tobytes())
        path = f.name
    try:
        return Array.load(path)
    finally:
        os.unlink(path)


def make_phantom(kind: str, d0: int, d1: int, d2: int, seed: int = 1) -> Array:
    return Array(lib().mlr_make_phantom(kind.encode(), d0, d1, d2, seed))


def project(cfg: Config, volume: Array) -> Array:
    return Array(lib().mlr_project(cfg._h, volume._h))


class Result:
    """mlr_result: reconstruction volume, CSV report, abort flag and memo audit."""

    def __init__(self, handle):
        self._h = _ptr(handle, "reconstruct")

    @property
    def volume(self) -> Array:
        return Array(lib().mlr_result_volume(self._h), owner=self)

    @property
    def csv(self) -> str:
        return _take_text(lib().mlr_result_csv(self._h))

    @property
    def aborted(self) -> bool:
        return bool(lib().mlr_result_aborted(self._h))

    @property
    def abort_reason(self) -> str:
        return _take_text(lib().mlr_result_abort_reason(self._h))

    def audit(self):
        n = lib().mlrg_result_audit(self._h, None, None, 0)
        meta = np.zeros((n, 4), np.int32)
        cs = np.zeros(n, np.float32)
        lib().mlrg_result_audit(self._h, meta.ctypes.data, cs.ctypes.data, n)
        return meta, cs

    def __del__(self):
        if getattr(self, "_h", None) and _LIB is not None:
            _LIB.mlr_result_free(self._h)
            self._h = None


def reconstruct(cfg: Config, data: Array, reference: Array | None = None) -> Result:
    return Result(lib().mlr_reconstruct(cfg._h, data._h, reference._h if reference is not None else None))


def parse_csv(text: str):
    lines = [l for l in text.strip().splitlines() if l]
    head = lines[0].split(",")
    return [dict(zip(head, (float(x) for x in l.split(",")))) for l in lines[1:]]


# ---------------------------------------------------------------------------------------------
# device mlrg.h surface (torch tensors or any object with data_ptr())
# ---------------------------------------------------------------------------------------------
def _dp(t):
    if t is None:
        return None
    return t.data_ptr() if hasattr(t, "data_ptr") else int(t)


def _gcheck(code: int):
    if code != MLR_OK:
        raise MlrError(code, (lib().mlrg_last_error() or b"").decode())


def _default_stream(stream):
    """None -> torch's current CUDA stream when torch is in use, so device
    calls are ordered with the torch work that produced their inputs."""
    if stream is not None:
        return stream
    import sys as _sys

    torch = _sys.modules.get("torch")
    if torch is not None and torch.cuda.is_available():
        return torch.cuda.current_stream().cuda_stream
    return None


class Context:
    """mlrg_ctx: device operator tables for one geometry, bound to a CUDA stream.
    kernel: "es" (10-tap, default) or "gaussian" (the reference's 24-tap plan)."""

    KERNELS = {"es": 0, "gaussian": 1}

    def __init__(self, n1, n0, n2, n_theta, h, w, phi=0.5235987755982988, stream=None, kernel="es"):
        self.geom = (n1, n0, n2, n_theta, h, w)
        self.kernel = kernel
        self._h = lib().mlrg_ctx_create_kernel(n1, n0, n2, n_theta, h, w, phi, _default_stream(stream),
                                               self.KERNELS[kernel])
        if not self._h:
            raise MlrError(MLR_ERR_RUNTIME, (lib().mlrg_last_error() or b"").decode())

    def fu1d(self, u, out):
        _gcheck(lib().mlrg_fu1d(self._h, _dp(u), _dp(out), u.shape[0]))
        return out

    def fu1d_adj(self, v, out):
        _gcheck(lib().mlrg_fu1d_adj(self._h, _dp(v), _dp(out), v.shape[0]))
        return out

    def fu2d(self, v, out, d_hat=None):
        _gcheck(lib().mlrg_fu2d(self._h, _dp(v), _dp(d_hat), _dp(out), v.shape[1]))
        return out

    def fu2d_adj(self, p, out):
        _gcheck(lib().mlrg_fu2d_adj(self._h, _dp(p), _dp(out), p.shape[1]))
        return out

    def f2d(self, p, out, adjoint=False):
        _gcheck(lib().mlrg_f2d(self._h, _dp(p), _dp(out), p.shape[0], int(adjoint)))
        return out

    def forward_L(self, u, out):
        _gcheck(lib().mlrg_forward_L(self._h, _dp(u), _dp(out)))
        return out

    def adjoint_L(self, d, out):
        _gcheck(lib().mlrg_adjoint_L(self._h, _dp(d), _dp(out)))
        return out

    def grad(self, u, g0, g1, g2):
        _gcheck(lib().mlrg_grad(self._h, _dp(u), _dp(g0), _dp(g1), _dp(g2)))

    def div(self, g0, g1, g2, out):
        _gcheck(lib().mlrg_div(self._h, _dp(g0), _dp(g1), _dp(g2), _dp(out)))
        return out

    def encode(self, op: str, x, chunk_extent=16, key_dim=60, seed=1337):
        ax = 1 if op in ("fu2d", "fu2d_adj") else 0
        ns = -(-x.shape[ax] // chunk_extent)
        keys = np.zeros((ns, key_dim), np.float32)
        norms = np.zeros(ns, np.float64)
        _gcheck(lib().mlrg_encode(self._h, OPS[op], _dp(x), chunk_extent, key_dim, seed,
                                  keys.ctypes.data, norms.ctypes.data, ns))
        return keys, norms

    def encode_cnn(self, op: str, x, chunk_extent=16, key_dim=60, seed=1337):
        """Raw CNN keys (before slot_mix) and input norms per slab."""
        ax = 1 if op in ("fu2d", "fu2d_adj") else 0
        ns = -(-x.shape[ax] // chunk_extent)
        keys = np.zeros((ns, key_dim), np.float32)
        norms = np.zeros(ns, np.float64)
        _gcheck(lib().mlrg_encode_cnn(self._h, OPS[op], _dp(x), chunk_extent, key_dim, seed,
                                      keys.ctypes.data, norms.ctypes.data, ns))
        return keys, norms

    def stats(self) -> dict:
        out = np.zeros(6, np.int64)
        _gcheck(lib().mlrg_ctx_stats(self._h, out.ctypes.data))
        return dict(zip(("nclass", "taps", "m1", "m2", "gather_ctas", "classes_per_cta"), (int(x) for x in out)))

    def sync(self):
        _gcheck(lib().mlrg_sync(self._h))

    def __del__(self):
        if getattr(self, "_h", None) and _LIB is not None:
            _LIB.mlrg_ctx_destroy(self._h)
            self._h = None


class DeviceRecon:
    def __init__(self, handle):
        self._h = handle

    @property
    def csv(self) -> str:
        p = lib().mlrg_recon_csv(self._h)
        s = C.cast(p, C.c_char_p).value.decode()
        lib().mlrg_free(p)
        return s

    @property
    def aborted(self) -> bool:
        return bool(lib().mlrg_recon_aborted(self._h))

    @property
    def abort_reason(self) -> str:
        p = lib().mlrg_recon_abort_reason(self._h)
        s = C.cast(p, C.c_char_p).value.decode()
        lib().mlrg_free(p)
        return s

    def audit(self):
        n = lib().mlrg_recon_audit(self._h, None, None, 0)
        meta = np.zeros((n, 4), np.int32)
        cs = np.zeros(n, np.float32)
        lib().mlrg_recon_audit(self._h, meta.ctypes.data, cs.ctypes.data, n)
        return meta, cs

    def counters(self) -> dict:
        out = np.zeros(11, np.uint64)
        _gcheck(lib().mlrg_recon_counters(self._h, out.ctypes.data))
        return dict(zip(COUNTER_NAMES, (int(x) for x in out)))

    def tiers(self) -> dict:
        """Memo value tiers: HBM ring arena bytes, values / bytes spilled to pinned host."""
        out = np.zeros(3, np.uint64)
        _gcheck(lib().mlrg_recon_tiers(self._h, out.ctypes.data))
        return dict(zip(("arena_bytes", "spilled_values", "spilled_bytes"), (int(x) for x in out)))

    def __del__(self):
        if getattr(self, "_h", None) and _LIB is not None:
            _LIB.mlrg_recon_free(self._h)
            self._h = None


def reconstruct_device(config_text: str, d, u_out, reference=None, stream=None) -> DeviceRecon:
    h = lib().mlrg_reconstruct(config_text.encode(), _dp(d), _dp(reference), _dp(u_out), _default_stream(stream))
    if not h:
        raise MlrError(MLR_ERR_RUNTIME, (lib().mlrg_last_error() or b"").decode())
    return DeviceRecon(h)


class Comm:
    """mlrg_comm: the node-local communicator of the sharded solver (one process
    per GPU; every rank passes the same `name` and `world`)."""

    def __init__(self, name: str, rank: int, world: int, timeout_s: float = 120.0):
        self.rank, self.world = rank, world
        self._h = lib().mlrg_comm_create(name.encode(), rank, world, timeout_s)
        if not self._h:
            raise MlrError(MLR_ERR_RUNTIME, (lib().mlrg_last_error() or b"").decode())

    @classmethod
    def from_torch(cls, timeout_s: float = 120.0):
        """Joins with the ranks of the default torch.distributed group (any backend):
        rank 0 picks a fresh segment name and broadcasts it."""
        import os
        import uuid

        import torch.distributed as dist

        name = [f"mlrg-{os.getpid()}-{uuid.uuid4().hex[:12]}" if dist.get_rank() == 0 else None]
        dist.broadcast_object_list(name, src=0)
        return cls(name[0], dist.get_rank(), dist.get_world_size(), timeout_s)

    def barrier(self):
        _gcheck(lib().mlrg_comm_barrier(self._h))

    def abort(self):
        _gcheck(lib().mlrg_comm_abort(self._h))

    def allreduce(self, v: np.ndarray) -> np.ndarray:
        v = np.ascontiguousarray(v, dtype=np.float64)
        _gcheck(lib().mlrg_comm_allreduce(self._h, v.ctypes.data, v.size))
        return v

    def allgather(self, b: bytes) -> list:
        out = C.create_string_buffer(len(b) * self.world)
        _gcheck(lib().mlrg_comm_allgather(self._h, b, len(b), out))
        raw = out.raw
        return [raw[r * len(b):(r + 1) * len(b)] for r in range(self.world)]

    def __del__(self):
        if getattr(self, "_h", None) and _LIB is not None:
            _LIB.mlrg_comm_free(self._h)
            self._h = None


def partition(n1: int, h: int, world: int, chunk: int = 16) -> np.ndarray:
    """[world, 4] = per rank {a, b, c, d}: planes [a, b) and detector rows [c, d)
    (the reference's assign() over 16-slabs, scalerun.cpp:14-27)."""
    out = np.zeros((world, 4), np.int64)
    _gcheck(lib().mlrg_partition(n1, h, chunk, world, out.ctypes.data))
    return out


class Solver:
    """mlrg_solver: the ADMM outer loop on the device, one outer iteration per step().
    With `comm` (world > 1) the solve is z-slab sharded: d and reference are the full
    arrays on this rank's device, volume() returns this rank's planes (shard())."""

    def __init__(self, config_text: str, d, reference=None, stream=None, comm: "Comm" = None):
        self._comm = comm  # keep the communicator alive as long as the solver
        self._h = lib().mlrg_solver_new_sharded(config_text.encode(), _dp(d), _dp(reference),
                                                _default_stream(stream), comm._h if comm else None)
        if not self._h:
            raise MlrError(MLR_ERR_RUNTIME, (lib().mlrg_last_error() or b"").decode())

    def shard(self):
        out = np.zeros(4, np.int64)
        _gcheck(lib().mlrg_solver_shard(self._h, out.ctypes.data))
        return tuple(int(x) for x in out)

    def step(self) -> bool:
        ab = C.c_int(0)
        _gcheck(lib().mlrg_solver_step(self._h, C.byref(ab)))
        return not ab.value

    def volume(self, out):
        _gcheck(lib().mlrg_solver_volume(self._h, _dp(out)))
        return out

    @property
    def csv(self) -> str:
        p = lib().mlrg_solver_csv(self._h)
        s = C.cast(p, C.c_char_p).value.decode()
        lib().mlrg_free(p)
        return s

    def counters(self) -> dict:
        out = np.zeros(11, np.uint64)
        _gcheck(lib().mlrg_solver_counters(self._h, out.ctypes.data))
        return dict(zip(COUNTER_NAMES, (int(x) for x in out)))

    def tiers(self) -> dict:
        out = np.zeros(3, np.uint64)
        _gcheck(lib().mlrg_solver_tiers(self._h, out.ctypes.data))
        return dict(zip(("arena_bytes", "spilled_values", "spilled_bytes"), (int(x) for x in out)))

    def audit(self):
        n = lib().mlrg_solver_audit(self._h, None, None, 0)
        meta = np.zeros((n, 4), np.int32)
        cs = np.zeros(n, np.float32)
        lib().mlrg_solver_audit(self._h, meta.ctypes.data, cs.ctypes.data, n)
        return meta, cs

    def __del__(self):
        if getattr(self, "_h", None) and _LIB is not None:
            _LIB.mlrg_solver_free(self._h)
            self._h = None
        self._comm = None


class Memo:
    """The host memo client + store (decision logic only), for replay tests."""

    def __init__(self, tau=0.92, nprobe=8, insert_cap=256, coalesce_bytes=4096, global_cache=False,
                 nlist=64, train_size=1024):
        self._h = lib().mlrg_memo_new(tau, nprobe, insert_cap, coalesce_bytes, int(global_cache), nlist,
                                      train_size)
        if not self._h:
            raise MlrError(MLR_ERR_RUNTIME, (lib().mlrg_last_error() or b"").decode())

    def lookup(self, keys, locations, ops, value_bytes):
        keys = np.ascontiguousarray(keys, np.float32)
        n, kd = keys.shape
        loc = np.ascontiguousarray(locations, np.int64)
        opa = np.ascontiguousarray(ops, np.int32)
        vb = np.ascontiguousarray(value_bytes, np.uint64)
        oc, cs, vid = np.zeros(n, np.int32), np.zeros(n, np.float32), np.zeros(n, np.uint64)
        _gcheck(lib().mlrg_memo_lookup(self._h, n, kd, keys.ctypes.data, loc.ctypes.data, opa.ctypes.data,
                                       vb.ctypes.data, oc.ctypes.data, cs.ctypes.data, vid.ctypes.data))
        return oc, cs, vid

    def insert(self, key, value_bytes) -> bool:
        key = np.ascontiguousarray(key, np.float32)
        r = lib().mlrg_memo_insert(self._h, key.size, key.ctypes.data, value_bytes)
        if r < 0:
            raise MlrError(-r, (lib().mlrg_last_error() or b"").decode())
        return bool(r)

    def flush(self):
        _gcheck(lib().mlrg_memo_flush(self._h))

    def counters(self) -> dict:
        out = np.zeros(11, np.uint64)
        _gcheck(lib().mlrg_memo_counters(self._h, out.ctypes.data))
        return dict(zip(COUNTER_NAMES, (int(x) for x in out)))

    def __del__(self):
        if getattr(self, "_h", None) and _LIB is not None:
            _LIB.mlrg_memo_free(self._h)
            self._h = None


def prof_query(name: str):
    """(total device ms, launches) of one profiled kernel since the last reset."""
    ms, n = C.c_double(0), C.c_int64(0)
    _gcheck(lib().mlrg_prof_query(name.encode(), C.byref(ms), C.byref(n)))
    return ms.value, n.value


def cnn_weights(key_dim=60, seed=1337):
    """init_cnn weights (conv1, conv2, fc) of the CNN key encoder."""
    c1 = np.zeros((32, 2, 5, 5), np.float32)
    c2 = np.zeros((64, 32, 3, 3), np.float32)
    fc = np.zeros((key_dim, 64), np.float32)
    _gcheck(lib().mlrg_cnn_weights(key_dim, seed, c1.ctypes.data, c2.ctypes.data, fc.ctypes.data))
    return c1, c2, fc


def projection_matrix(shape, key_dim=60, seed=1337, count=None) -> np.ndarray:
    n = 2 * int(np.prod(shape))
    count = key_dim * n if count is None else count
    out = np.zeros(count, np.float32)
    _gcheck(lib().mlrg_projection_matrix(*shape, key_dim, seed, out.ctypes.data, count))
    return out


def slot_mix(key, location: int, op: int, seed=1337) -> np.ndarray:
    k = np.array(key, np.float32)
    _gcheck(lib().mlrg_slot_mix(k.ctypes.data, k.size, seed, location, op))
    return k
