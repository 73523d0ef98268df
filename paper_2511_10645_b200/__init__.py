"""paper_2511_10645_b200 -- B200-native ParoQuant hot path (scaled pairwise rotation +
INT4 weight-only linear), arXiv 2511.10645.

Thin ctypes binding over the C ABI in include/paro.h (libparo.so, built in-tree by
``_build.build()``).  Every function here only marshals arguments: torch tensors
-> device pointers + the current CUDA stream.  All arithmetic runs in the CUDA
kernels of libparo.so; there is no CPU fallback -- if the library is missing,
importing this package raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libparo.so")

PARO_OK, PARO_ERR_INVALID_ARGUMENT, PARO_ERR_SHAPE, PARO_ERR_PAIRS, PARO_ERR_UNSUPPORTED, PARO_ERR_CUDA, \
    PARO_ERR_NCCL = range(7)
STATUS_NAMES = {0: "ok", 1: "invalid_argument", 2: "shape", 3: "pairs", 4: "unsupported", 5: "cuda", 6: "nccl"}
PARO_F16, PARO_BF16, PARO_F32 = 0, 1, 2
PARO_LINEAR_NO_ROTATION = 0x1
PARO_LINEAR_PDL = 0x2
PARO_LINEAR_FORCE_GEMV = 0x4
PARO_LINEAR_FORCE_GEMM = 0x8
PARO_LINEAR_TCGEN05 = 0x10
GROUP = 128
SLOTS = 64


class ParoError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"paro {STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status
        self.kind = STATUS_NAMES.get(status, str(status))


class paro_packed_sizes(ctypes.Structure):
    _fields_ = [(n, ctypes.c_size_t) for n in ("codes", "scales", "zeros", "rot_cs", "rot_idx", "svec")]


class paro_packed(ctypes.Structure):
    _fields_ = [("codes", ctypes.c_void_p), ("scales", ctypes.c_void_p), ("zeros", ctypes.c_void_p),
                ("rot_cs", ctypes.c_void_p), ("rot_idx", ctypes.c_void_p), ("svec", ctypes.c_void_p),
                ("N", ctypes.c_int64), ("K", ctypes.c_int64), ("group", ctypes.c_int32), ("n_rot", ctypes.c_int32)]


class paro_chain_stage(ctypes.Structure):
    _fields_ = [("x", ctypes.c_void_p), ("n", ctypes.c_int32), ("packed", ctypes.POINTER(paro_packed)),
                ("bias", ctypes.POINTER(ctypes.c_void_p)), ("y", ctypes.POINTER(ctypes.c_void_p))]


# (name, restype, argtypes) of every symbol declared in include/paro.h
_P, _I64, _I32, _U32, _SZ = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32, ctypes.c_size_t
_PP = ctypes.POINTER(paro_packed)
SIGNATURES = {
    "paro_pack_sizes": (ctypes.c_int, [_I64, _I64, _I32, _I32, ctypes.POINTER(paro_packed_sizes)]),
    "paro_pack": (ctypes.c_int, [_P, _P, _P, _P, _I64, _I64, _I32, _I32, _I32, _PP, _P]),
    "paro_linear_workspace": (_SZ, [_I64, _I64, _I64, _I32, _I32, _I32, _U32]),
    "paro_linear": (ctypes.c_int, [_P, ctypes.c_int, _I64, _PP, _P, _P, _P, _I32, _P, _P, ctypes.c_int, _U32, _P,
                                   _SZ, _P]),
    "paro_linear_multi": (ctypes.c_int, [_P, ctypes.c_int, _I64, _I32, _PP, _P, _P, ctypes.c_int, _U32, _P, _SZ,
                                         _P]),
    "paro_linear_chain_workspace": (_SZ, [_I64, _I32, ctypes.POINTER(paro_chain_stage)]),
    "paro_linear_chain": (ctypes.c_int, [_I32, ctypes.POINTER(paro_chain_stage), ctypes.c_int, _I64, ctypes.c_int, _U32,
                                         _P, _SZ, _P]),
    "paro_transform_activations": (ctypes.c_int, [_P, ctypes.c_int, _I64, _PP, _P, _P]),
    "paro_transform_dense_workspace": (_SZ, [_I64]),
    "paro_transform_activations_dense": (ctypes.c_int, [_P, ctypes.c_int, _I64, _PP, _P, _P, _SZ, _P]),
    "paro_unpack_logical": (ctypes.c_int, [_PP, _P, _P, _P, _P]),
    "paro_comm_unique_id": (ctypes.c_int, [_P]),
    "paro_comm_init": (ctypes.c_int, [_P, _I32, _I32, ctypes.POINTER(ctypes.c_void_p)]),
    "paro_comm_destroy": (ctypes.c_int, [_P]),
    "paro_comm_check": (ctypes.c_int, [_P]),
    "paro_linear_allgather_workspace": (_SZ, [_I64, _I64, _I64, _I32, ctypes.c_int, _U32]),
    "paro_linear_allgather": (ctypes.c_int, [_P, ctypes.c_int, _I64, _PP, _P, _P, ctypes.c_int, _U32, _P, _SZ, _P,
                                             _I32, _I32, _P]),
    "paro_select_pairs": (ctypes.c_int, [_I64, _I32, _I32, _I32, ctypes.c_uint64, _P]),
    "paro_p2p_buffer_bytes": (_SZ, [_I64, _I64, ctypes.c_int, _I32]),
    "paro_ipc_get_handle": (ctypes.c_int, [_P, _P]),
    "paro_ipc_open_handle": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_void_p)]),
    "paro_ipc_close_handle": (ctypes.c_int, [_P]),
    "paro_linear_allgather_p2p": (ctypes.c_int, [_P, ctypes.c_int, _I64, _PP, _P, ctypes.c_int, _U32,
                                                 ctypes.POINTER(ctypes.c_void_p), _I32, _I32, _P]),
    "paro_fwht": (ctypes.c_int, [_P, ctypes.c_int, _I64, _I64, _P, ctypes.c_float, _P, _P]),
    "paro_copy": (ctypes.c_int, [_P, _P, _SZ, _U32, _P]),
    "paro_last_error": (ctypes.c_char_p, []),
    "paro_version": (ctypes.c_char_p, []),
}


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = _load()


def last_error() -> str:
    return (_lib.paro_last_error() or b"").decode()


def _check(st: int) -> None:
    if st != PARO_OK:
        raise ParoError(st, last_error())


# ---------------------------------------------------------------- torch marshalling helpers
def _torch():
    import torch
    return torch


def _stream(stream=None) -> int:
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _dt(t) -> int:
    torch = _torch()
    return {torch.float16: PARO_F16, torch.bfloat16: PARO_BF16, torch.float32: PARO_F32}[t.dtype]


@dataclass
class PackedLinear:
    """Device buffers of one packed linear layer (caller-owned torch tensors) and the
    C struct that points at them."""
    codes: object
    scales: object
    zeros: object
    rot_cs: object
    rot_idx: object
    svec: object
    N: int
    K: int
    n_rot: int

    def struct(self) -> paro_packed:
        return paro_packed(_ptr(self.codes), _ptr(self.scales), _ptr(self.zeros), _ptr(self.rot_cs),
                           _ptr(self.rot_idx), _ptr(self.svec), self.N, self.K, GROUP, self.n_rot)

    def nbytes_algorithmic(self) -> int:
        """W4A16 bytes the GEMV must stream: codes + fp16 scales + uint4 zeros."""
        G = self.K // GROUP
        return self.N * self.K // 2 + self.N * G * 2 + self.N * G // 2


def paro_pack_sizes(N: int, K: int, group: int = GROUP, n_rot: int = 8) -> paro_packed_sizes:
    out = paro_packed_sizes()
    _check(_lib.paro_pack_sizes(N, K, group, n_rot, ctypes.byref(out)))
    return out


def alloc_packed(N: int, K: int, n_rot: int = 8, device="cuda") -> PackedLinear:
    torch = _torch()
    sz = paro_pack_sizes(N, K, GROUP, n_rot)

    def buf(n):
        return torch.empty(max(int(n), 16), dtype=torch.uint8, device=device)

    return PackedLinear(buf(sz.codes), buf(sz.scales), buf(sz.zeros), buf(sz.rot_cs), buf(sz.rot_idx),
                        buf(sz.svec), N, K, n_rot)


def paro_pack(W, s, theta, pairs, group: int = GROUP, out: PackedLinear | None = None, stream=None) -> PackedLinear:
    """W fp16 [N,K], s fp32 [K], theta fp32 [K/128,L,P], pairs int16 [K/128,L,P,2] (all CUDA)."""
    N, K = W.shape
    L = 0 if theta is None else theta.shape[1]
    P = 0 if theta is None else theta.shape[2]
    if out is None:
        out = alloc_packed(N, K, L, device=W.device)
    st = out.struct()
    _check(_lib.paro_pack(_ptr(W), _ptr(s), _ptr(theta), _ptr(pairs), N, K, group, L, P, ctypes.byref(st),
                          _stream(stream)))
    return out


def paro_linear_workspace(B: int, N: int, K: int, n_rot: int = 8, n_pairs: int = 64, on_the_fly: bool = False,
                          flags: int = 0) -> int:
    return int(_lib.paro_linear_workspace(B, N, K, n_rot, n_pairs, int(on_the_fly), flags))


def paro_linear(x, packed: PackedLinear, s=None, theta=None, pairs=None, bias=None, y=None, out_dtype=None,
                flags: int = 0, workspace=None, stream=None):
    """y[B,N] = transform(x) . dequant(Q)^T + bias.  x fp16/bf16 [B,K] (CUDA)."""
    torch = _torch()
    B = x.shape[0]
    if y is None:
        y = torch.empty((B, packed.N), dtype=out_dtype or x.dtype, device=x.device)
    P = 0 if theta is None else theta.shape[2]
    need = paro_linear_workspace(B, packed.N, packed.K, packed.n_rot, P or 64, s is not None, flags)
    if need and (workspace is None or workspace.numel() < need):
        workspace = torch.empty(need, dtype=torch.uint8, device=x.device)
    st = packed.struct()
    _check(_lib.paro_linear(_ptr(x), _dt(x), B, ctypes.byref(st), _ptr(s), _ptr(theta), _ptr(pairs), P, _ptr(bias),
                            _ptr(y), _dt(y), flags, _ptr(workspace), 0 if workspace is None else workspace.numel(),
                            _stream(stream)))
    return y


def paro_linear_multi(x, packed: list, bias=None, y=None, out_dtype=None, flags: int = 0, workspace=None,
                      stream=None):
    """Several linears sharing x (q/k/v, gate/up) in one decode launch; returns [y_i]."""
    torch = _torch()
    B = x.shape[0]
    n = len(packed)
    if y is None:
        y = [torch.empty((B, p.N), dtype=out_dtype or x.dtype, device=x.device) for p in packed]
    need = len(packed) * max(paro_linear_workspace(B, p.N, p.K, p.n_rot, 64, False, flags) for p in packed)
    if need and (workspace is None or workspace.numel() < need):
        workspace = torch.empty(need, dtype=torch.uint8, device=x.device)
    structs = (paro_packed * n)(*[p.struct() for p in packed])
    ys = (ctypes.c_void_p * n)(*[t.data_ptr() for t in y])
    bs = None if bias is None else (ctypes.c_void_p * n)(*[_ptr(b) for b in bias])
    _check(_lib.paro_linear_multi(_ptr(x), _dt(x), B, n, structs, bs, ys, _dt(y[0]), flags, _ptr(workspace),
                                  0 if workspace is None else workspace.numel(), _stream(stream)))
    return y


class ChainStage:
    """One stage of a decode chain: linears `packed` sharing activation `x` (a [B, K] tensor that
    may be a view of an earlier stage's output), outputs `y` (list of [B, N_i] tensors), `bias`."""

    def __init__(self, x, packed: list, y: list, bias=None):
        self.x, self.packed, self.y, self.bias = x, list(packed), list(y), bias


def _chain_structs(stages):
    keep, arr = [], (paro_chain_stage * len(stages))()
    for k, st in enumerate(stages):
        n = len(st.packed)
        structs = (paro_packed * n)(*[p.struct() for p in st.packed])
        ys = (ctypes.c_void_p * n)(*[t.data_ptr() for t in st.y])
        bs = None if st.bias is None else (ctypes.c_void_p * n)(*[_ptr(b) for b in st.bias])
        keep += [structs, ys, bs]
        arr[k].x = _ptr(st.x)
        arr[k].n = n
        arr[k].packed = ctypes.cast(structs, ctypes.POINTER(paro_packed))
        arr[k].bias = None if bs is None else ctypes.cast(bs, ctypes.POINTER(ctypes.c_void_p))
        arr[k].y = ctypes.cast(ys, ctypes.POINTER(ctypes.c_void_p))
    return arr, keep


def paro_linear_chain_workspace(B: int, stages) -> int:
    arr, _keep = _chain_structs(stages)
    return int(_lib.paro_linear_chain_workspace(B, len(stages), arr))


def chain_workspace(B: int, stages, device=None):
    """A zero-initialised workspace for paro_linear_chain (its barrier words must start at 0)."""
    torch = _torch()
    dev = device if device is not None else stages[0].x.device
    return torch.zeros(max(256, paro_linear_chain_workspace(B, stages)), dtype=torch.uint8, device=dev)


def paro_linear_chain(stages, flags: int = 0, workspace=None, stream=None):
    """Run decode stages in order in one persistent launch (<= 16 stages per launch): stage s + 1
    may read an earlier stage's y as its x (include/paro.h, paro_linear_chain)."""
    B = stages[0].x.shape[0]
    if workspace is None:
        workspace = chain_workspace(B, stages)
    arr, _keep = _chain_structs(stages)
    _check(_lib.paro_linear_chain(len(stages), arr, _dt(stages[0].x), B, _dt(stages[0].y[0]), flags,
                                  _ptr(workspace), workspace.numel(), _stream(stream)))
    return [st.y for st in stages]


def paro_transform_activations(x, packed: PackedLinear, out=None, stream=None):
    torch = _torch()
    if out is None:
        out = torch.empty(x.shape, dtype=torch.float16, device=x.device)
    st = packed.struct()
    _check(_lib.paro_transform_activations(_ptr(x), _dt(x), x.shape[0], ctypes.byref(st), _ptr(out),
                                           _stream(stream)))
    return out


def paro_transform_activations_dense(x, packed: PackedLinear, out=None, workspace=None, stream=None):
    """x' via the dense per-group form (M_g = R_L..R_1 diag(s_g) built per call, fp16 contraction)."""
    torch = _torch()
    if out is None:
        out = torch.empty(x.shape, dtype=torch.float16, device=x.device)
    need = _lib.paro_transform_dense_workspace(packed.K)
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device=x.device)
    st = packed.struct()
    _check(_lib.paro_transform_activations_dense(_ptr(x), _dt(x), x.shape[0], ctypes.byref(st), _ptr(out),
                                                 _ptr(workspace), workspace.numel(), _stream(stream)))
    return out


def paro_unpack_logical(packed: PackedLinear, stream=None):
    torch = _torch()
    dev = packed.codes.device
    G = packed.K // GROUP
    codes = torch.empty((packed.N, packed.K), dtype=torch.uint8, device=dev)
    scales = torch.empty((packed.N, G), dtype=torch.float16, device=dev)
    zeros = torch.empty((packed.N, G), dtype=torch.uint8, device=dev)
    st = packed.struct()
    _check(_lib.paro_unpack_logical(ctypes.byref(st), _ptr(codes), _ptr(scales), _ptr(zeros), _stream(stream)))
    return codes, scales, zeros


def paro_copy(dst, src, flags: int = 0, stream=None):
    """dst <- src by the SMs (device or pinned host tensors, same byte size; include/paro.h)."""
    nbytes = dst.numel() * dst.element_size()
    if src.numel() * src.element_size() != nbytes:
        raise ValueError("paro_copy: dst and src differ in size")
    _check(_lib.paro_copy(_ptr(dst), _ptr(src), nbytes, flags, _stream(stream)))
    return dst


def paro_fwht(x, signs=None, scale: float = 1.0, out=None, stream=None):
    """y (fp16) = scale * H_n diag(signs) x per row of x [T, n] (include/paro.h, paro_fwht)."""
    torch = _torch()
    T, n = x.shape
    if out is None:
        out = torch.empty((T, n), dtype=torch.float16, device=x.device)
    _check(_lib.paro_fwht(_ptr(x), _dt(x), T, n, _ptr(signs), float(scale), _ptr(out), _stream(stream)))
    return out


# ---------------------------------------------------------------- Alg. A1 (host)
def paro_select_pairs(n_groups: int, g: int = GROUP, n_rot: int = 8, n_pairs: int = SLOTS, seed: int = 0):
    """Alg. A1 pair lists for n_groups groups: numpy int16 [n_groups, n_rot, n_pairs, 2] (host),
    (-1, -1) in the slots of a short rotation (include/paro.h, paro_select_pairs)."""
    import numpy as np
    out = np.empty((max(n_groups, 0), max(n_rot, 0), max(n_pairs, 0), 2), dtype=np.int16)
    _check(_lib.paro_select_pairs(n_groups, g, n_rot, n_pairs, seed & ((1 << 64) - 1),
                                  out.ctypes.data if out.size else None))
    return out


# ---------------------------------------------------------------- NCCL-sharded linear
def paro_comm_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.paro_comm_unique_id(buf))
    return buf.raw


def paro_comm_init(uid: bytes, rank: int, world: int) -> int:
    comm = ctypes.c_void_p()
    buf = ctypes.create_string_buffer(uid, 128)
    _check(_lib.paro_comm_init(buf, rank, world, ctypes.byref(comm)))
    return comm.value


def paro_comm_destroy(comm: int) -> None:
    _check(_lib.paro_comm_destroy(comm))


def paro_comm_check(comm: int) -> None:
    """Raise ParoError(PARO_ERR_NCCL) if NCCL reported an asynchronous error on comm."""
    _check(_lib.paro_comm_check(comm))


def paro_linear_allgather(x, packed_shard: PackedLinear, comm: int, rank: int, world: int, bias_shard=None, y=None,
                          out_dtype=None, flags: int = 0, workspace=None, stream=None):
    torch = _torch()
    B = x.shape[0]
    N = packed_shard.N * world
    if y is None:
        y = torch.empty((B, N), dtype=out_dtype or x.dtype, device=x.device)
    need = int(_lib.paro_linear_allgather_workspace(B, packed_shard.N, packed_shard.K, world, _dt(y), flags))
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device=x.device)
    st = packed_shard.struct()
    _check(_lib.paro_linear_allgather(_ptr(x), _dt(x), B, ctypes.byref(st), _ptr(bias_shard), _ptr(y), _dt(y), flags,
                                      _ptr(workspace), workspace.numel(), comm, rank, world, _stream(stream)))
    return y


# ---------------------------------------------------------------- NVLink-native all-gather (P2P)
def p2p_buffer(N_full: int, world: int, out_dtype=None, device="cuda"):
    """Zeroed per-rank exchange buffer (y_full + flags) for paro_linear_allgather_p2p."""
    torch = _torch()
    dt = out_dtype or torch.float16
    nb = int(_lib.paro_p2p_buffer_bytes(1, N_full, _dt(torch.empty(0, dtype=dt)), world))
    if nb == 0:
        raise ParoError(PARO_ERR_INVALID_ARGUMENT, "bad p2p buffer arguments")
    return torch.zeros(nb, dtype=torch.uint8, device=device)


def paro_ipc_get_handle(t) -> bytes:
    buf = ctypes.create_string_buffer(64)
    _check(_lib.paro_ipc_get_handle(_ptr(t), buf))
    return buf.raw


def paro_ipc_open_handle(handle: bytes) -> int:
    p = ctypes.c_void_p()
    _check(_lib.paro_ipc_open_handle(ctypes.create_string_buffer(handle, 64), ctypes.byref(p)))
    return p.value


def paro_ipc_close_handle(ptr: int) -> None:
    _check(_lib.paro_ipc_close_handle(ptr))


def paro_linear_allgather_p2p(x, packed_shard: PackedLinear, peer_ptrs: list, rank: int, world: int, local_buf,
                              bias_shard=None, out_dtype=None, flags: int = 0, stream=None):
    """y_full [1, N] on every rank: this rank's shard GEMV stores into all ranks' buffers over NVLink
    (include/paro.h, paro_linear_allgather_p2p); returns the view of y_full in local_buf."""
    torch = _torch()
    dt = out_dtype or x.dtype
    N_full = packed_shard.N * world
    ptrs = (ctypes.c_void_p * world)(*peer_ptrs)
    st = packed_shard.struct()
    _check(_lib.paro_linear_allgather_p2p(_ptr(x), _dt(x), x.shape[0], ctypes.byref(st), _ptr(bias_shard),
                                          _dt(torch.empty(0, dtype=dt)), flags, ptrs, rank, world, _stream(stream)))
    es = torch.empty(0, dtype=dt).element_size()
    return local_buf[:N_full * es].view(dt).view(1, N_full)


def shard_rows(N: int, world: int, rank: int) -> tuple[int, int]:
    """Row range [r0, r1) of output channels owned by `rank`."""
    if N % world:
        raise ParoError(PARO_ERR_SHAPE, f"N={N} not divisible by world={world}")
    n = N // world
    return rank * n, (rank + 1) * n


def version() -> str:
    return _lib.paro_version().decode()
