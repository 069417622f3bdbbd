"""B200-native coarse-grid Dirac operator (arXiv:1612.07873) -- Python binding.

A thin ctypes layer over the C ABI in ``include/coarse_dslash.h`` (library
``libcoarse_dslash.so``, built in-tree by ``paper_1612_07873_b200.build``).  Every step of
the operator runs in the library's sm_100a kernels; this module only marshals arguments.
PyTorch, when used, supplies device memory (``torch.empty(..., device="cuda")``), streams
(``torch.cuda.current_stream().cuda_stream``) and process groups (NCCL-id broadcast).

There is no CPU fallback: if the library is missing this import fails loudly.

Function names mirror the C ABI (``coarse_field_alloc``, ``coarse_links_upload``,
``coarse_dslash_apply``, ``coarse_dslash_apply_dagger``, ...); the classes ``Context``,
``Field`` and ``Links`` are conveniences over them.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CD_LIB_PATH") or os.path.join(_HERE, "libcoarse_dslash.so")   # override: A/B experiments

CD_OK, CD_ERR_INVALID, CD_ERR_UNSUPPORTED, CD_ERR_OOM, CD_ERR_CUDA, CD_ERR_NCCL, CD_ERR_MISMATCH = 0, -1, -2, -3, -4, -5, -6
CD_ERR_COMM = -7
CD_FP32, CD_FP16 = 0, 1
CD_C64, CD_C128 = 0, 1
CD_LINKS_GENERAL, CD_LINKS_HERMITIAN, CD_LINKS_TI_GENERAL, CD_LINKS_TI_HERMITIAN = 0, 1, 2, 3
CD_OPT_VARIANT, CD_OPT_TUNE, CD_OPT_HALO_SELF_MASK, CD_OPT_PDL = 0, 1, 2, 3
CD_OPT_TRANSPORT, CD_OPT_NCCL_SM_RESERVE, CD_OPT_PEER_TIMEOUT_MS = 4, 5, 6
TRANSPORT = {"auto": 0, "nccl": 1, "peer": 2, "copy": 3}

PREC = {"fp32": CD_FP32, "fp16": CD_FP16, CD_FP32: CD_FP32, CD_FP16: CD_FP16}
LINK_KIND = {"general": 0, "hermitian": 1, "ti_general": 2, "ti_hermitian": 3}

# Every symbol include/coarse_dslash.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "cd_version", "cd_last_error", "cd_get_unique_id", "cd_context_create", "cd_context_destroy",
    "cd_context_set_option", "cd_context_local", "cd_variant_count", "cd_variant_name",
    "cd_context_chosen_variant", "cd_launch_count", "coarse_field_bytes", "coarse_field_alloc",
    "coarse_field_free", "coarse_field_import", "coarse_field_export", "coarse_field_generate",
    "coarse_field_stored_bytes", "coarse_field_read_stored", "coarse_links_upload", "coarse_links_generate",
    "coarse_links_stored_bytes", "coarse_links_read_stored", "coarse_links_free", "coarse_dslash_apply",
    "coarse_dslash_apply_dagger", "coarse_halo_pack", "cd_flush_l2", "cd_halo_plan_create",
    "coarse_dslash_apply_chain", "coarse_field_bytes_mrhs", "coarse_field_alloc_mrhs", "coarse_dslash_apply_mrhs",
    "coarse_links_compress_hermitian", "coarse_field_bytes_parity", "coarse_field_alloc_parity",
    "coarse_links_prepare_eo", "coarse_dslash_apply_eo", "coarse_transfer_create", "coarse_transfer_free",
    "coarse_transfer_fine_bytes", "coarse_transfer_read_basis", "coarse_transfer_orthonormalise", "coarse_restrict",
    "coarse_prolong", "cd_context_peer_handle", "cd_context_peer_connect", "coarse_halo_exchange",
)


class CDError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[cd status {code}] {msg}")
        self.code = code


class _Geometry(ctypes.Structure):
    _fields_ = [("global_dims", ctypes.c_int32 * 4), ("nvec", ctypes.c_int32), ("proc_grid", ctypes.c_int32 * 4)]


class HaloPlan(ctypes.Structure):
    """cd_halo_plan (include/coarse_dslash.h): decomposition + halo wire layout of one rank."""
    _fields_ = [("local_dims", ctypes.c_int32 * 4), ("grid_coords", ctypes.c_int32 * 4),
                ("local_volume", ctypes.c_int64), ("split_mask", ctypes.c_int32),
                ("nbr_rank", (ctypes.c_int32 * 2) * 4), ("face_sites", ctypes.c_int64 * 4),
                ("record_bytes", ctypes.c_int64), ("scale_bytes", ctypes.c_int64),
                ("block_offset", (ctypes.c_int64 * 2) * 4), ("block_bytes", ctypes.c_int64 * 4),
                ("total_bytes", ctypes.c_int64)]


class _TransferDesc(ctypes.Structure):
    """cd_transfer_desc (include/coarse_dslash.h)."""
    _fields_ = [("block", ctypes.c_int32 * 4), ("nspin", ctypes.c_int32), ("ncolor", ctypes.c_int32)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_1612_07873_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P, I, I64, SZ, U64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_size_t, ctypes.c_uint64
    PP = ctypes.POINTER(ctypes.c_void_p)
    sig = {
        "cd_version": ([], ctypes.c_char_p),
        "cd_last_error": ([], ctypes.c_char_p),
        "cd_get_unique_id": ([P], I),
        "cd_context_create": ([ctypes.POINTER(_Geometry), I, I, I, P, PP], I),
        "cd_context_destroy": ([P], I),
        "cd_context_set_option": ([P, I, I64], I),
        "cd_context_local": ([P, P, P, P], I),
        "cd_variant_count": ([P, I], I),
        "cd_variant_name": ([P, I, I], ctypes.c_char_p),
        "cd_context_chosen_variant": ([P, I, I], I),
        "cd_launch_count": ([], U64),
        "coarse_field_bytes": ([P, I], SZ),
        "coarse_field_alloc": ([P, I, P, SZ, PP], I),
        "coarse_field_free": ([P], I),
        "coarse_field_import": ([P, P, I, I, P], I),
        "coarse_field_export": ([P, P, I, I, P], I),
        "coarse_field_generate": ([P, U64, ctypes.c_uint32, ctypes.c_int32, P], I),
        "coarse_field_stored_bytes": ([P], SZ),
        "coarse_field_read_stored": ([P, P, I, P], I),
        "coarse_links_upload": ([P, I, P, I, I, P, PP], I),
        "coarse_links_generate": ([P, I, I, U64, ctypes.c_int32, P, PP], I),
        "coarse_links_stored_bytes": ([P], SZ),
        "coarse_links_read_stored": ([P, P, I, P], I),
        "coarse_links_free": ([P], I),
        "coarse_dslash_apply": ([P, P, P, P], I),
        "coarse_dslash_apply_dagger": ([P, P, P, P], I),
        "coarse_halo_pack": ([P, P, P, I, ctypes.POINTER(SZ), P], I),
        "cd_flush_l2": ([P, SZ, P], I),
        "cd_halo_plan_create": ([ctypes.POINTER(_Geometry), I, I, I, ctypes.c_int32, ctypes.POINTER(HaloPlan)], I),
        "coarse_dslash_apply_chain": ([P, P, P, I, I, P], I),
        "coarse_field_bytes_mrhs": ([P, I, I], SZ),
        "coarse_field_alloc_mrhs": ([P, I, I, P, SZ, PP], I),
        "coarse_dslash_apply_mrhs": ([P, P, P, I, P], I),
        "coarse_links_compress_hermitian": ([P, ctypes.POINTER(ctypes.c_double), P, PP], I),
        "coarse_field_bytes_parity": ([P, I], SZ),
        "coarse_field_alloc_parity": ([P, I, I, P, SZ, PP], I),
        "coarse_links_prepare_eo": ([P, P, PP], I),
        "coarse_dslash_apply_eo": ([P, P, P, I, P], I),
        "coarse_transfer_create": ([P, ctypes.POINTER(_TransferDesc), P, I, I, P, PP], I),
        "coarse_transfer_free": ([P], I),
        "coarse_transfer_fine_bytes": ([P], SZ),
        "coarse_transfer_read_basis": ([P, P, I, P], I),
        "coarse_transfer_orthonormalise": ([P, P], I),
        "coarse_restrict": ([P, P, P, P], I),
        "coarse_prolong": ([P, P, P, P], I),
        "cd_context_peer_handle": ([P, P], I),
        "cd_context_peer_connect": ([P, P, I], I),
        "coarse_halo_exchange": ([P, P, P, I, ctypes.POINTER(SZ), P], I),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    return lib


lib = _load()


def _check(rc):
    if rc != CD_OK:
        raise CDError(rc, lib.cd_last_error().decode())
    return rc


def default_stream(device=None):
    """The current torch CUDA stream handle of `device` (default: torch's current device);
    0 = legacy default stream if torch is unusable."""
    try:
        import torch
        if torch.cuda.is_available():
            return torch.cuda.current_stream(device).cuda_stream
    except Exception:
        pass
    return 0


def _stream(s, device=None):
    if s is None:
        return ctypes.c_void_p(default_stream(device))
    if hasattr(s, "cuda_stream"):
        return ctypes.c_void_p(s.cuda_stream)
    return ctypes.c_void_p(int(s))


def _ptr(x):
    """(pointer, on_device, keepalive) for numpy arrays, torch tensors or raw ints."""
    if isinstance(x, np.ndarray):
        if not x.flags.c_contiguous:
            raise ValueError("array must be C-contiguous")
        return x.ctypes.data, 0, x
    try:
        import torch
        if isinstance(x, torch.Tensor):
            if not x.is_contiguous():
                raise ValueError("tensor must be contiguous")
            return x.data_ptr(), 1 if x.is_cuda else 0, x
    except ImportError:
        pass
    return int(x), 1, None


# ------------------------------------------------------------------ C-ABI-named functions
def cd_version() -> str:
    return lib.cd_version().decode()


def cd_launch_count() -> int:
    return int(lib.cd_launch_count())


def cd_get_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(lib.cd_get_unique_id(buf))
    return bytes(buf)


def cd_context_create(global_dims, nvec, proc_grid=(1, 1, 1, 1), device=0, nranks=1, rank=0, nccl_id=None):
    g = _Geometry((ctypes.c_int32 * 4)(*global_dims), nvec, (ctypes.c_int32 * 4)(*proc_grid))
    out = ctypes.c_void_p()
    idb = None if nccl_id is None else (ctypes.c_uint8 * 128)(*nccl_id)
    _check(lib.cd_context_create(ctypes.byref(g), device, nranks, rank, idb, ctypes.byref(out)))
    return out


def cd_halo_plan_create(global_dims, nvec, proc_grid, rank, prec="fp32", self_mask=0) -> HaloPlan:
    """Host-only decomposition + halo layout of `rank` (no GPU needed)."""
    g = _Geometry((ctypes.c_int32 * 4)(*global_dims), nvec, (ctypes.c_int32 * 4)(*proc_grid))
    nranks = int(np.prod(proc_grid))
    out = HaloPlan()
    _check(lib.cd_halo_plan_create(ctypes.byref(g), nranks, rank, PREC[prec], self_mask, ctypes.byref(out)))
    return out


def coarse_field_alloc(ctx, prec, device_mem=None, nbytes=0):
    out = ctypes.c_void_p()
    _check(lib.coarse_field_alloc(ctx, PREC[prec], device_mem, nbytes, ctypes.byref(out)))
    return out


def coarse_links_upload(ctx, prec, links, stream=None):
    """links: canonical LOCAL [V, 9, N, N] complex128/complex64 (numpy or torch)."""
    p, dev, keep = _ptr(links)
    out = ctypes.c_void_p()
    _check(lib.coarse_links_upload(ctx, PREC[prec], p, dev, CD_C128 if _is_c128(links) else CD_C64,
                                   _stream(stream), ctypes.byref(out)))
    del keep
    return out


def _is_c128(x):
    if isinstance(x, np.ndarray):
        if x.dtype == np.complex128:
            return True
        if x.dtype == np.complex64:
            return False
        raise TypeError(f"expected complex64/complex128, got {x.dtype}")
    import torch
    if x.dtype == torch.complex128:
        return True
    if x.dtype == torch.complex64:
        return False
    raise TypeError(f"expected complex64/complex128, got {x.dtype}")


def coarse_links_generate(ctx, prec, kind="general", seed=0x1612, scale_log2=0, stream=None):
    out = ctypes.c_void_p()
    k = LINK_KIND[kind] if isinstance(kind, str) else int(kind)
    _check(lib.coarse_links_generate(ctx, PREC[prec], k, seed, scale_log2, _stream(stream), ctypes.byref(out)))
    return out


def coarse_dslash_apply(links, out, in_, stream=None, device=None):
    _check(lib.coarse_dslash_apply(links, out, in_, _stream(stream, device)))


def coarse_dslash_apply_dagger(links, out, in_, stream=None, device=None):
    _check(lib.coarse_dslash_apply_dagger(links, out, in_, _stream(stream, device)))


def coarse_dslash_apply_chain(links, x, y, n, dagger=False, stream=None, device=None):
    """n chained applies in one persistent kernel: t even y = D x, t odd x = D y."""
    _check(lib.coarse_dslash_apply_chain(links, x, y, int(n), int(bool(dagger)), _stream(stream, device)))


# ------------------------------------------------------------------ classes
class Context:
    """A lattice geometry on one GPU (one rank of a process grid)."""

    def __init__(self, global_dims, nvec, proc_grid=(1, 1, 1, 1), device=0, nranks=1, rank=0, nccl_id=None):
        self.global_dims = tuple(int(x) for x in global_dims)
        self.nvec = int(nvec)
        self.N = 2 * self.nvec
        self.proc_grid = tuple(int(x) for x in proc_grid)
        self.device = int(device)
        self.handle = cd_context_create(self.global_dims, self.nvec, self.proc_grid, device, nranks, rank, nccl_id)
        ld = (ctypes.c_int32 * 4)()
        gc = (ctypes.c_int32 * 4)()
        vol = ctypes.c_int64()
        _check(lib.cd_context_local(self.handle, ld, ctypes.byref(vol), gc))
        self.local_dims = tuple(ld)
        self.grid_coords = tuple(gc)
        self.V = int(vol.value)
        self._objs = []

    def set_option(self, option, value):
        _check(lib.cd_context_set_option(self.handle, option, int(value)))

    def variants(self, prec):
        p = PREC[prec]
        return [lib.cd_variant_name(self.handle, p, i).decode() for i in range(lib.cd_variant_count(self.handle, p))]

    def chosen_variant(self, prec, dagger=False):
        return lib.cd_context_chosen_variant(self.handle, PREC[prec], int(bool(dagger)))

    def chosen_chain_variant(self, prec, dagger=False):
        """apply_chain's tuned variant id (see cd_context_chosen_variant), -1 if not tuned yet."""
        return lib.cd_context_chosen_variant(self.handle, PREC[prec], 2 + int(bool(dagger)))

    def field(self, prec="fp32", torch_memory=True, nrhs=1, parity=None):
        return Field(self, prec, torch_memory, nrhs, parity)

    def links_upload(self, links, prec="fp32", stream=None):
        return Links(self, prec, coarse_links_upload(self.handle, prec, np.ascontiguousarray(links)
                                                     if isinstance(links, np.ndarray) else links, stream))

    def links_generate(self, prec="fp32", kind="general", seed=0x1612, scale_log2=0, stream=None):
        return Links(self, prec, coarse_links_generate(self.handle, prec, kind, seed, scale_log2, stream))

    def set_transport(self, name):
        """Halo transport: "auto", "nccl", "peer" or "copy" (CD_OPT_TRANSPORT)."""
        self.set_option(CD_OPT_TRANSPORT, TRANSPORT[name] if isinstance(name, str) else int(name))

    def peer_handle(self) -> bytes:
        """Allocate + export this rank's peer window (64-byte CUDA IPC handle)."""
        buf = (ctypes.c_uint8 * 64)()
        _check(lib.cd_context_peer_handle(self.handle, buf))
        return bytes(buf)

    def peer_connect(self, handles):
        """Map the neighbours' windows; handles: the 64-byte handles of ranks 0..nranks-1."""
        blob = b"".join(bytes(h) for h in handles)
        buf = (ctypes.c_uint8 * len(blob)).from_buffer_copy(blob)
        _check(lib.cd_context_peer_connect(self.handle, buf, len(handles)))

    def connect_peers(self, group=None):
        """Collective: exchange peer-window handles over torch.distributed and connect."""
        import torch.distributed as dist
        h = self.peer_handle()
        allh = [None] * dist.get_world_size(group)
        dist.all_gather_object(allh, h, group=group)
        self.peer_connect(allh)

    def halo_exchange(self, field, stream=None, copy_out=True) -> bytes:
        """One halo exchange of `field` (pack + transport + arrival wait); returns the received
        buffer in the DESIGN.md R13 wire order (collective)."""
        n = ctypes.c_size_t()
        if not copy_out:
            _check(lib.coarse_halo_exchange(self.handle, field.handle, None, 0, ctypes.byref(n),
                                            _stream(stream, self.device)))
            return b""
        _check(lib.coarse_halo_pack(self.handle, field.handle, None, 0, ctypes.byref(n), _stream(stream, self.device)))
        buf = np.zeros(max(n.value, 16), np.uint8)
        _check(lib.coarse_halo_exchange(self.handle, field.handle, buf.ctypes.data, 0, ctypes.byref(n),
                                        _stream(stream, self.device)))
        return buf[:n.value].tobytes()

    def halo_pack(self, field, stream=None) -> bytes:
        n = ctypes.c_size_t()
        _check(lib.coarse_halo_pack(self.handle, field.handle, None, 0, ctypes.byref(n), _stream(stream, self.device)))
        buf = np.zeros(max(n.value, 1), np.uint8)
        if n.value:
            _check(lib.coarse_halo_pack(self.handle, field.handle, buf.ctypes.data, 0, ctypes.byref(n),
                                        _stream(stream, self.device)))
        return buf[:n.value].tobytes()

    def transfer(self, block, nspin, ncolor, basis, stream=None):
        """Prolongator / restrictor for aggregates `block` of a fine grid with nspin x ncolor dofs per
        site; basis: complex [Vf, nspin, ncolor, Nvec] (numpy or torch, host or device)."""
        return Transfer(self, block, nspin, ncolor, basis, stream)

    def flush_l2(self, nbytes=512 << 20, stream=None):
        _check(lib.cd_flush_l2(self.handle, nbytes, _stream(stream, self.device)))

    def close(self):
        if self.handle:
            _check(lib.cd_context_destroy(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Field:
    """A colour-spinor field in the library's stored layout (device memory from torch)."""

    def __init__(self, ctx: Context, prec="fp32", torch_memory=True, nrhs=1, parity=None):
        self.ctx = ctx
        self.prec = PREC[prec]
        self.nrhs = int(nrhs)
        self.parity = parity
        self.sites = ctx.V if parity is None else ctx.V // 2
        self.nbytes = int(lib.coarse_field_bytes_mrhs(ctx.handle, self.prec, self.nrhs) if parity is None
                          else lib.coarse_field_bytes_parity(ctx.handle, self.prec))
        self._mem = None
        ptr = None
        if torch_memory:
            import torch
            self._mem = torch.empty(self.nbytes, dtype=torch.uint8, device=f"cuda:{ctx.device}")
            ptr = self._mem.data_ptr()
        if parity is not None:
            out = ctypes.c_void_p()
            _check(lib.coarse_field_alloc_parity(ctx.handle, self.prec, int(parity), ptr, self.nbytes if ptr else 0,
                                                 ctypes.byref(out)))
            self.handle = out
        elif self.nrhs == 1:
            self.handle = coarse_field_alloc(ctx.handle, self.prec, ptr, self.nbytes if ptr else 0)
        else:
            out = ctypes.c_void_p()
            _check(lib.coarse_field_alloc_mrhs(ctx.handle, self.prec, self.nrhs, ptr, self.nbytes if ptr else 0,
                                               ctypes.byref(out)))
            self.handle = out

    def import_(self, v, stream=None):
        """v: canonical LOCAL [V, N] complex64/complex128 (numpy host or torch host/device)."""
        p, dev, keep = _ptr(v)
        _check(lib.coarse_field_import(self.handle, p, dev, CD_C128 if _is_c128(v) else CD_C64, _stream(stream, self.ctx.device)))
        return keep

    def export(self, dst=None, dtype=np.complex128, stream=None, sync=True):
        if dst is None:
            shape = (self.sites, self.ctx.N) if self.nrhs == 1 else (self.nrhs, self.sites, self.ctx.N)
            dst = np.empty(shape, dtype)
        p, dev, _ = _ptr(dst)
        _check(lib.coarse_field_export(self.handle, p, dev, CD_C128 if _is_c128(dst) else CD_C64, _stream(stream, self.ctx.device)))
        if sync:
            _sync(stream)
        return dst

    def generate(self, seed=0x7873, tag=2, scale_log2=0, stream=None):
        _check(lib.coarse_field_generate(self.handle, seed, tag, scale_log2, _stream(stream, self.ctx.device)))

    def read_stored(self, stream=None) -> bytes:
        n = int(lib.coarse_field_stored_bytes(self.handle))
        buf = np.empty(n, np.uint8)
        _check(lib.coarse_field_read_stored(self.handle, buf.ctypes.data, 0, _stream(stream, self.ctx.device)))
        return buf.tobytes()

    def close(self):
        if self.handle:
            _check(lib.coarse_field_free(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Links:
    """An immutable link set (9 matrices per site) in the library's stored layout."""

    def __init__(self, ctx: Context, prec, handle):
        self.ctx = ctx
        self.prec = PREC[prec]
        self.handle = handle

    def apply(self, out: Field, in_: Field, stream=None):
        coarse_dslash_apply(self.handle, out.handle, in_.handle, stream, self.ctx.device)

    def apply_dagger(self, out: Field, in_: Field, stream=None):
        coarse_dslash_apply_dagger(self.handle, out.handle, in_.handle, stream, self.ctx.device)

    def apply_chain(self, x: Field, y: Field, n: int, dagger=False, stream=None):
        coarse_dslash_apply_chain(self.handle, x.handle, y.handle, n, dagger, stream, self.ctx.device)

    def prepare_eo(self, stream=None):
        """Even-odd preconditioned operator (X_o^-1 L_k(o) precomputed); returns new Links."""
        out = ctypes.c_void_p()
        _check(lib.coarse_links_prepare_eo(self.handle, _stream(stream), ctypes.byref(out)))
        return Links(self.ctx, self.prec, out)

    def apply_eo(self, out: Field, in_: Field, dagger=False, stream=None):
        """out_e = M_ee in_e (Schur complement on even sites; parity-0 fields)."""
        _check(lib.coarse_dslash_apply_eo(self.handle, out.handle, in_.handle, int(bool(dagger)), _stream(stream, self.ctx.device)))

    def compress_hermitian(self, check=True, stream=None):
        """tau3-hermitian compressed copy (X + 4 forward links per site); returns (Links, max_dev)."""
        dev = ctypes.c_double(-1.0)
        out = ctypes.c_void_p()
        _check(lib.coarse_links_compress_hermitian(self.handle, ctypes.byref(dev) if check else None,
                                                   _stream(stream), ctypes.byref(out)))
        return Links(self.ctx, self.prec, out), (dev.value if check else None)

    def apply_mrhs(self, out: Field, in_: Field, dagger=False, stream=None):
        """out_r = D in_r for all right-hand sides (tcgen05 tensor cores, fp16 storage)."""
        _check(lib.coarse_dslash_apply_mrhs(self.handle, out.handle, in_.handle, int(bool(dagger)), _stream(stream, self.ctx.device)))

    def read_stored(self, stream=None) -> bytes:
        n = int(lib.coarse_links_stored_bytes(self.handle))
        buf = np.empty(n, np.uint8)
        _check(lib.coarse_links_read_stored(self.handle, buf.ctypes.data, 0, _stream(stream, self.ctx.device)))
        return buf.tobytes()

    def close(self):
        if self.handle:
            _check(lib.coarse_links_free(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Transfer:
    """P and R = P^dagger between a fine lattice (local dims x block) and this context's lattice."""

    def __init__(self, ctx: Context, block, nspin, ncolor, basis, stream=None):
        self.ctx = ctx
        self.block = tuple(int(b) for b in block)
        self.nspin, self.ncolor = int(nspin), int(ncolor)
        self.fine_dims = tuple(l * b for l, b in zip(ctx.local_dims, self.block))
        self.Vf = int(np.prod(self.fine_dims))
        d = _TransferDesc((ctypes.c_int32 * 4)(*self.block), self.nspin, self.ncolor)
        if isinstance(basis, np.ndarray):
            basis = np.ascontiguousarray(basis)
        p, dev, keep = _ptr(basis)
        out = ctypes.c_void_p()
        _check(lib.coarse_transfer_create(ctx.handle, ctypes.byref(d), p, dev, CD_C128 if _is_c128(basis) else CD_C64,
                                          _stream(stream), ctypes.byref(out)))
        _sync(stream)
        del keep
        self.handle = out

    def fine_field(self):
        """A device complex64 fine field [Vf, nspin, ncolor] (torch)."""
        import torch
        return torch.zeros((self.Vf, self.nspin, self.ncolor), dtype=torch.complex64, device=f"cuda:{self.ctx.device}")

    def orthonormalise(self, stream=None):
        _check(lib.coarse_transfer_orthonormalise(self.handle, _stream(stream, self.ctx.device)))

    def read_basis(self, stream=None):
        out = np.empty((self.Vf, self.nspin, self.ncolor, self.ctx.nvec), np.complex64)
        _check(lib.coarse_transfer_read_basis(self.handle, out.ctypes.data, 0, _stream(stream, self.ctx.device)))
        return out

    def restrict(self, coarse_out: Field, fine_in, stream=None):
        """coarse_out = P^dagger fine_in (fine_in: device complex64 [Vf, nspin, ncolor])."""
        p, dev, _ = _ptr(fine_in)
        if not dev:
            raise ValueError("fine_in must be device memory")
        _check(lib.coarse_restrict(self.handle, coarse_out.handle, p, _stream(stream, self.ctx.device)))

    def prolong(self, fine_out, coarse_in: Field, stream=None):
        """fine_out = P coarse_in (fine_out: device complex64 [Vf, nspin, ncolor])."""
        p, dev, _ = _ptr(fine_out)
        if not dev:
            raise ValueError("fine_out must be device memory")
        _check(lib.coarse_prolong(self.handle, p, coarse_in.handle, _stream(stream, self.ctx.device)))

    def close(self):
        if self.handle:
            _check(lib.coarse_transfer_free(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _sync(stream=None):
    try:
        import torch
        if torch.cuda.is_available():
            if stream is None:
                torch.cuda.current_stream().synchronize()
            elif hasattr(stream, "synchronize"):
                stream.synchronize()
            else:
                torch.cuda.synchronize()
    except ImportError:
        pass
