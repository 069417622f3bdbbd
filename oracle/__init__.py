"""float64 CPU oracle of the coarse-grid Dirac operator (ctypes wrapper over oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The product
(``paper_1612_07873_b200``) never imports it and shares no code with it.

Every function follows PAPER.md §3.4 Eq. 3 as read in DESIGN.md
(R1-R13); see the C source header for the term-by-term definition and the list of pins.
Arrays are numpy complex128 in the canonical layout:
    links [V, 9, N, N]   (k = 2*mu + dir, k = 8 the diagonal X)
    v, y  [V, N]         (site index x0 fastest; dof i = spin*Nvec + colour)
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (plain gcc, -O2 -fopenmp, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-std=gnu11", "-O2", "-fopenmp", "-fPIC", "-shared", "-fno-fast-math",
               "-ffp-contract=off", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            P = ctypes.c_void_p
            I4 = ctypes.POINTER(ctypes.c_int)
            lib.oracle_apply.argtypes = [I4, ctypes.c_int, P, P, P]
            lib.oracle_apply_dagger_tau3.argtypes = [I4, ctypes.c_int, P, P, P]
            lib.oracle_apply_generated.argtypes = [I4, ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_int, P, P]
            lib.oracle_apply_generated.restype = ctypes.c_int
            lib.oracle_set_threads.argtypes = [ctypes.c_int]
            lib.oracle_get_threads.restype = ctypes.c_int
            lib.oracle_adjoint.argtypes = [I4, ctypes.c_int, P, P, P]
            lib.oracle_dense.argtypes = [I4, ctypes.c_int, P, P]
            lib.oracle_partitioned_apply.argtypes = [I4, I4, ctypes.c_int, P, P, P]
            lib.oracle_pack_halo.argtypes = [I4, I4, P, ctypes.c_size_t, P, ctypes.c_size_t, P]
            lib.oracle_pack_halo.restype = ctypes.c_size_t
            lib.oracle_neighbours.argtypes = [I4, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)]
            lib.oracle_site_apply.argtypes = [ctypes.c_int, P, P, P]
            lib.oracle_quantise_fp16.argtypes = [ctypes.c_int64, ctypes.c_int64, P, P, P]
            lib.oracle_dequantise_fp16.argtypes = [ctypes.c_int64, ctypes.c_int64, P, P, P]
            lib.oracle_invert.argtypes = [ctypes.c_int, P, P]
            lib.oracle_schur_apply.argtypes = [I4, ctypes.c_int, P, P, P]
            CI = ctypes.c_int
            lib.oracle_prolong.argtypes = [I4, I4, CI, CI, CI, P, P, P]
            lib.oracle_restrict.argtypes = [I4, I4, CI, CI, CI, P, P, P]
            lib.oracle_block_orthonormalise.argtypes = [I4, I4, CI, CI, CI, P]
            _lib = lib
    return _lib


def _dims(d):
    d = [int(x) for x in d]
    if len(d) != 4 or min(d) < 1:
        raise ValueError(f"dims must be 4 positive ints, got {d}")
    return (ctypes.c_int * 4)(*d)


def _c128(a, shape):
    a = np.ascontiguousarray(a, dtype=np.complex128)
    if a.size != int(np.prod(shape)):
        raise ValueError(f"expected {shape}, got {a.shape}")
    return a


def _geom(dims, links):
    V = int(np.prod(dims))
    N = links.shape[-1]
    return V, N


def apply(dims, links, v):
    """y = D v (Eq. 3; R1-R3, R10)."""
    V, N = _geom(dims, links)
    L = _c128(links, (V, 9, N, N))
    x = _c128(v, (V, N))
    y = np.empty((V, N), np.complex128)
    _load().oracle_apply(_dims(dims), N, L.ctypes.data, x.ctypes.data, y.ctypes.data)
    return y


def set_threads(n: int) -> None:
    """OpenMP threads of the oracle's site loops (timing only)."""
    _load().oracle_set_threads(int(n))


def get_threads() -> int:
    return int(_load().oracle_get_threads())


KINDS = {"general": 0, "hermitian": 1, "ti_general": 2, "ti_hermitian": 3}


def apply_generated(dims, N, v, kind="general", seed=0x1612, scale_log2=0):
    """Matrix-free y = D v: the links of recipe `kind` (synth.links(dims, N, seed, kind,
    scale_log2)) are regenerated per site instead of being passed in, so whole
    full-size lattices need memory for the vectors only.  Same term order as
    apply(): bit-identical to apply(dims, synth.links(...), v) (pinned)."""
    V = int(np.prod(dims))
    v = _c128(v, (V, N))
    y = np.empty((V, N), np.complex128)
    rc = _load().oracle_apply_generated(_dims(dims), int(N), KINDS[kind], int(seed) & 0xFFFFFFFFFFFFFFFF,
                                        int(scale_log2), v.ctypes.data, y.ctypes.data)
    if rc != 0:
        raise ValueError(f"oracle_apply_generated failed ({rc})")
    return y


def apply_dagger_tau3(dims, links, w):
    """y = tau3 D tau3 w (R5; PAPER.md:121 footnote 1)."""
    V, N = _geom(dims, links)
    L = _c128(links, (V, 9, N, N))
    x = _c128(w, (V, N))
    y = np.empty((V, N), np.complex128)
    _load().oracle_apply_dagger_tau3(_dims(dims), N, L.ctypes.data, x.ctypes.data, y.ctypes.data)
    return y


def adjoint(dims, links, w):
    """y = D^H w (true adjoint, from its definition)."""
    V, N = _geom(dims, links)
    L = _c128(links, (V, 9, N, N))
    x = _c128(w, (V, N))
    y = np.empty((V, N), np.complex128)
    _load().oracle_adjoint(_dims(dims), N, L.ctypes.data, x.ctypes.data, y.ctypes.data)
    return y


def dense(dims, links):
    """Dense D in C^{VN x VN} assembled block by block with += (tiny lattices only)."""
    V, N = _geom(dims, links)
    if V * N > 8192:
        raise ValueError("dense oracle is for tiny lattices")
    L = _c128(links, (V, 9, N, N))
    D = np.empty((V * N, V * N), np.complex128)
    _load().oracle_dense(_dims(dims), N, L.ctypes.data, D.ctypes.data)
    return D


def partitioned_apply(dims, proc_grid, links, v):
    """Emulated multi-rank apply with explicit halo buffers (must equal apply bit-for-bit)."""
    V, N = _geom(dims, links)
    for mu in range(4):
        if dims[mu] % proc_grid[mu]:
            raise ValueError("dims must be divisible by proc_grid")
    L = _c128(links, (V, 9, N, N))
    x = _c128(v, (V, N))
    y = np.empty((V, N), np.complex128)
    _load().oracle_partitioned_apply(_dims(dims), _dims(proc_grid), N, L.ctypes.data, x.ctypes.data,
                                     y.ctypes.data)
    return y


def pack_halo(local_dims, split, payload, rec_bytes, scales=None, scale_bytes=0) -> bytes:
    """Byte-exact canonical halo send buffer (R13) of a local field.

    payload: contiguous array of V records of rec_bytes each; scales: optional V records of
    scale_bytes each (fp16 storage)."""
    lib = _load()
    d = _dims(local_dims)
    sp = (ctypes.c_int * 4)(*[1 if s else 0 for s in split])
    p = np.ascontiguousarray(payload)
    sc = None if scales is None else np.ascontiguousarray(scales)
    n = lib.oracle_pack_halo(d, sp, p.ctypes.data, rec_bytes, None if sc is None else sc.ctypes.data,
                             scale_bytes, None)
    out = np.empty(max(n, 1), np.uint8)
    lib.oracle_pack_halo(d, sp, p.ctypes.data, rec_bytes, None if sc is None else sc.ctypes.data,
                         scale_bytes, out.ctypes.data)
    return out[:n].tobytes()


def neighbours(dims, s: int):
    """Site indices of the 9 vectors multiplying L_0..L_8 at site s (k = 8: s itself)."""
    out = (ctypes.c_int64 * 9)()
    _load().oracle_neighbours(_dims(dims), int(s), out)
    return list(out)


def site_apply(links9, vnbr):
    """y(x) from the site's 9 matrices [9,N,N] and the 9 vectors they multiply [9,N]."""
    L = np.ascontiguousarray(links9, dtype=np.complex128)
    u = np.ascontiguousarray(vnbr, dtype=np.complex128)
    N = L.shape[-1]
    y = np.empty(N, np.complex128)
    _load().oracle_site_apply(N, L.ctypes.data, u.ctypes.data, y.ctypes.data)
    return y


def quantise_fp16(x, reals_per_rec: int):
    """16-bit storage emulation (R12): returns (uint16 payload, float32 scales)."""
    xr = np.ascontiguousarray(x).view(np.float64).reshape(-1)
    if xr.size % reals_per_rec:
        raise ValueError("size not a multiple of the record length")
    nrec = xr.size // reals_per_rec
    q = np.empty(xr.size, np.uint16)
    s = np.empty(nrec, np.float32)
    _load().oracle_quantise_fp16(nrec, reals_per_rec, xr.ctypes.data, q.ctypes.data, s.ctypes.data)
    return q, s


def dequantise_fp16(q, s, reals_per_rec: int):
    q = np.ascontiguousarray(q, dtype=np.uint16).reshape(-1)
    s = np.ascontiguousarray(s, dtype=np.float32).reshape(-1)
    x = np.empty(q.size, np.float64)
    _load().oracle_dequantise_fp16(s.size, reals_per_rec, q.ctypes.data, s.ctypes.data, x.ctypes.data)
    return x.view(np.complex128)


def invert(A):
    """N x N complex inverse by Gauss-Jordan with partial pivoting (fp64)."""
    A = np.ascontiguousarray(A, dtype=np.complex128)
    N = A.shape[0]
    out = np.empty_like(A)
    if _load().oracle_invert(N, A.ctypes.data, out.ctypes.data) != 0:
        raise ValueError("singular matrix")
    return out


def parity(dims):
    """Site parity (x0+x1+x2+x3) mod 2 of every site, canonical order."""
    V = int(np.prod(dims))
    s = np.arange(V)
    x0 = s % dims[0]; s1 = s // dims[0]
    x1 = s1 % dims[1]; s2 = s1 // dims[1]
    x2 = s2 % dims[2]; x3 = s2 // dims[2]
    return (x0 + x1 + x2 + x3) & 1


def schur_apply(dims, links, v):
    """Even-odd Schur complement y_e = X_e v_e - D_eo X_o^-1 D_oe v_e on FULL fields (only even
    sites read / written; odd sites of y are 0).  PAPER.md:95 §3.3."""
    if any(int(d) % 2 for d in dims):
        raise ValueError("even-odd needs every L_mu even")
    V, N = _geom(dims, links)
    L = _c128(links, (V, 9, N, N))
    x = _c128(v, (V, N))
    y = np.empty((V, N), np.complex128)
    if _load().oracle_schur_apply(_dims(dims), N, L.ctypes.data, x.ctypes.data, y.ctypes.data) != 0:
        raise ValueError("singular X on an odd site")
    return y


# ---------------------------------------------------------------- transfer operators
# Fine lattice = coarse dims x block B; fine field [Vf, Ns, Nc]; basis W [Vf, Ns, Nc, Nvec];
# coarse field [Vc, 2*Nvec] (§3.4; §6.6; R20).
def fine_dims(cdims, block):
    return tuple(int(c) * int(b) for c, b in zip(cdims, block))


def prolong(cdims, block, Ns, Nc, Nvec, W, vc):
    """vf = P vc (gather per fine dof)."""
    Vf, Vc = int(np.prod(fine_dims(cdims, block))), int(np.prod(cdims))
    Wc = _c128(W, (Vf, Ns, Nc, Nvec))
    x = _c128(vc, (Vc, 2 * Nvec))
    out = np.empty((Vf, Ns, Nc), np.complex128)
    _load().oracle_prolong(_dims(cdims), _dims(block), Ns, Nc, Nvec, Wc.ctypes.data, x.ctypes.data, out.ctypes.data)
    return out


def restrict(cdims, block, Ns, Nc, Nvec, W, vf):
    """vc = P^dagger vf (restrictor = hermitian conjugate of the prolongator)."""
    Vf, Vc = int(np.prod(fine_dims(cdims, block))), int(np.prod(cdims))
    Wc = _c128(W, (Vf, Ns, Nc, Nvec))
    x = _c128(vf, (Vf, Ns, Nc))
    out = np.empty((Vc, 2 * Nvec), np.complex128)
    _load().oracle_restrict(_dims(cdims), _dims(block), Ns, Nc, Nvec, Wc.ctypes.data, x.ctypes.data, out.ctypes.data)
    return out


def block_orthonormalise(cdims, block, Ns, Nc, Nvec, W):
    """Per (aggregate, chirality) block: Q of the QR decomposition by modified Gram-Schmidt."""
    Vf = int(np.prod(fine_dims(cdims, block)))
    Wc = _c128(W, (Vf, Ns, Nc, Nvec)).copy()
    if _load().oracle_block_orthonormalise(_dims(cdims), _dims(block), Ns, Nc, Nvec, Wc.ctypes.data) != 0:
        raise ValueError("rank-deficient aggregate block")
    return Wc
