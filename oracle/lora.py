"""ORACLE ONLY — ctypes over oracle/liboracle.so (lora_oracle.c): the CPU
restatement of the paged LoRA apply, y_t += scale·(x_t·Aᵀ)·Bᵀ with every
weight read through the adapter's page table (PAPER.md:64-69,
src/memory.cpp:55-62).  bf16 tensors travel as uint16 numpy arrays."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
MAX_PROJ = 8

_lib = None


class OracleModel(C.Structure):
    _fields_ = [("n_layers", C.c_uint32), ("n_proj", C.c_uint32),
                ("d_in", C.c_uint32 * MAX_PROJ), ("d_out", C.c_uint32 * MAX_PROJ),
                ("esize", C.c_uint32)]


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            raise ImportError(f"{ORACLE_SO} missing: run `make -C oracle`")
        L = C.CDLL(ORACLE_SO)
        P = C.POINTER
        L.oracle_block_offset.restype = C.c_uint64
        L.oracle_block_offset.argtypes = [P(OracleModel), C.c_uint32, C.c_uint32, C.c_uint32]
        L.oracle_adapter_bytes.restype = C.c_uint64
        L.oracle_adapter_bytes.argtypes = [P(OracleModel), C.c_uint32]
        L.oracle_scatter_pages.restype = None
        L.oracle_scatter_pages.argtypes = [C.c_void_p, C.c_uint64, P(C.c_uint32), C.c_uint64,
                                           C.c_void_p, C.c_uint64]
        L.oracle_gather_pages.restype = None
        L.oracle_gather_pages.argtypes = [C.c_void_p, C.c_uint64, P(C.c_uint32), C.c_uint64,
                                          C.c_void_p, C.c_uint64]
        L.oracle_paged_lora_apply.restype = C.c_int
        L.oracle_paged_lora_apply.argtypes = [
            P(OracleModel), C.c_void_p, C.c_uint64, P(C.c_uint32), P(C.c_uint64), P(C.c_uint32),
            C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p, P(C.c_int32), C.c_uint32,
            C.c_float, C.c_int, C.c_int]
        L.oracle_f32_to_bf16.restype = C.c_uint16
        L.oracle_f32_to_bf16.argtypes = [C.c_float]
        L.oracle_bf16_to_f32.restype = C.c_float
        L.oracle_bf16_to_f32.argtypes = [C.c_uint16]
        _lib = L
    return _lib


def model(n_layers: int, d_in, d_out, esize: int) -> OracleModel:
    m = OracleModel()
    m.n_layers = n_layers
    m.n_proj = len(d_in)
    for i, (a, b) in enumerate(zip(d_in, d_out)):
        m.d_in[i] = a
        m.d_out[i] = b
    m.esize = esize
    return m


def adapter_bytes(m: OracleModel, rank: int) -> int:
    return lib().oracle_adapter_bytes(C.byref(m), rank)


def block_offset(m: OracleModel, rank: int, layer: int, proj: int) -> int:
    return lib().oracle_block_offset(C.byref(m), rank, layer, proj)


def _u32(a):
    a = np.ascontiguousarray(a, dtype=np.uint32)
    return a, a.ctypes.data_as(C.POINTER(C.c_uint32))


def scatter_pages(arena: np.ndarray, page_bytes: int, entries, src: np.ndarray) -> None:
    e, ep = _u32(entries)
    src = np.ascontiguousarray(src).view(np.uint8)
    lib().oracle_scatter_pages(arena.ctypes.data, page_bytes, ep, len(e), src.ctypes.data,
                               src.nbytes)


def gather_pages(arena: np.ndarray, page_bytes: int, entries, nbytes: int) -> np.ndarray:
    e, ep = _u32(entries)
    out = np.zeros(nbytes, np.uint8)
    lib().oracle_gather_pages(arena.ctypes.data, page_bytes, ep, len(e), out.ctypes.data, nbytes)
    return out


class PreparedTables:
    """Page tables flattened once for repeated calls: entries, per-adapter
    offsets into them, ranks."""

    def __init__(self, tables: dict[int, list[int]], ranks: dict[int, int]):
        self.n_adapters = max(list(ranks) + [-1]) + 1
        self.offs = np.zeros(self.n_adapters, np.uint64)
        self.rk = np.zeros(self.n_adapters, np.uint32)
        parts, pos = [], 0
        for a in range(self.n_adapters):
            self.offs[a] = pos
            if a in tables:
                t = np.asarray(tables[a], np.uint32)
                parts.append(t)
                pos += len(t)
                self.rk[a] = ranks[a]
        self.ent = np.ascontiguousarray(np.concatenate(parts) if parts else np.zeros(1, np.uint32))


def paged_lora_apply(m: OracleModel, arena: np.ndarray, page_bytes: int,
                     tables, ranks: dict[int, int] | None, layer: int, proj: int,
                     x: np.ndarray, y: np.ndarray, token_adapter, scale: float = 1.0,
                     v_bf16: bool = False, nthreads: int = 1) -> np.ndarray:
    """Updates y in place (and returns it).  x/y: uint16 (bf16 bits) when
    m.esize == 2, float32 when 4; rows = tokens.  `tables` is a dict of page
    tables (with `ranks`) or a PreparedTables."""
    pt = tables if isinstance(tables, PreparedTables) else PreparedTables(tables, ranks)
    ta = np.ascontiguousarray(np.asarray(token_adapter, np.int32))
    assert x.flags.c_contiguous and y.flags.c_contiguous
    rc = lib().oracle_paged_lora_apply(
        C.byref(m), arena.ctypes.data, page_bytes, pt.ent.ctypes.data_as(C.POINTER(C.c_uint32)),
        pt.offs.ctypes.data_as(C.POINTER(C.c_uint64)),
        pt.rk.ctypes.data_as(C.POINTER(C.c_uint32)), pt.n_adapters, layer, proj, x.ctypes.data,
        y.ctypes.data, ta.ctypes.data_as(C.POINTER(C.c_int32)), len(ta), scale,
        1 if v_bf16 else 0, nthreads)
    if rc != 0:
        raise ValueError("oracle rejected its arguments")
    return y


def bf16_bits_to_f32(a: np.ndarray) -> np.ndarray:
    return (a.astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16_bits(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even, as lora_oracle.c and the GPU do."""
    u = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    nan = (u & 0x7FFFFFFF) > 0x7F800000
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    r[nan] = ((u[nan] >> 16) | 0x40).astype(np.uint16)
    return r
