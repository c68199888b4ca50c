"""ctypes binding of libdrgraph_b200.so (the C ABI in include/drgraph_b200.h).

The extension is REQUIRED: there is no CPU fallback anywhere in this package.
If the shared library is missing or no CUDA device is visible, every compute
entry point raises.  ctypes releases the GIL for the duration of each foreign
call, so device work never holds the interpreter (the reference's nogil
contract, _kernels.py:48, test_optimizer.py:339-363).
"""

from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdrgraph_b200.so")
ABI_VERSION = 1

DRG_OK = 0
DRG_ERR_INVALID = -1
DRG_ERR_CUDA = -2
DRG_ERR_NONFINITE = -3
DRG_ERR_UNSUPPORTED = -4
DRG_ERR_NOMEM = -5
DRG_FLAG_INPLACE = 1
DRG_SAMPLED_AGGREGATE = 1
DRG_SAMPLED_FUSED = 2
DRG_SAMPLED_DETERMINISTIC = 4
DRG_SHARD_LAGGED = 1
DRG_SAMPLED_L2_HINTS = 8
DRG_SAMPLED_SRC_RECORDS = 16
DRG_SAMPLED_LOCKED = 32
DRG_SAMPLED_SNAPSHOT = 64

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int
_U32 = ctypes.c_uint
_U64 = ctypes.c_uint64
_F64 = ctypes.c_double

# name -> argtypes (every symbol include/drgraph_b200.h declares)
SIGNATURES = {
    "drg_abi_version": [],
    "drg_last_error": [],
    "drg_launch_count": [],
    "drg_khop_count": [_P, _P, _I64, _I32, _I64, _P, _P, _P],
    "drg_khop_fill": [_P, _P, _I64, _I32, _I64, _P, _P, _P, _P],
    "drg_gaussian_table": [_I32, _F64, _P, _P],
    "drg_rows_sigma": [_P, _P, _I64, _F64, _F64, _I32, _F64, _F64, _P, _P],
    "drg_rows_conditional": [_P, _P, _I64, _P, _P, _P],
    "drg_gradients": [_P, _P, _I64, _I32, _F64, _F64, _F64, _I32, _P, _P],
    "drg_shard_create": [_I32, _I32, _I64, _P],
    "drg_shard_destroy": [_P],
    "drg_shard_ipc_handle": [_P, _P],
    "drg_shard_open_peer": [_P, _I32, _P],
    "drg_nccl_unique_id": [_P],
    "drg_shard_nccl_init": [_P, _P],
    "drg_shard_level": [_P, _I64, _P, _P, _P, _P],
    "drg_shard_load": [_P, _P, _P],
    "drg_shard_store": [_P, _P, _P],
    "drg_shard_exchange": [_P, _P],
    "drg_shard_fold": [_P, _P, _P],
    "drg_shard_read_part": [_P, _P, _P],
    "drg_shard_epoch": [_P, _P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _F64, _P, _I32, _P, _P, _P, _P, _P, _I32, _I32,
                        _F64, _F64, _F64, _F64, _I32, _I32, _U64, _I32, _I64, _P, _P, _P],
    "drg_shard_run": [_P, _P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _F64, _P, _I32, _P, _P, _P, _P, _P, _I32, _I32,
                      _I32, _F64, _F64, _F64, _F64, _I32, _I32, _U64, _I32, _I64, _I32, _I32, _P, _P],
    "drg_khop_source": [_P, _P, _I64, _I32, _I64, _P, _P, _I64, _P, _P],
    "drg_similarity": [_P, _P, _P, _I64, _I64, _I32, _F64, _F64, _I32, _F64, _F64, _P, _P, _P,
                       _P, _P, _P],
    "drg_similarity_union": [_P, _P, _P, _I64, _I64, _I32, _F64, _F64, _I32, _F64, _F64, _P, _P,
                             _P, _P, _P, _P, _P, _P, _P],
    "drg_coarsen": [_P, _P, _I64, _P, _P, _P, _P, _P],
    "drg_coarse_graph": [_P, _P, _I64, _P, _I64, _P, _P, _P, _P],
    "drg_compose_maps": [_P, _P, _I64, _P, _P],
    "drg_aggregate_pairs": [_P, _P, _P, _I64, _I64, _P, _I64, _P, _P, _P, _P, _P],
    "drg_aggregate_nodes": [_P, _P, _I64, _I64, _P, _P],
    "drg_negative_weights": [_P, _I64, _F64, _P, _P],
    "drg_alias_build": [_P, _I64, _P, _P, _P],
    "drg_level_pack": [_P, _P, _P, _P, _P, _F64, _I64, _I64, _I32, _P, _P, _P],
    "drg_layout_iters": [_P, _P, _P, _P, _I64, _I64, _I64, _P, _P, _I32, _I32, _I32, _F64, _F64,
                         _F64, _F64, _I32, _I32, _U64, _I32, _P, _P, _P, _U32, _P],
    "drg_row_alias": [_P, _P, _P, _I64, _I64, _P, _P, _P],
    "drg_layout_sampled": [_P, _P, _P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _F64, _P, _I64, _I64, _I32, _I32, _I32,
                           _F64, _F64, _F64, _F64, _I32, _I32, _U64, _I32, _I64, _I32, _I64, _P,
                           _P, _I32, _P],
    "drg_sampled_draws": [_P, _P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _F64, _I64, _I64, _I32, _I32, _I32, _U64, _I32,
                          _P, _P],
    "drg_row_spans": [_P, _I64, _P, _P],
    "drg_src_records": [_P, _I64, _P, _P, _P, _P],
    "drg_sampled_apply": [_P, _I64, _P, _F64, _F64, _F64, _F64, _I32, _I32, _I64, _I32, _P],
    "drg_text_lines": [_P, _I64, _I32, _P, _P, _P, _P],
    "drg_parse_lines": [_P, _I64, _P, _I64, _I32, _I64, _I64, _P, _P, _P, _P, _P, _P],
    "drg_id_remap": [_P, _I64, _I32, _P, _P],
    "drg_format_coords": [_P, _I64, _P, _P, _P, _P],
    "drg_format_edge_list": [_P, _P, _I64, _I64, _P, _P, _P],
    "drg_bbox2": [_P, _I64, _P, _P],
    "drg_format_svg": [_P, _I64, _P, _I64, _F64, _F64, _F64, _F64, _F64, _F64, ctypes.c_char_p,
                       ctypes.c_char_p, _P, _P, _P, _P, _P, _P],
    "drg_layout_sgather": [_P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _P, _P, _I32, _I32, _I32,
                           _F64, _F64, _F64, _F64, _I32, _I32, _I32, _U64, _I32, _P, _P, _U32,
                           _P],
    "drg_layout_radius": [_P, _I64, _P, _P],
    "drg_prolong": [_P, _P, _I64, _F64, _U64, _P, _P],
    "drg_kl_terms": [_P, _P, _P, _I64, _P, _I32, _I64, _U64, _P, _P],
    "drg_neighborhood_preservation": [_P, _I64, _P, _P, _P, _I64, _P, _P],
    "drg_from_edges": [_P, _I64, _I64, _P, _P, _P, _P],
    "drg_components": [_P, _P, _I64, _P, _P, _P],
    "drg_pcg64_permutation": [_U64, _U64, _U64, _U64, _I32, _U32, _I64, _P],
}
RESTYPES = {"drg_last_error": ctypes.c_char_p, "drg_launch_count": ctypes.c_uint64}

DRG_HEAVY_CHUNK = 2048


class HeavySplit(ctypes.Structure):
    """drg_heavy_split (include/drgraph_b200.h)."""
    _fields_ = [("slot", ctypes.c_void_p), ("chunk_ptr", ctypes.c_void_p),
                ("chunk_row", ctypes.c_void_p), ("chunk_begin", ctypes.c_void_p),
                ("n_chunks", ctypes.c_int64), ("partial", ctypes.c_void_p)]


_lib = None


class ExtensionMissing(RuntimeError):
    """libdrgraph_b200.so is not built or cannot be loaded."""


def load(require_cuda: bool = True):
    """Load the extension (built by __graft_entry__.build() / make -C csrc)."""
    global _lib
    if require_cuda and not torch.cuda.is_available():
        raise RuntimeError("paper_2008_07799_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU path")
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ExtensionMissing(f"{LIB_PATH} is missing: run `python -c 'import "
                                   f"__graft_entry__ as g; g.build()'` (no CPU fallback)")
        try:
            lib = ctypes.CDLL(LIB_PATH)
        except OSError as e:  # pragma: no cover - environment specific
            raise ExtensionMissing(f"cannot load {LIB_PATH}: {e}") from e
        for name, args in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = RESTYPES.get(name, ctypes.c_int)
        if lib.drg_abi_version() != ABI_VERSION:
            raise ExtensionMissing(f"ABI version mismatch: {lib.drg_abi_version()} "
                                   f"!= {ABI_VERSION}")
        _lib = lib
    return _lib


def check(rc: int, what: str = "") -> None:
    """Map a DRG status to the reference's exception types."""
    if rc == DRG_OK:
        return
    msg = (_lib.drg_last_error() or b"").decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == DRG_ERR_INVALID:
        raise ValueError(text)
    if rc == DRG_ERR_NONFINITE:
        raise FloatingPointError(text)
    if rc == DRG_ERR_NOMEM:
        raise MemoryError(text)
    raise RuntimeError(f"{text} (status {rc})")


def call(name: str, *args) -> None:
    lib = load()
    check(getattr(lib, name)(*args), name)


def call_host(name: str, *args) -> None:
    """A host-only entry point (no device work): loads without requiring CUDA."""
    lib = load(require_cuda=False)
    check(getattr(lib, name)(*args), name)


def ptr(t: torch.Tensor | None):
    if t is None:
        return None
    assert t.is_cuda and t.is_contiguous(), "expected a contiguous CUDA tensor"
    return ctypes.c_void_p(t.data_ptr())


def stream_ptr(stream: torch.cuda.Stream | None = None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def launch_count() -> int:
    return int(load(require_cuda=False).drg_launch_count())


class HostInt64(ctypes.c_int64):
    pass


def out_i32() -> ctypes.c_int32:
    return ctypes.c_int32(0)


def out_i64() -> ctypes.c_int64:
    return ctypes.c_int64(0)


def out_f64() -> ctypes.c_double:
    return ctypes.c_double(0.0)


def byref(x):
    return ctypes.byref(x)
