"""ctypes binding of libddilu_b200.so (the C ABI declared in include/ddilu_b200.h).

There is no CPU fallback: if the library is missing the import of any compute
entry point raises, and every call checks the library's status code.
"""

from __future__ import annotations

import ctypes
import os

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libddilu_b200.so")

_P = ctypes.c_void_p
_I = ctypes.c_int
_L = ctypes.c_longlong
_D = ctypes.c_double
_S = ctypes.c_char_p

# name -> (restype, argtypes); must stay in sync with include/ddilu_b200.h
SIGNATURES = {
    "ddilu_scan_tmp_elems": (_L, [_L]),
    "ddilu_exclusive_scan_i32": (_I, [_P, _P, _L, _P, _P]),
    "ddilu_sort_tmp_elems": (_L, [_L]),
    "ddilu_sort_pairs_i32": (_I, [_P, _P, _P, _P, _L, _I, _P, _P]),
    "ddilu_spmv_csr_f64": (_I, [_I, _I, _P, _P, _P, _P, _P, _P, _I, _P]),
    "ddilu_spmv_csr_f64_tuned": (_I, [_I, _I, _P, _P, _P, _P, _P, _P, _I, _D, _P]),
    "ddilu_levels": (_I, [_I, _P, _P, _I, _P, _P, _P]),
    "ddilu_schedule_build": (_I, [_I, _P, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "ddilu_sptrsv": (_I, [_I, _I, _P, _P, _P, _P, _P, _P, _I, _I, _P, _P]),
    "ddilu_sptrsv_warprow": (_I, [_I, _I, _P, _P, _P, _P, _P, _P, _I, _I, _P, _P]),
    "ddilu_sell_width": (_I, [_I, _P, _P, _P, _P, _I, _I, _P, _P, _P, _P, _P, _P]),
    "ddilu_sell_fill": (_I, [_I, _P, _P, _P, _P, _I, _P, _I, _P, _P, _P]),
    "ddilu_compose_wait": (_I, [_I, _P, _P, _P, _P, _P]),
    "ddilu_sptrsv_sell": (_I, [_I, _I, _I, _P, _P, _I, _P, _P, _P, _P, _P, _P, _D, _P, _P, _P]),
    "ddilu_iluk_smem_bytes": (_L, [_I]),
    "ddilu_iluk_symbolic": (_I, [_I, _P, _P, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "ddilu_compact_cols": (_I, [_I, _I, _P, _P, _P, _P, _P]),
    "ddilu_prefill": (_I, [_I, _P, _P, _P, _P, _P, _P, _I, _I, _P]),
    "ddilu_tile_box_keys": (_I, [_I, _P, _I, _P, _P, _P, _P, _P, _P]),
    "ddilu_tile_heads": (_I, [_I, _P, _P, _P]),
    "ddilu_tile_assign": (_I, [_I, _P, _P, _P, _P, _P, _P, _P]),
    "ddilu_tile_edges_count": (_I, [_I, _P, _P, _I, _P, _P, _P]),
    "ddilu_tile_edges_fill": (_I, [_I, _P, _P, _I, _P, _P, _P, _P]),
    "ddilu_tile_relax": (_I, [_L, _P, _I, _P, _P, _I, _P]),
    "ddilu_tile_build": (_I, [_I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _P, _P, _P, _P]),
    "ddilu_tiled_smem_bytes": (_L, [_I, _I, _I]),
    "ddilu_fastdiv_selftest": (_I, [_L, ctypes.c_ulonglong, _P, _P]),
    "ddilu_sptrsv_tiled": (_I, [_I, _I, _P, _P, _I, _I, _I, _I, _I, _P, _P, _P]),
    "ddilu_sweep_page_rows": (_I, [_I]),
    "ddilu_sweep_helper_threads": (_I, []),
    "ddilu_sweep_page_bytes": (_L, [_I, _I]),
    "ddilu_sweep_smem_bytes": (_L, [_I, _I, _I, _I]),
    "ddilu_sweep_fill": (_I, [_I, _P, _P, _P, _I, _I, _P, _P, _P, _I, _P, _P, _P]),
    "ddilu_sweep_rhs": (_I, [_I, _P, _P, _P, _P, _P, _P, _I, _P, _P, _P, _P, _P]),
    "ddilu_sweep_solve": (_I, [_I, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P]),
    "ddilu_csweep_threads": (_I, [_I]),
    "ddilu_csweep_window": (_I, [_I]),
    "ddilu_csweep_max_push": (_I, [_I]),
    "ddilu_csweep_rank_bits": (_I, [_I]),
    "ddilu_csweep_code_words": (_I, [_I]),
    "ddilu_csweep_smem_bytes": (_L, [_I, _I, _I, _I]),
    "ddilu_csweep_active_clusters": (_I, [_I, _I, _I, _I]),
    "ddilu_csweep_fill": (_I, [_I, _P, _P, _P, _I, _I, _P, _P, _L, _P, _P, _P, _P, _P, _P]),
    "ddilu_csweep_long_record_bytes": (_I, [_I, _I]),
    "ddilu_csweep_fill_long": (_I, [_I, _P, _P, _P, _I, _I, _P, _P, _P, _P, _P, _P, _P]),
    "ddilu_csweep_solve": (_I, [_I, _I, _P, _P, _P, _P, _P, _P, _P, _L, _I, _I, _I, _I, _P, _P, _P]),
    "ddilu_peer_allreduce": (_I, [_I, _I, _P, _P, _P, _P, _I, _I, _L, _L, _P, _P]),
    "ddilu_peer_send": (_I, [_I, _I, _I, _P, _P, _P, _P, _P, _P, _L, _L, _L, _P, _P, _P]),
    "ddilu_peer_recv": (_I, [_I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _I, _L, _L, _L, _P, _P, _P]),
    "ddilu_split_count": (_I, [_I, _P, _P, _P, _I, _P, _P, _P, _P]),
    "ddilu_split_fill": (_I, [_I, _P, _P, _P, _I, _P, _P, _P, _P, _P, _P, _P]),
    "ddilu_ilu0_numeric": (_I, [_I, _I, _P, _P, _P, _P, _P, _P, _P, _I, _I, _P, _P, _D, _P, _P, _P]),
    "ddilu_ilut_smem_bytes": (_L, [_I]),
    "ddilu_ilut_caps": (_I, [_I, _I, _P]),
    "ddilu_ilut_factor": (_I, [_I, _P, _P, _P, _I, _D, _I, _D, _D, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "ddilu_compact_rows": (_I, [_I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P]),
    "ddilu_csr_block_count": (_I, [_P, _P, _I, _I, _I, _I, _P, _P]),
    "ddilu_csr_block_fill": (_I, [_P, _P, _P, _I, _I, _I, _I, _P, _P, _P, _P]),
    "ddilu_reduce_ws_bytes": (_L, []),
    "ddilu_dot": (_I, [_L, _P, _P, _P, _P, _P]),
    "ddilu_dot_dir": (_I, [_L, _P, _P, _P, _P, _I, _P]),
    "ddilu_axpy_dot": (_I, [_L, _P, _D, _P, _P, _P, _P, _P, _P]),
    "ddilu_axpy_dot_dir": (_I, [_L, _P, _D, _P, _P, _P, _P, _P, _I, _P]),
    "ddilu_mgs_ws_bytes": (_L, []),
    "ddilu_mgs_max_block": (_I, []),
    "ddilu_mgs_block": (_I, [_L, _L, _I, _P, _P, _P, _P, _I, _P, _P, _P, _I, _P]),
    "ddilu_mgs_small_max": (_I, []),
    "ddilu_mgs_small_step": (_I, [_L, _L, _I, _P, _P, _P, _P, _P, _P, _I, _I, _P]),
    "ddilu_norm_scale_small": (_I, [_L, _P, _P, _P, _P, _P, _P]),
    "ddilu_scale": (_I, [_L, _P, _P, _D, _I, _I, _P, _P]),
    "ddilu_l2_persist_window": (_I, [_P, _L, _P]),
    "ddilu_multi_axpy": (_I, [_L, _I, _P, _L, _P, _P, _I, _P]),
    "ddilu_gmres_small_max": (_I, []),
    "ddilu_gmres_small_solve": (_I, [_I, _P, _I, _P, _D, _P, _P, _P]),
    "ddilu_ewise": (_I, [_L, _P, _P, _I, _P, _P]),
    "ddilu_gather": (_I, [_L, _P, _P, _P, _P]),
    "ddilu_scatter": (_I, [_L, _P, _P, _P, _P]),
    "ddilu_mark_exterior": (_I, [_I, _P, _P, _P, _P, _P]),
    "ddilu_layout_keys": (_I, [_I, _P, _P, _I, _P, _P, _P]),
    "ddilu_lower_bounds": (_I, [_P, _I, _I, _P, _P]),
    "ddilu_box_owner": (_I, [_I, _I, _P, _P, _P, _P]),
    "ddilu_build_map": (_I, [_I, _P, _I, _P, _P]),
    "ddilu_gather_rows_count": (_I, [_I, _P, _P, _P, _P, _P, _I, _P, _P]),
    "ddilu_gather_rows_fill": (_I, [_I, _P, _P, _P, _P, _P, _P, _I, _P, _P, _P, _I, _P]),
    "ddilu_mark_foreign_cols": (_I, [_I, _P, _P, _P, _P, _P, _P]),
    "ddilu_mark_sends": (_I, [_I, _P, _P, _P, _I, _I, _P, _I, _P, _P]),
    "ddilu_sym_adj_count": (_I, [_I, _P, _P, _P, _P]),
    "ddilu_sym_adj_fill": (_I, [_I, _P, _P, _P, _P, _P, _P]),
    "ddilu_sort_rows_i32": (_I, [_I, _P, _P, _P]),
    "ddilu_grow_regions": (_I, [_I, _P, _P, _I, _P, _P, _P, _P]),
    "ddilu_spgemm_bound": (_I, [_I, _P, _P, _P, _P, _P]),
    "ddilu_spgemm_expand": (_I, [_I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "ddilu_spgemm_compact": (_I, [_I, _P, _P, _P, _P, _P, _P, _P]),
    "ddilu_l1_row_shifts": (_I, [_I, _P, _P, _P, _P, _P, _P, _P]),
    "ddilu_add_to_diagonal": (_I, [_I, _P, _P, _P, _P, _P, _P]),
    "ddilu_drop_small_count": (_I, [_I, _P, _P, _P, _D, _P, _P]),
    "ddilu_drop_small_fill": (_I, [_I, _P, _P, _P, _D, _P, _P, _P, _P]),
    "ddilu_row_lengths": (_I, [_I, _P, _P, _P]),
    "ddilu_cm_work_elems": (_L, [_I]),
    "ddilu_cm_order": (_I, [_I, _P, _P, _P, _P, _P]),
    "ddilu_cm_order_segments": (_I, [_I, _P, _P, _I, _P, _P, _P, _P]),
    "ddilu_reverse_segments": (_I, [_I, _P, _I, _P, _P, _P]),
    "ddilu_narrow_i64": (_I, [_L, _P, _P, _P]),
    "ddilu_widen_i32": (_I, [_L, _P, _P, _P]),
}

# entries that exist only in a -DDDILU_EXPERIMENTS build (include/ddilu_b200_experiments.h): measured-slower
# alternative kernels, tuning knobs, diagnostics.  Bound when the library has them.
EXPERIMENT_SIGNATURES = {
    "ddilu_tsweep_page_bytes": (_L, [_I, _I]),
    "ddilu_tsweep_smem_bytes": (_L, [_I, _I, _I, _I, _I, _I]),
    "ddilu_tsweep_fill": (_I, [_I, _P, _P, _P, _I, _I, _P, _P, _P, _I, _P, _P, _P]),
    "ddilu_tsweep_permute": (_I, [_I, _P, _P, _P, _I, _P]),
    "ddilu_tsweep_solve": (_I, [_I, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _I, _P, _P, _P]),
    "ddilu_set_tuning": (_I, [_S, _I]),
    "ddilu_blocklocal_table": (_I, [_I, _I, _P, _I, _P, _P, _P, _P, _P]),
    "ddilu_sptrsv_blocklocal": (_I, [_I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _P, _P]),
    "ddilu_sptrsv_blocklocal_sell": (_I, [_I, _I, _P, _P, _P, _P, _I, _P, _P, _P, _P, _P, _P]),
    "ddilu_sptrsv_blockwin_sell": (_I, [_I, _I, _P, _P, _P, _P, _P, _I, _P, _P, _P, _P, _I, _P, _P, _P]),
    "ddilu_sptrsv_sell_trace": (_I, [_I, _I, _I, _P, _P, _I, _P, _P, _P, _P, _P, _P, _P, _P]),
    "ddilu_tiled_set_tuning": (_I, [_S, _I]),
    "ddilu_tiled_set_debug": (_I, [_P]),
    "ddilu_tile_slab_keys": (_I, [_I, _P, _I, _P, _P, _P, _I, _I, _P, _I, _P, _P, _P]),
    "ddilu_warptile_smem_per_warp": (_L, [_I, _I, _I]),
    "ddilu_sptrsv_lean": (_I, [_I, _I, _P, _P, _I, _I, _I, _I, _I, _P, _P, _P]),
    "ddilu_sptrsv_warptile": (_I, [_I, _I, _P, _P, _I, _I, _I, _I, _I, _P, _P, _P]),
    "ddilu_sweep_set_debug": (_I, [_P]),
    "ddilu_csweep_set_debug": (_I, [_P]),
    "ddilu_sweep_set_tuning": (_I, [_I, _I]),
    "ddilu_lattice_build": (_I, [_I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _P, _P, _P, _P, _P]),
    "ddilu_lattice_max_ext": (_I, []),
    "ddilu_lattice_set_tuning": (_I, [_S, _I]),
    "ddilu_lattice_smem_bytes": (_L, [_I, _I, _I]),
    "ddilu_lattice_set_debug": (_I, [_P]),
    "ddilu_sptrsv_lattice": (_I, [_I, _P, _P, _P, _I, _I, _I, _I, _I, _P, _P, _P]),
}

_lib = None
_experiments = False
launches = 0  # kernels-launching C-ABI calls made so far (bench.py reports the delta)

# Optional per-entry timing with CUDA events on the launching stream (bench.py):
# profile = {"name": [(start_event, end_event, tag), ...]} for the watched entries.
profile = None
profile_tag = None


class DdiluError(RuntimeError):
    pass


def load() -> ctypes.CDLL:
    """Load the shared library (no device needed); raises if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DdiluError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2303_08881_b200.build` "
                "(there is no CPU fallback for the DD-ILU path)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        global _experiments
        _experiments = hasattr(lib, next(iter(EXPERIMENT_SIGNATURES)))
        if _experiments:
            for name, (res, args) in EXPERIMENT_SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
        _lib = lib
    return _lib


def has_experiments() -> bool:
    """Whether the loaded library was built with -DDDILU_EXPERIMENTS (alternative kernels, knobs, diagnostics)."""
    load()
    return _experiments


def _entry(name: str):
    lib = load()
    if name in EXPERIMENT_SIGNATURES and not _experiments:
        raise DdiluError(f"{name} is an experiments-only entry: rebuild with DDILU_EXPERIMENTS=1 "
                         "python -m paper_2303_08881_b200.build")
    return getattr(lib, name)


def require_cuda() -> None:
    if not torch.cuda.is_available():
        raise DdiluError("the DD-ILU path runs on a CUDA device only (sm_100a); no CPU fallback exists")


def _arg(a):
    if a is None:
        return None
    if isinstance(a, torch.Tensor):
        return a.data_ptr()
    return a


def stream_ptr():
    return torch.cuda.current_stream().cuda_stream


def call(name: str, *args):
    """Call a status-returning entry point with torch tensors / scalars; the
    current torch stream is appended as the last argument."""
    global launches
    fn = _entry(name)
    if profile is not None and name in profile:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rc = fn(*[_arg(a) for a in args], stream_ptr())
        e1.record()
        profile[name].append((e0, e1, profile_tag))
    else:
        rc = fn(*[_arg(a) for a in args], stream_ptr())
    launches += 1
    if rc != 0:
        raise DdiluError(f"{name} failed with status {rc}")


def query(name: str, *args):
    """Call a size-query entry point (no stream, returns a number)."""
    return _entry(name)(*args)
