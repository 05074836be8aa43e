"""Loader for the in-tree native libraries.

* ``libhyperball_b200.so`` -- the sm_100a kernels behind the C-ABI declared in
  ``include/hyperball_b200.h``.  There is no CPU fallback: every device entry point
  raises ``RuntimeError`` when the library is missing or a call fails.
* ``libhbgraph.so`` -- host C builders for the synthetic benchmark graphs.

Both are built in place by ``__graft_entry__.build()`` (``make -C
paper_1308_2144_b200/csrc``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
HB_LIB_PATH = os.environ.get("HB_LIB") or os.path.join(_HERE, "libhyperball_b200.so")
GRAPH_LIB_PATH = os.path.join(_HERE, "libhbgraph.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "hyperball_b200.h")

_lock = threading.Lock()
_hb = None
_graph = None

_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_int = ctypes.c_int
_dbl = ctypes.c_double
_vp = ctypes.c_void_p

# name -> (restype, argtypes), in header order
HB_SIGNATURES = {
    "hb_version": (ctypes.c_char_p, []),
    "hb_last_error": (ctypes.c_char_p, []),
    "hb_min_log2m": (_int, []),
    "hb_max_log2m": (_int, []),
    "hb_seed": (_int, [_vp, _vp, _i64, _int, _int, _u64, _vp, _vp, _vp, _dbl, _dbl, _vp]),
    "hb_estimate_rows": (_int, [_vp, _i64, _i64, _int, _vp, _dbl, _dbl, _vp, _vp]),
    "hb_union_step": (_int, [_i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _int, _vp, _vp,
                             _vp, _i64, _vp, _dbl, _dbl, _int, _int, _i64, _vp, _vp, _i64,
                             _vp, _i64, _vp, _vp, _i64, _i64, _vp, _vp, _vp, _i64,
                             _vp, _i64, _int, _vp, _int, _vp, _int, _vp, _vp, _vp]),
    "hb_union_step_v2": (_int, [_vp]),
    "hb_set_l2_persist": (None, [_int]),
    "hb_step_args_size": (_u64, []),
    "hb_step_args_min_size": (_u64, []),
    "hb_push_row_stride": (_int, [_int]),
    "hb_max_degree": (_int, [_i64, _vp, _vp, _vp, _vp]),
    "hb_schedule_order": (_int, [_i64, _vp, _int, _int, _int, _vp, _vp, _vp, _vp, _vp, _vp,
                                 _vp]),
    "hb_heavy_items": (_int, [_i64, _i64, _vp, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp,
                              _vp, _vp, _vp, _vp]),
    "hb_unpack_inbox": (_int, [_i64, _i64, _i64, _int, _vp, _vp, _vp, _vp, _vp, _vp]),
    "hb_union_step_runs": (_int, [_i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                  _vp, _vp, _i64, _i64, _vp, _dbl, _dbl, _int, _int, _int,
                                  _i64, _vp, _vp, _i64, _vp, _i64, _vp, _vp, _i64, _i64, _vp,
                                  _vp, _vp, _vp, _i64, _vp, _i64, _int, _vp, _int, _vp, _vp]),
    "hb_mark_active": (_int, [_i64, _vp, _vp, _vp, _vp, _vp]),
    "hb_pack_registers": (_int, [_i64, _int, _int, _vp, _vp, _vp, _vp]),
    "hb_unpack_registers": (_int, [_i64, _int, _int, _vp, _vp, _vp, _vp]),
    "hb_mark_pull": (_int, [_i64, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _i64, _i64, _vp]),
    "hb_mark_pull_filtered": (_int, [_i64, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _i64, _i64,
                                     _i64, _i64, _vp, _vp]),
    "hb_change_filter_words": (_i64, []),
    "hb_exact_seed": (_int, [_i64, _i64, _vp, _vp, _vp, _vp]),
    "hb_exact_union_step": (_int, [_i64, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp,
                                   _i64, _int, _vp, _vp, _i64, _int, _vp, _int, _vp, _vp,
                                   _vp]),
    "hb_forward_csr": (_int, [_i64, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "hb_finalize": (_int, [_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "hb_packed_row_bytes": (_int, [_int]),
    "hb_gather_changed": (_int, [_i64, _i64, _vp, _vp, _int, _int, _vp, _vp, _vp, _vp]),
    "hb_scatter_rows": (_int, [_i64, _vp, _vp, _int, _int, _vp, _vp, _vp]),
    "hb_refresh_rows": (_int, [_i64, _i64, _i64, _vp, _vp, _vp, _int, _vp]),
    "hb_relabel_csr": (_int, [_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "hb_relabel_csr_rows": (_int, [_i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "hb_sample_flagged_arcs": (_int, [_i64, _vp, _vp, _i64, _u64, _vp, _vp]),
    "hb_relabel_csr_src_rows": (_int, [_i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "hb_sort_rows": (_int, [_i64, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "hb_gen_rmat_keys": (_int, [_int, _i64, _u64, _u64, _u64, _u64, _vp, _vp]),
    "hb_keys_to_csr": (_int, [_i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "hb_hash_items": (_int, [_i64, _vp, _vp, _u64, _vp, _vp]),
    "hb_map_ids": (_int, [_i64, _vp, _vp, _vp, _vp]),
    "hb_gen_degrees": (_int, [_int, _i64, _u64, _vp, _i64, _i64, _vp, _vp]),
    "hb_gen_blocks": (_int, [_i64, _i64, _dbl, _u64, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "hb_gen_arc_keys": (_int, [_int, _i64, _u64, _vp, _vp, _vp, _dbl, _i64, _vp, _vp]),
    "hb_transpose_csr": (_int, [_i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "hb_die_map": (_int, [_vp, _i64, _vp, _vp, _vp]),
    "hb_die_map_words": (_i64, [_vp, _i64]),
    "hb_die_partition": (_int, [_i64, _vp, _vp, _vp, _vp, _i64, _int, _vp, _i64, _vp, _vp, _vp]),
    "hb_item_arcs": (_i64, [_int]),
    "hb_light_max_deg": (_i64, [_int]),
    "hb_light_npw": (_i64, [_int]),
    "hb_light_window": (_i64, [_int]),
}

class StepArgs(ctypes.Structure):
    """``hb_step_args`` (include/hyperball_b200.h): hb_union_step_v2's named arguments."""

    _fields_ = [
        ("struct_size", ctypes.c_uint64),
        ("n", _i64), ("lo", _i64), ("hi", _i64),
        ("offsets", _vp), ("succ", _vp),
        ("cur", _vp), ("nxt", _vp), ("chg_prev", _vp), ("chg_now", _vp), ("est", _vp),
        ("b", ctypes.c_int32), ("dense", ctypes.c_int32), ("clear_chg_now", ctypes.c_int32),
        ("n_disc", ctypes.c_int32),
        ("t", _i64),
        ("lc_table", _vp), ("alpha_p2", _dbl), ("lc_cut", _dbl),
        ("sum_dist", _vp), ("sum_recip", _vp), ("disc", _vp), ("disc_stride", _i64),
        ("disc_scale", _vp), ("disc_div", ctypes.c_int32), ("n_peers", ctypes.c_int32),
        ("light_max_deg", _i64), ("heavy_nodes", _vp), ("item_first", _vp), ("n_heavy", _i64),
        ("finish_order", _vp), ("n_mega", _i64), ("item_node", _vp), ("item_beg", _vp),
        ("n_items", _i64), ("item_arcs", _i64), ("partial", _vp),
        ("nch_out", _vp), ("merged_out", _vp), ("hot_rows", _i64), ("active", _vp),
        ("peer_nxt", _vp), ("peer_chg", _vp), ("stream", _vp),
        ("check_rows", _i64), ("check_m", _i64),
        ("peer_packed_stride", _i64),
        ("ticket", _vp),
        ("die_head", _vp), ("die_rows", _i64), ("item_split", _vp),
    ]

    def __init__(self, **kw):
        super().__init__(struct_size=ctypes.sizeof(StepArgs))
        for k, v in kw.items():
            setattr(self, k, v)


def schedule_args(s) -> dict:
    """The heavy-node schedule fields of StepArgs from a schedule.Schedule."""
    return dict(light_max_deg=s.light_max_deg, heavy_nodes=s.heavy_nodes.data_ptr(),
                item_first=s.item_first.data_ptr(), n_heavy=s.n_heavy,
                finish_order=s.finish_order.data_ptr(), n_mega=s.n_mega,
                item_node=s.item_node.data_ptr(), item_beg=s.item_beg.data_ptr(),
                n_items=s.n_items, item_arcs=s.item_arcs, partial=s.partial.data_ptr(),
                hot_rows=s.hot_rows, check_m=int(s.succ_buf.numel()))


def union_step(args: StepArgs, what: str = "hb_union_step_v2") -> None:
    check(hb().hb_union_step_v2(ctypes.byref(args)), what)


GRAPH_SIGNATURES = {
    "hbg_er": (_vp, [_i64, _dbl, _u64, _int]),
    "hbg_rmat": (_vp, [_int, _i64, _dbl, _dbl, _dbl, _u64, _int]),
    "hbg_disconnected": (_vp, [_i64, _i64, _dbl, _dbl, _u64, _int]),
    "hbg_weblike": (_vp, [_i64, _dbl, _i64, _i64, _dbl, _i64, _u64, _int]),
    "hbg_from_arcs": (_vp, [_i64, _i64, _vp, _vp, _int]),
    "hbg_poisson_cdf": (_int, [_dbl, _vp]),
    "hbg_zipf_cdf": (None, [_dbl, _i64, _i64, _vp]),
    "hbg_gather_rows": (_i64, [_vp, _vp, _int, _vp, _i64, _vp, _vp, _int]),
    "hbg_stage_ids": (_int, [_vp, _int, _i64, _vp, _int]),
    "hbg_stage_bytes": (None, [_vp, _i64, _vp, _int]),
    "hbg_n": (_i64, [_vp]),
    "hbg_m": (_i64, [_vp]),
    "hbg_copy": (None, [_vp, _vp, _vp]),
    "hbg_free": (None, [_vp]),
}


def build_native() -> None:
    """Compile both libraries in place (nvcc for sm_100a + gcc)."""
    subprocess.run(["make", "-s", "-C", os.path.join(_HERE, "csrc")], check=True)


def _bind(path: str, sigs: dict):
    L = ctypes.CDLL(path)
    for name, (res, args) in sigs.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    return L


def hb():
    """The CUDA kernel library; raises if it was not built."""
    global _hb
    if _hb is None:
        with _lock:
            if _hb is None:
                if not os.path.exists(HB_LIB_PATH):
                    raise RuntimeError(
                        f"{HB_LIB_PATH} is missing: build it with __graft_entry__.build() "
                        "(there is no CPU fallback for the HyperBall hot path)")
                _hb = _bind(HB_LIB_PATH, HB_SIGNATURES)
    return _hb


def use_graph_library(path: str) -> None:
    """Bind the synthetic-graph builders (hbg_*) from another library exporting them --
    bench.py's CPU reference arm uses the oracle's copy, so that process maps no product
    library.  Must be called before the first graphlib()."""
    global GRAPH_LIB_PATH, _graph
    with _lock:
        if _graph is not None and GRAPH_LIB_PATH != path:
            raise RuntimeError("graph library already bound")
        GRAPH_LIB_PATH = path


def graphlib():
    global _graph
    if _graph is None:
        with _lock:
            if _graph is None:
                if not os.path.exists(GRAPH_LIB_PATH):
                    raise RuntimeError(f"{GRAPH_LIB_PATH} is missing: run __graft_entry__.build()")
                _graph = _bind(GRAPH_LIB_PATH, GRAPH_SIGNATURES)
    return _graph


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = hb().hb_last_error().decode(errors="replace")
        raise RuntimeError(f"{what} failed (code {rc}): {msg}")
