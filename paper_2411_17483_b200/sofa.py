"""Thin ctypes binding of libsofa.so (include/sofa.h) — argument marshalling only.

Every function keeps the C name and argument order; device arrays are passed as torch CUDA
tensors (their data_ptr), host arrays as numpy arrays.  Errors raise SofaError with the
library's message.  There is no fallback: if libsofa.so is missing or no CUDA device is
present the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .build import LIB

MAX_L = 64
MAX_K = 128
BINNING = {"equi-depth": 0, "equi-width": 1, "isax": 2}


class SofaError(RuntimeError):
    pass


class sofa_model(C.Structure):
    _fields_ = [("len", C.c_int32), ("l", C.c_int32), ("alphabet", C.c_int32), ("binning", C.c_int32),
                ("best_pos", C.c_int32 * MAX_L), ("weights", C.c_double * MAX_L),
                ("edges", C.c_double * (MAX_L * 255))]

    def to_dict(self) -> dict:
        l, a = self.l, self.alphabet
        e = np.ctypeslib.as_array(self.edges).reshape(MAX_L, 255)[:l, :a - 1].copy()
        return {"n": self.len, "l": l, "a": a, "best_pos": np.array(self.best_pos[:l], dtype=np.int64),
                "weights": np.array(self.weights[:l]), "edges": e,
                "binning": {0: "equi-depth", 1: "equi-width", 2: "isax"}[self.binning]}

    @classmethod
    def from_dict(cls, m: dict) -> "sofa_model":
        out = cls()
        out.len, out.l, out.alphabet = int(m["n"]), int(m["l"]), int(m["a"])
        out.binning = BINNING[m.get("binning", "equi-depth")]
        for j in range(out.l):
            out.best_pos[j] = int(m["best_pos"][j])
            out.weights[j] = float(m["weights"][j])
            for i in range(out.alphabet - 1):
                out.edges[j * 255 + i] = float(m["edges"][j][i])
        return out


class sofa_build_opts(C.Structure):
    _fields_ = [("sample_size", C.c_int64), ("sample_ratio", C.c_double), ("block_size", C.c_int32),
                ("candidate_limit", C.c_int32), ("binning", C.c_int32), ("dense_permille", C.c_int32),
                ("global_offset", C.c_int64), ("global_n", C.c_int64), ("model", C.POINTER(sofa_model))]


class sofa_tuning(C.Structure):
    _fields_ = [(f, C.c_int32) for f in ("front_batches", "rev_rounds", "topm_min", "topm_leaves",
                                         "refine_rows_front", "refine_rows_scan", "front_wide", "scan_wide")] + \
        [("dense_cand_cap", C.c_int64), ("dense_batch_rows", C.c_int64), ("dense_pair", C.c_int32),
         ("dense_diag", C.c_int32), ("dense_mcast", C.c_int32), ("dense_klist", C.c_int32),
         ("scan_fused", C.c_int32)]


class sofa_knn_stats(C.Structure):
    _fields_ = [(f, C.c_int64) for f in ("queries", "blocks_total", "blocks_survived", "words_scanned",
                                         "candidates", "refined", "abandoned", "env_nodes", "list_blocks",
                                         "rounds", "batches", "waves")] + [("phase_cycles", C.c_int64 * 4)] + \
        [(f, C.c_int64) for f in ("max_query_cycles", "max_list_blocks", "max_batches", "dense_queries",
                                  "dense_candidates", "dense_refined", "scan_tasks", "scan_queries")] + \
        [("kernel_ms", C.c_double * 3)]

    def to_dict(self) -> dict:
        d = {f: int(getattr(self, f)) for f, _ in self._fields_ if f not in ("phase_cycles", "kernel_ms")}
        d["phase_cycles"] = dict(zip(("prep", "seed", "tree", "scan_refine"), map(int, self.phase_cycles)))
        d["kernel_ms"] = dict(zip(("front", "dense", "scan"), map(float, self.kernel_ms)))
        return d


class sofa_index_info(C.Structure):
    _fields_ = [("n", C.c_int64), ("n_blocks", C.c_int64), ("global_offset", C.c_int64), ("global_n", C.c_int64),
                ("len", C.c_int32), ("l", C.c_int32), ("alphabet", C.c_int32), ("block_size", C.c_int32),
                ("word_stride", C.c_int32), ("build_ms", C.c_double * 4), ("dense_enabled", C.c_int32)]


_LIB = None
VP, I64, I32, P = C.c_void_p, C.c_int64, C.c_int32, C.POINTER


def lib() -> C.CDLL:
    """Load libsofa.so (built by build.py); raises if it is absent."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB):
            raise SofaError(f"{LIB} is missing: run `python -m paper_2411_17483_b200.build` "
                            "(there is no CPU fallback)")
        L = C.CDLL(LIB)
        L.sofa_last_error.restype = C.c_char_p
        L.sofa_launch_count.restype = I64
        L.sofa_kernel_timing.argtypes = [VP, I32, VP, P(I64)]
        L.sofa_default_opts.argtypes = [P(sofa_build_opts)]
        L.sofa_default_tuning.argtypes = [P(sofa_tuning)]
        L.sofa_set_tuning.argtypes = [VP, P(sofa_tuning)]
        L.sofa_learn_model.argtypes = [VP, I64, I32, I32, I32, P(sofa_build_opts), VP, P(sofa_model)]
        L.sofa_build.argtypes = [VP, I64, I32, I32, I32, P(sofa_build_opts), VP, P(VP)]
        L.sofa_knn.argtypes = [VP, VP, I32, I32, VP, VP, VP, P(sofa_knn_stats), VP]
        L.sofa_knn_host.argtypes = [VP, VP, I32, I32, VP, VP, P(sofa_knn_stats), VP]
        L.sofa_merge_topk.argtypes = [VP, VP, I32, I32, I32, VP, VP, VP]
        L.sofa_get_model.argtypes = [VP, P(sofa_model)]
        L.sofa_knn_trace.argtypes = [VP, VP, I32]
        L.sofa_lower_bounds.argtypes = [VP, VP, I32, I64, VP, VP, VP, VP]
        L.sofa_knn_seed.argtypes = [VP, VP, I32, I32, VP, VP]
        L.sofa_transform.argtypes = [VP, I64, P(sofa_model), VP, VP, VP]
        L.sofa_get_info.argtypes = [VP, P(sofa_index_info)]
        L.sofa_export_index.argtypes = [VP, VP, VP, VP, VP, VP]
        L.sofa_dense_dots.argtypes = [VP, I64, I32, VP, I32, VP, VP]
        L.sofa_free.argtypes = [VP]
        L.sofa_free.restype = None
        _LIB = L
    return _LIB


def _ck(rc: int):
    if rc != 0:
        raise SofaError(f"libsofa error {rc}: {lib().sofa_last_error().decode()}")


def _ptr(t) -> int | None:
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def _stream(stream) -> int | None:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return stream if isinstance(stream, int) else stream.cuda_stream


def sofa_last_error() -> str:
    return lib().sofa_last_error().decode()


def sofa_launch_count() -> int:
    return int(lib().sofa_launch_count())


def sofa_kernel_timing(ix: int, enable: int) -> tuple[dict, int]:
    """drain the live timing events; returns ({front, dense, scan} summed ms, sub-batches timed) and
    then enables (1), disables (0) or keeps (-1) timing; see include/sofa.h"""
    ms = (C.c_double * 4)()
    groups = I64(0)
    _ck(lib().sofa_kernel_timing(ix, enable, ms, C.byref(groups)))
    front, screen, post, scan = map(float, ms)
    return {"front": front, "dense": screen + post, "scan": scan, "dense_screen": screen, "dense_post": post}, \
        int(groups.value)


def sofa_default_opts() -> sofa_build_opts:
    o = sofa_build_opts()
    _ck(lib().sofa_default_opts(C.byref(o)))
    return o


def sofa_default_tuning() -> sofa_tuning:
    t = sofa_tuning()
    _ck(lib().sofa_default_tuning(C.byref(t)))
    return t


def sofa_set_tuning(ix, tuning: sofa_tuning):
    _ck(lib().sofa_set_tuning(ix, C.byref(tuning)))


def sofa_learn_model(sample_dev, S, len_, l, alphabet, opts=None, stream=None) -> sofa_model:
    m = sofa_model()
    _ck(lib().sofa_learn_model(_ptr(sample_dev), S, len_, l, alphabet, C.byref(opts) if opts else None,
                               _stream(stream), C.byref(m)))
    return m


def sofa_build(series_dev, n, len_, l, alphabet, opts=None, stream=None) -> int:
    h = VP()
    _ck(lib().sofa_build(_ptr(series_dev), n, len_, l, alphabet, C.byref(opts) if opts else None,
                         _stream(stream), C.byref(h)))
    return h.value


def sofa_knn(ix, queries_dev, q, k, bsf_init_dev, out_dist_dev, out_idx_dev, stats=None, stream=None):
    _ck(lib().sofa_knn(ix, _ptr(queries_dev), q, k, _ptr(bsf_init_dev), _ptr(out_dist_dev), _ptr(out_idx_dev),
                       C.byref(stats) if stats is not None else None, _stream(stream)))


def sofa_knn_host(ix, queries_host, q, k, out_dist_host, out_idx_host, stats=None, stream=None):
    _ck(lib().sofa_knn_host(ix, _ptr(queries_host), q, k, _ptr(out_dist_host), _ptr(out_idx_host),
                            C.byref(stats) if stats is not None else None, _stream(stream)))


def sofa_merge_topk(dist_dev, idx_dev, parts, q, k, out_dist_dev, out_idx_dev, stream=None):
    _ck(lib().sofa_merge_topk(_ptr(dist_dev), _ptr(idx_dev), parts, q, k, _ptr(out_dist_dev), _ptr(out_idx_dev),
                              _stream(stream)))


TRACE_FIELDS = ("cyc_prep", "cyc_seed", "cyc_tree", "cyc_scan", "blocks_survived", "words_scanned",
                "candidates", "refined", "abandoned", "env_nodes", "list_blocks", "rounds", "batches", "waves",
                "cta", "sm", "dense_flag", "leaves_after_take", "take_pass", "take_words",
                "cyc_scan_topm", "cyc_scan_decide", "cyc_scan_blocks", "cyc_scan_rest")


def sofa_knn_trace(ix, q) -> np.ndarray:
    out = np.zeros((q, len(TRACE_FIELDS)), dtype=np.int64)
    _ck(lib().sofa_knn_trace(ix, out.ctypes.data, q))
    return out


def sofa_lower_bounds(ix, queries_dev, q, m, out_lb2_dev, out_ed2_dev, out_rows_dev, stream=None):
    _ck(lib().sofa_lower_bounds(ix, _ptr(queries_dev), q, m, _ptr(out_lb2_dev), _ptr(out_ed2_dev),
                                _ptr(out_rows_dev), _stream(stream)))


def sofa_knn_seed(ix, queries_dev, q, k, out_bound_dev, stream=None):
    _ck(lib().sofa_knn_seed(ix, _ptr(queries_dev), q, k, _ptr(out_bound_dev), _stream(stream)))


def sofa_get_model(ix) -> sofa_model:
    m = sofa_model()
    _ck(lib().sofa_get_model(ix, C.byref(m)))
    return m


def sofa_transform(series_dev, n, model: sofa_model, out_values_dev=None, out_words_dev=None, stream=None):
    _ck(lib().sofa_transform(_ptr(series_dev), n, C.byref(model), _ptr(out_values_dev), _ptr(out_words_dev),
                             _stream(stream)))


def sofa_get_info(ix) -> sofa_index_info:
    o = sofa_index_info()
    _ck(lib().sofa_get_info(ix, C.byref(o)))
    return o


def sofa_export_index(ix, words_sorted_dev=None, perm_dev=None, env_dev=None, block_keys_dev=None, stream=None):
    _ck(lib().sofa_export_index(ix, _ptr(words_sorted_dev), _ptr(perm_dev), _ptr(env_dev), _ptr(block_keys_dev),
                                _stream(stream)))


def sofa_dense_dots(rows_dev, m, len_, queries_dev, q, out_dev, stream=None):
    _ck(lib().sofa_dense_dots(_ptr(rows_dev), m, len_, _ptr(queries_dev), q, _ptr(out_dev), _stream(stream)))


def sofa_free(ix):
    if ix:
        lib().sofa_free(ix)
