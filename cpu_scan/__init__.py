"""UCR-Suite-P-style multithreaded CPU brute-force scan (cpu_scan/ucr_scan.cpp): a reported CPU
baseline for bench.py, not the oracle and not part of the product path."""
import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "lib", "libucrscan.so")
SRC = os.path.join(HERE, "ucr_scan.cpp")


def build(force: bool = False) -> str:
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    # x86-64-v3 (AVX2 + FMA): portable to the GPU box's host CPU, vectorised inner loop
    cmd = ["g++", "-O3", "-march=x86-64-v3", "-fopenmp", "-fPIC", "-shared", SRC, "-o", LIB]
    subprocess.run(cmd, check=True, capture_output=True)
    return LIB


_L = None


def _lib():
    global _L
    if _L is None:
        _L = C.CDLL(build())
        _L.ucr_row_stats.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_void_p]
        _L.ucr_knn.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_void_p, C.c_int, C.c_int,
                               C.c_void_p, C.c_void_p, C.c_int]
    return _L


def row_stats(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    out = np.empty((x.shape[0], 2), dtype=np.float32)
    _lib().ucr_row_stats(x.ctypes.data, x.shape[0], x.shape[1], out.ctypes.data)
    return out


def knn(x: np.ndarray, stats: np.ndarray, queries: np.ndarray, k: int, threads: int = 0):
    x = np.ascontiguousarray(x, dtype=np.float32)
    queries = np.ascontiguousarray(queries, dtype=np.float32)
    q = queries.shape[0]
    d = np.empty((q, k), dtype=np.float32)
    i = np.empty((q, k), dtype=np.int64)
    _lib().ucr_knn(x.ctypes.data, stats.ctypes.data, x.shape[0], x.shape[1], queries.ctypes.data, q, k,
                   d.ctypes.data, i.ctypes.data, threads)
    return d, i
