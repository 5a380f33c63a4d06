"""ctypes wrapper over oracle/_ref/libtreeattn_ref.so -- the unmodified
reference headers compiled in place by oracle/Makefile.

TEST INFRASTRUCTURE ONLY (golden-fixture generation, CPU baseline timing).
``available()`` is False where the .so was never built (no /root/reference).
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libtreeattn_ref.so")
REF_INCLUDE = "/root/reference/proj/include"
_lib = None

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
u64p = C.POINTER(C.c_uint64)
f32p = C.POINTER(C.c_float)
f64p = C.POINTER(C.c_double)
u8p = C.POINTER(C.c_uint8)


def build() -> bool:
    """Compile _ref from /root/reference when present (never copies sources)."""
    if not os.path.isdir(REF_INCLUDE):
        return os.path.exists(LIB_PATH)
    subprocess.run(["make", "-s", "-C", _HERE, "ref"], check=True)
    return True


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not available():
        raise RuntimeError("reference harness not built (oracle/_ref/libtreeattn_ref.so)")
    L = C.CDLL(LIB_PATH)
    snap = [C.c_int32, C.c_int, i32p, i32p, i64p]
    sig = {
        "ref_last_error": (C.c_char_p, []),
        "ref_free": (None, [C.c_void_p]),
        "ref_set_threads": (None, [C.c_int]),
        "ref_tune_malloc": (None, []),
        "ref_trace_few_shot": (C.c_void_p, [C.c_int64, C.c_int, C.c_int]),
        "ref_trace_preset": (C.c_void_p, [C.c_char_p]),
        "ref_trace_spec_json": (C.c_void_p, [C.c_char_p]),
        "ref_random_trees": (C.c_void_p, [C.c_uint64, C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int, C.c_int]),
        "ref_snaps_len": (C.c_int, [C.c_void_p]),
        "ref_snaps_iteration": (C.c_int, [C.c_void_p, C.c_int]),
        "ref_snaps_get": (C.c_int, [C.c_void_p, C.c_int, i32p, i32p, i32p, i64p]),
        "ref_snaps_free": (None, [C.c_void_p]),
        "ref_tree_leaves": (C.c_int, snap + [i32p]),
        "ref_plan_json": (C.c_void_p, snap + [C.c_char_p, C.c_int]),
        "ref_io_measured": (C.c_int, snap + [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, u64p]),
        "ref_io_analytical": (C.c_int, snap + [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, u64p]),
        "ref_instance_new": (C.c_void_p, snap + [C.c_int, C.c_int, C.c_uint64]),
        "ref_instance_new_gqa": (C.c_void_p, snap + [C.c_int, C.c_int, C.c_int, C.c_uint64]),
        "ref_instance_new_content": (C.c_void_p, snap + [C.c_int, C.c_int, f32p, f32p, f32p]),
        "ref_instance_free": (None, [C.c_void_p]),
        "ref_instance_dim": (C.c_int, [C.c_void_p]),
        "ref_instance_leaves": (C.c_int, [C.c_void_p, i32p]),
        "ref_instance_node_kv": (C.c_int, [C.c_void_p, C.c_int32, f32p, f32p]),
        "ref_instance_queries": (C.c_int, [C.c_void_p, f32p]),
        "ref_run_iteration": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int, C.c_int, C.c_int, f64p, u8p, f64p]),
        "ref_naive": (C.c_int, [C.c_void_p, f64p, f64p]),
        "ref_fill_uniform": (None, [f32p, C.c_int64, C.c_uint64]),
        "ref_content_seed": (C.c_uint64, [C.c_uint64, C.c_uint64, C.c_uint64]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def _p(a, t):
    return a.ctypes.data_as(t)


def _snap_args(snap):
    root, ids, par, cnt = snap
    ids = np.ascontiguousarray(ids, np.int32)
    par = np.ascontiguousarray(par, np.int32)
    cnt = np.ascontiguousarray(cnt, np.int64)
    return (int(root), len(ids), _p(ids, i32p), _p(par, i32p), _p(cnt, i64p)), (ids, par, cnt)


def _err():
    return lib().ref_last_error().decode()


def _snaps(h):
    if not h:
        raise RuntimeError(_err())
    out = []
    try:
        for i in range(lib().ref_snaps_len(h)):
            n = lib().ref_snaps_get(h, i, None, None, None, None)
            root = C.c_int32()
            ids = np.zeros(n, np.int32)
            par = np.zeros(n, np.int32)
            cnt = np.zeros(n, np.int64)
            lib().ref_snaps_get(h, i, C.byref(root), _p(ids, i32p), _p(par, i32p), _p(cnt, i64p))
            out.append((root.value, ids, par, cnt))
    finally:
        lib().ref_snaps_free(h)
    return out


def few_shot(prefix, branches, iterations):
    """gen_few_shot (workloads.hpp:98-111) -> list of snapshots."""
    return _snaps(lib().ref_trace_few_shot(prefix, branches, iterations))


def preset(name):
    return _snaps(lib().ref_trace_preset(name.encode()))


def spec(spec_obj: dict):
    return _snaps(lib().ref_trace_spec_json(json.dumps(spec_obj).encode()))


def random_trees(seed, n, max_leaves=64, max_tokens=8192, max_node_tokens=400,
                 max_branch_width=4, mutation_steps=24):
    return _snaps(lib().ref_random_trees(seed, n, max_leaves, max_tokens, max_node_tokens,
                                         max_branch_width, mutation_steps))


def leaves(snap):
    args, keep = _snap_args(snap)
    n = lib().ref_tree_leaves(*args, None)
    if n < 0:
        raise RuntimeError(_err())
    out = np.zeros(n, np.int32)
    lib().ref_tree_leaves(*args, _p(out, i32p))
    return out


def plan_json(snap, block_size=128, strategy="flatten") -> str:
    args, keep = _snap_args(snap)
    p = lib().ref_plan_json(*args, strategy.encode(), block_size)
    if not p:
        raise RuntimeError(_err())
    s = C.cast(p, C.c_char_p).value.decode()
    lib().ref_free(p)
    return s


def io_measured(snap, block_size, d_head, n_heads, n_layers, dtype_bytes, strategy="flatten"):
    args, keep = _snap_args(snap)
    out = np.zeros(4, np.uint64)
    if lib().ref_io_measured(*args, strategy.encode(), block_size, d_head, n_heads, n_layers,
                             dtype_bytes, _p(out, u64p)) != 0:
        raise RuntimeError(_err())
    return tuple(int(x) for x in out)


def io_analytical(snap, algorithm, block_size, d_head, n_heads, n_layers, dtype_bytes):
    args, keep = _snap_args(snap)
    out = np.zeros(4, np.uint64)
    if lib().ref_io_analytical(*args, algorithm.encode(), block_size, d_head, n_heads, n_layers,
                               dtype_bytes, _p(out, u64p)) != 0:
        raise RuntimeError(_err())
    return tuple(int(x) for x in out)


class Instance:
    """A reference (tree, PagePool, queries) triple held inside _ref."""

    def __init__(self, h):
        if not h:
            raise RuntimeError(_err())
        self._h = h

    @classmethod
    def synth(cls, snap, d_head, n_heads, seed):
        args, keep = _snap_args(snap)
        return cls(lib().ref_instance_new(*args, d_head, n_heads, seed))

    @classmethod
    def gqa(cls, snap, d_head, h_q, h_kv, seed):
        args, keep = _snap_args(snap)
        return cls(lib().ref_instance_new_gqa(*args, d_head, h_q, h_kv, seed))

    @classmethod
    def from_content(cls, snap, d_head, n_heads, keys: dict, values: dict, q: np.ndarray):
        args, keep = _snap_args(snap)
        ids = sorted(int(i) for i in snap[1])
        dim = d_head * n_heads
        K = np.ascontiguousarray(np.concatenate([keys[i].reshape(-1, dim) for i in ids]), np.float32)
        V = np.ascontiguousarray(np.concatenate([values[i].reshape(-1, dim) for i in ids]), np.float32)
        Q = np.ascontiguousarray(q, np.float32)
        return cls(lib().ref_instance_new_content(*args, d_head, n_heads, _p(K, f32p), _p(V, f32p), _p(Q, f32p)))

    def __del__(self):
        if getattr(self, "_h", None):
            lib().ref_instance_free(self._h)
            self._h = None

    @property
    def dim(self):
        return lib().ref_instance_dim(self._h)

    def leaves(self):
        n = lib().ref_instance_leaves(self._h, None)
        out = np.zeros(n, np.int32)
        lib().ref_instance_leaves(self._h, _p(out, i32p))
        return out

    def node_kv(self, node, n_tokens):
        k = np.zeros((n_tokens, self.dim), np.float32)
        v = np.zeros((n_tokens, self.dim), np.float32)
        if lib().ref_instance_node_kv(self._h, node, _p(k, f32p), _p(v, f32p)) < 0:
            raise RuntimeError(_err())
        return k, v

    def queries(self):
        q = np.zeros((len(self.leaves()), self.dim), np.float32)
        lib().ref_instance_queries(self._h, _p(q, f32p))
        return q

    def run_iteration(self, block_size=128, use_double=False, tile_size=32, strategy="flatten"):
        L = len(self.leaves())
        out = np.zeros((L, self.dim), np.float64)
        present = np.zeros(L, np.uint8)
        secs = C.c_double()
        if lib().ref_run_iteration(self._h, strategy.encode(), block_size, int(use_double), tile_size,
                                   _p(out, f64p), _p(present, u8p), C.byref(secs)) != 0:
            raise RuntimeError(_err())
        return out, present.astype(bool), secs.value

    def naive(self):
        out = np.zeros((len(self.leaves()), self.dim), np.float64)
        secs = C.c_double()
        if lib().ref_naive(self._h, _p(out, f64p), C.byref(secs)) != 0:
            raise RuntimeError(_err())
        return out, secs.value


def fill_uniform(n, seed):
    v = np.zeros(n, np.float32)
    lib().ref_fill_uniform(_p(v, f32p), n, seed)
    return v


def content_seed(seed, a, b):
    return lib().ref_content_seed(seed, a, b)


def set_threads(n):
    lib().ref_set_threads(n)


def tune_malloc():
    lib().ref_tune_malloc()
