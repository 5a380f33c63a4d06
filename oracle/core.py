"""ctypes wrapper over liboracle.so -- the C restatement of the reference.

TEST INFRASTRUCTURE ONLY.  Each helper names the reference function it
restates (paths relative to /root/reference/proj/include/treeattn/).
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
u64p = C.POINTER(C.c_uint64)
f32p = C.POINTER(C.c_float)
f64p = C.POINTER(C.c_double)
u8p = C.POINTER(C.c_uint8)


class _Rng(C.Structure):
    _fields_ = [("mt", C.c_uint64 * 312), ("idx", C.c_int)]


class _Plan(C.Structure):
    _fields_ = [
        ("n_groups", C.c_int), ("block_size", C.c_int),
        ("group_id", C.POINTER(C.c_int)), ("seg_begin", C.POINTER(C.c_int)),
        ("q_begin", C.POINTER(C.c_int)), ("seg_node", i32p), ("seg_offset", i64p),
        ("seg_len", i64p), ("seg_mask", u64p), ("queries", i32p),
        ("seg_cap", C.c_int), ("q_cap", C.c_int), ("g_cap", C.c_int),
    ]


class _Kv(C.Structure):
    _fields_ = [("dim", C.c_int), ("n_nodes", C.c_int),
                ("keys", C.POINTER(f32p)), ("values", C.POINTER(f32p))]


def build() -> str:
    """Compile liboracle.so with oracle/Makefile (gcc is in the image)."""
    subprocess.run(["make", "-s", "-C", _HERE, "liboracle.so"], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is not None:
        return _lib
    src = os.path.join(_HERE, "treeattn_oracle.c")
    if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        build()
    L = C.CDLL(_LIB_PATH)
    sig = {
        "to_rng_seed": (None, [C.POINTER(_Rng), C.c_uint64]),
        "to_rng_next": (C.c_uint64, [C.POINTER(_Rng)]),
        "to_rng_uniform_float": (C.c_float, [C.POINTER(_Rng), C.c_float, C.c_float]),
        "to_rng_uniform_int": (C.c_int64, [C.POINTER(_Rng), C.c_int64, C.c_int64]),
        "to_mix64": (C.c_uint64, [C.c_uint64]),
        "to_content_seed": (C.c_uint64, [C.c_uint64, C.c_uint64, C.c_uint64]),
        "to_fill_uniform": (None, [f32p, C.c_int64, C.c_uint64]),
        "to_fill_node_kv": (None, [C.c_int32, C.c_int64, C.c_int64, C.c_int, C.c_uint64, f32p, f32p]),
        "to_fill_query": (None, [C.c_int32, C.c_int, C.c_uint64, f32p]),
        "to_tree_new": (C.c_void_p, [C.c_int64]),
        "to_tree_restore": (C.c_void_p, [C.c_int32, C.c_int, i32p, i32p, i64p]),
        "to_tree_free": (None, [C.c_void_p]),
        "to_tree_branch": (C.c_int, [C.c_void_p, C.c_int32, C.c_int, i64p, i32p]),
        "to_tree_prune": (C.c_int, [C.c_void_p, C.c_int32]),
        "to_tree_append": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64]),
        "to_tree_root": (C.c_int32, [C.c_void_p]),
        "to_tree_node_count": (C.c_int, [C.c_void_p]),
        "to_tree_n_leaves": (C.c_int, [C.c_void_p]),
        "to_tree_leaves": (i32p, [C.c_void_p]),
        "to_tree_total_tokens": (C.c_int64, [C.c_void_p]),
        "to_tree_path_tokens": (C.c_int64, [C.c_void_p, C.c_int32]),
        "to_tree_token_count": (C.c_int64, [C.c_void_p, C.c_int32]),
        "to_tree_parent": (C.c_int32, [C.c_void_p, C.c_int32]),
        "to_tree_snapshot": (C.c_int, [C.c_void_p, i32p, i32p, i64p]),
        "to_tree_dfs": (C.c_int, [C.c_void_p, i32p]),
        "to_random_tree": (C.c_void_p, [C.POINTER(_Rng), C.c_int, C.c_int64, C.c_int64, C.c_int, C.c_int]),
        "to_partition_flatten": (C.POINTER(_Plan), [C.c_void_p, C.c_int]),
        "to_plan_free": (None, [C.POINTER(_Plan)]),
        "to_run_iteration_flatten": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(f32p), C.POINTER(_Kv),
                                               C.c_int, C.c_int, C.c_int, C.c_int, f64p, u8p]),
        "to_naive_attention": (None, [C.c_void_p, C.POINTER(f32p), C.POINTER(_Kv), C.c_int, C.c_int, f64p]),
        "to_relative_error": (C.c_double, [f64p, f64p, C.c_int64]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def _p(a, t):
    return a.ctypes.data_as(t)


# ---------------------------------------------------------------------------
# RNG (std::mt19937_64 + libstdc++ distributions)
class Rng:
    def __init__(self, seed: int):
        self._s = _Rng()
        lib().to_rng_seed(C.byref(self._s), C.c_uint64(seed))

    def next(self) -> int:
        return lib().to_rng_next(C.byref(self._s))

    def uniform_int(self, a: int, b: int) -> int:
        return lib().to_rng_uniform_int(C.byref(self._s), a, b)

    def uniform_float(self, a: float, b: float) -> float:
        return lib().to_rng_uniform_float(C.byref(self._s), a, b)


# ---------------------------------------------------------------------------
# DecodingTree (tree.hpp:38-269)
class TreeError(Exception):
    pass


def _check(rc, what):
    if rc == -1:
        raise ValueError(f"{what}: invalid_argument")
    if rc == -2:
        raise KeyError(f"{what}: out_of_range")
    if rc != 0:
        raise TreeError(f"{what}: error {rc}")


class Tree:
    def __init__(self, root_tokens: int | None = None, _ptr=None):
        if _ptr is None:
            _ptr = lib().to_tree_new(int(root_tokens))
            if not _ptr:
                raise ValueError("new_tree: root_token_count must be >= 1")
        self._t = _ptr

    @classmethod
    def restore(cls, root, ids, parents, counts):
        ids = np.ascontiguousarray(ids, np.int32)
        parents = np.ascontiguousarray(parents, np.int32)
        counts = np.ascontiguousarray(counts, np.int64)
        p = lib().to_tree_restore(int(root), len(ids), _p(ids, i32p), _p(parents, i32p), _p(counts, i64p))
        if not p:
            raise ValueError("restore: invalid snapshot")
        return cls(_ptr=p)

    @classmethod
    def from_snapshot(cls, snap):
        return cls.restore(*snap)

    def __del__(self):
        if getattr(self, "_t", None):
            lib().to_tree_free(self._t)
            self._t = None

    def branch(self, at, counts):
        counts = np.ascontiguousarray(counts, np.int64)
        out = np.zeros(len(counts), np.int32)
        _check(lib().to_tree_branch(self._t, int(at), len(counts), _p(counts, i64p), _p(out, i32p)), "branch")
        return [int(x) for x in out]

    def prune(self, at):
        _check(lib().to_tree_prune(self._t, int(at)), "prune")

    def append_tokens(self, leaf, n):
        _check(lib().to_tree_append(self._t, int(leaf), int(n)), "append_tokens")

    @property
    def root(self) -> int:
        return lib().to_tree_root(self._t)

    def leaves(self) -> np.ndarray:
        n = lib().to_tree_n_leaves(self._t)
        ptr = lib().to_tree_leaves(self._t)
        return np.ctypeslib.as_array(ptr, shape=(n,)).copy() if n else np.zeros(0, np.int32)

    def node_count(self) -> int:
        return lib().to_tree_node_count(self._t)

    def total_tokens(self) -> int:
        return lib().to_tree_total_tokens(self._t)

    def path_tokens(self, leaf) -> int:
        return lib().to_tree_path_tokens(self._t, int(leaf))

    def token_count(self, node) -> int:
        return lib().to_tree_token_count(self._t, int(node))

    def parent(self, node) -> int:
        return lib().to_tree_parent(self._t, int(node))

    def snapshot(self):
        n = lib().to_tree_snapshot(self._t, None, None, None)
        ids = np.zeros(n, np.int32)
        par = np.zeros(n, np.int32)
        cnt = np.zeros(n, np.int64)
        lib().to_tree_snapshot(self._t, _p(ids, i32p), _p(par, i32p), _p(cnt, i64p))
        return (self.root, ids, par, cnt)

    def depth_first_order(self) -> np.ndarray:
        n = self.node_count()
        out = np.zeros(n, np.int32)
        lib().to_tree_dfs(self._t, _p(out, i32p))
        return out

    def shared_factor(self):
        total = self.total_tokens()
        paths = sum(self.path_tokens(l) for l in self.leaves())
        return paths, total


def random_tree(rng: Rng, max_leaves=64, max_tokens=8192, max_node_tokens=400,
                max_branch_width=4, mutation_steps=24) -> Tree:
    """synth.hpp:80-111 (RandomTreeConfig defaults synth.hpp:71-77)."""
    p = lib().to_random_tree(C.byref(rng._s), max_leaves, max_tokens, max_node_tokens,
                             max_branch_width, mutation_steps)
    return Tree(_ptr=p)


# ---------------------------------------------------------------------------
# content (synth.hpp:20-69)
def fill_uniform(n: int, seed: int) -> np.ndarray:
    v = np.zeros(n, np.float32)
    lib().to_fill_uniform(_p(v, f32p), n, C.c_uint64(seed))
    return v


def node_kv(node: int, n_tokens: int, dim: int, seed: int, t0: int = 0):
    k = np.zeros((n_tokens, dim), np.float32)
    v = np.zeros((n_tokens, dim), np.float32)
    if n_tokens:
        lib().to_fill_node_kv(node, t0, n_tokens, dim, C.c_uint64(seed), _p(k, f32p), _p(v, f32p))
    return k, v


def query(leaf: int, dim: int, seed: int) -> np.ndarray:
    q = np.zeros(dim, np.float32)
    lib().to_fill_query(leaf, dim, C.c_uint64(seed), _p(q, f32p))
    return q


class Content:
    """Per-node K/V rows ([token_count][dim] fp32) and per-leaf queries.

    ``synth(tree, dim, seed)`` reproduces fill_tree_kv + make_queries
    (synth.hpp:52-69).  ``gqa(tree, d, h_q, h_kv, seed)`` generates K/V at
    h_kv*d and queries at h_q*d (the GQA oracle extension)."""

    def __init__(self, keys: dict, values: dict, queries: dict, dim: int):
        self.keys, self.values, self.queries, self.dim = keys, values, queries, dim

    @classmethod
    def synth(cls, tree: Tree, dim: int, seed: int, qdim: int | None = None):
        root, ids, par, cnt = tree.snapshot()
        keys, values = {}, {}
        for i, c in zip(ids, cnt):
            keys[int(i)], values[int(i)] = node_kv(int(i), int(c), dim, seed)
        qd = dim if qdim is None else qdim
        queries = {int(l): query(int(l), qd, seed) for l in tree.leaves()}
        return cls(keys, values, queries, dim)

    def expanded(self, d_head: int, h_q: int, h_kv: int) -> "Content":
        """GQA -> MHA expansion: q head h reads kv head h // (h_q/h_kv)."""
        g = h_q // h_kv
        idx = np.concatenate([np.arange(d_head) + (h // g) * d_head for h in range(h_q)])
        k = {n: np.ascontiguousarray(a[:, idx]) for n, a in self.keys.items()}
        v = {n: np.ascontiguousarray(a[:, idx]) for n, a in self.values.items()}
        return Content(k, v, self.queries, h_q * d_head)

    def map(self, fn) -> "Content":
        return Content({n: fn(a) for n, a in self.keys.items()},
                       {n: fn(a) for n, a in self.values.items()},
                       {n: fn(a) for n, a in self.queries.items()}, self.dim)

    def _kv_struct(self):
        n = max(self.keys) + 1 if self.keys else 1
        kp = (f32p * n)()
        vp = (f32p * n)()
        keep = []
        for i in range(n):
            if i in self.keys:
                k = np.ascontiguousarray(self.keys[i], np.float32)
                v = np.ascontiguousarray(self.values[i], np.float32)
                keep += [k, v]
                kp[i] = _p(k, f32p)
                vp[i] = _p(v, f32p)
        kv = _Kv(self.dim, n, C.cast(kp, C.POINTER(f32p)), C.cast(vp, C.POINTER(f32p)))
        return kv, keep + [kp, vp]

    def _q_table(self, tree: Tree):
        n = max(int(x) for x in tree.snapshot()[1]) + 1
        tab = (f32p * n)()
        keep = []
        for l, q in self.queries.items():
            if q is None:
                continue
            a = np.ascontiguousarray(q, np.float32)
            keep.append(a)
            tab[l] = _p(a, f32p)
        return C.cast(tab, C.POINTER(f32p)), keep + [tab]

    def q_matrix(self, tree: Tree) -> np.ndarray:
        return np.stack([self.queries[int(l)] for l in tree.leaves()]).astype(np.float32)


# ---------------------------------------------------------------------------
# partition_flatten (partition.hpp:212-253) + plan_to_json (serde.hpp:41-61)
def partition_flatten(tree: Tree, block_size: int = 128):
    P = lib().to_partition_flatten(tree._t, block_size)
    if not P:
        raise ValueError("partition: block_size must be >= 1")
    p = P.contents
    groups = []
    for g in range(p.n_groups):
        s0, s1 = p.seg_begin[g], p.seg_begin[g + 1]
        q0, q1 = p.q_begin[g], p.q_begin[g + 1]
        groups.append({
            "id": p.group_id[g],
            "segments": [(p.seg_node[s], p.seg_offset[s], p.seg_len[s]) for s in range(s0, s1)],
            "queries": [p.queries[q] for q in range(q0, q1)],
            "masks": [p.seg_mask[s] for s in range(s0, s1)],
        })
    lib().to_plan_free(P)
    return {"strategy": "flatten", "block_size": block_size, "groups": groups}


def plan_to_json(plan) -> str:
    """Byte-identical to nlohmann's plan_to_json(plan).dump()."""
    obj = {
        "strategy": plan["strategy"],
        "block_size": plan["block_size"],
        "groups": [{
            "id": g["id"],
            "segments": [{"node": n, "offset": o, "len": l} for (n, o, l) in g["segments"]],
            "queries": list(g["queries"]),
            "masks": ["%016x" % m for m in g["masks"]],
        } for g in plan["groups"]],
    }
    return json.dumps(obj, separators=(",", ":"), sort_keys=True)


def io_measured(plan, d_head, n_heads, n_layers, dtype_bytes):
    """io_model.hpp:158-170 -> (kv, q, mask, partial) bytes."""
    u = n_heads * n_layers * dtype_bytes
    kv = q = mask = 0
    for g in plan["groups"]:
        kv += 2 * d_head * sum(s[2] for s in g["segments"]) * u
        q += len(g["queries"]) * d_head * u
        mask += len(g["segments"]) * 8 * n_layers
    return kv, q, mask, 0


# ---------------------------------------------------------------------------
# attention (attention.hpp:117-346)
def run_iteration_flatten(tree: Tree, content: Content, d_head: int, n_heads: int,
                          block_size: int = 128, tile_size: int = 32, use_double: bool = False):
    """Returns (out [L][dim] fp64 in leaves() order, present [L] bool)."""
    L = len(tree.leaves())
    dim = d_head * n_heads
    out = np.zeros((L, dim), np.float64)
    present = np.zeros(L, np.uint8)
    kv, keep1 = content._kv_struct()
    qt, keep2 = content._q_table(tree)
    rc = lib().to_run_iteration_flatten(tree._t, block_size, qt, C.byref(kv), d_head, n_heads,
                                        tile_size, int(use_double), _p(out, f64p), _p(present, u8p))
    _check(rc, "run_iteration")
    del keep1, keep2
    return out, present.astype(bool)


def naive_attention(tree: Tree, content: Content, d_head: int, n_heads: int) -> np.ndarray:
    L = len(tree.leaves())
    out = np.zeros((L, d_head * n_heads), np.float64)
    kv, keep1 = content._kv_struct()
    qt, keep2 = content._q_table(tree)
    lib().to_naive_attention(tree._t, qt, C.byref(kv), d_head, n_heads, _p(out, f64p))
    del keep1, keep2
    return out


def relative_error(got, ref) -> float:
    """attention.hpp:337-346 (max|got-ref| / (max|ref| + 1e-12))."""
    got = np.asarray(got, np.float64).ravel()
    ref = np.asarray(ref, np.float64).ravel()
    return float(np.max(np.abs(got - ref), initial=0.0) / (np.max(np.abs(ref), initial=0.0) + 1e-12))


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 -> fp32 (the bf16 oracle input, §8c)."""
    a = np.ascontiguousarray(a, np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).reshape(a.shape)
