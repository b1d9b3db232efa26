"""ctypes binding of include/turboreg.h (same names; argument marshalling only).

Inputs may be numpy arrays (host) or CUDA torch tensors (device pointers + the current torch stream).
Every step of the path runs inside ``libturboreg.so``; this module never computes any part of it.
"""
from __future__ import annotations

import ctypes
import enum
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# TURBOREG_LIBRARY selects another in-tree build (the tests' checked build, lib/libturboreg_checked.so)
_LIB_PATH = os.environ.get("TURBOREG_LIBRARY") or os.path.join(_HERE, "lib", "libturboreg.so")


class TurboRegError(RuntimeError):
    def __init__(self, status, what=""):
        self.status = int(status)
        super().__init__(f"turboreg: {what}: {Status(self.status).name} ({self.status})")


class Status(enum.IntEnum):
    OK = 0
    INVALID_ARGUMENT = 1
    TOO_FEW_POINTS = 2
    TOO_MANY_POINTS = 3
    NONFINITE_INPUT = 4
    NO_HYPOTHESIS = 5
    CUDA = 6
    OUT_OF_MEMORY = 7
    EDGE_CAPACITY = 8


PER_PAIR_STATUSES = (0, 2, 3, 4, 5, 8)  # statuses of a pair (the call itself succeeded)


F_STAGE_TIMING = 0x1
F_KERNEL_TIMING = 0x2
F_HYP_ERRORS = 0x4
F_RANK_MAE = 0x8
F_RANK_MSE = 0x10
F_ROW_SUMS = 0x20

SPLIT_BITS, SPLIT_EDGES, SPLIT_RESULT = 0, 1, 2

I_BITS, I_BITS_BASE, I_SC2, I_PIVOTS, I_CLIQUES, I_HYPS, I_STATE, I_ERRORS, I_EDGES, I_ROWSUM = 1, 2, 3, 4, 5, 6, 7, 8, 9, 10
METRICS = {"in": 0, "mae": 1, "mse": 2}


class Params(ctypes.Structure):
    _fields_ = [
        ("tau", ctypes.c_float),
        ("tau_base", ctypes.c_float),
        ("k1", ctypes.c_int32),
        ("k2", ctypes.c_int32),
        ("inlier_threshold", ctypes.c_float),
        ("graph_mode", ctypes.c_int32),
        ("flags", ctypes.c_uint32),
    ]


class Result(ctypes.Structure):
    _fields_ = [
        ("R", ctypes.c_float * 9),
        ("t", ctypes.c_float * 3),
        ("inlier_count", ctypes.c_int32),
        ("clique", ctypes.c_int32 * 3),
        ("clique_weight", ctypes.c_int32),
        ("num_pivots", ctypes.c_int32),
        ("num_cliques", ctypes.c_int32),
        ("hypotheses_evaluated", ctypes.c_int32),
        ("status", ctypes.c_int32),
        ("stage_ms", ctypes.c_float * 3),
        ("num_edges", ctypes.c_int64),
    ]


RESULT_DTYPE = np.dtype(
    {
        "names": ["R", "t", "inlier_count", "clique", "clique_weight", "num_pivots", "num_cliques",
                  "hypotheses_evaluated", "status", "stage_ms", "num_edges"],
        "formats": [("<f4", (9,)), ("<f4", (3,)), "<i4", ("<i4", (3,)), "<i4", "<i4", "<i4", "<i4", "<i4",
                    ("<f4", (3,)), "<i8"],
        "offsets": [0, 36, 48, 52, 64, 68, 72, 76, 80, 84, 96],
        "itemsize": 104,
    }
)
assert ctypes.sizeof(Result) == RESULT_DTYPE.itemsize == 104

HYPOTHESIS_DTYPE = np.dtype(  # turboreg_hypothesis
    {
        "names": ["clique", "clique_weight", "R", "t", "inlier_count", "slot", "mae", "mse"],
        "formats": [("<i4", (3,)), "<i4", ("<f4", (9,)), ("<f4", (3,)), "<i4", "<i4", "<f8", "<f8"],
        "offsets": [0, 12, 16, 52, 64, 68, 72, 80],
        "itemsize": 88,
    }
)

_lib = None


def library_path() -> str:
    return _LIB_PATH


def library():
    """Load libturboreg.so; raises (never falls back) when it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"{_LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(_LIB_PATH)
    P, i32, i64, u64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
    lib.turboreg_create.argtypes = [ctypes.POINTER(Params), ctypes.c_int, i32, i32, ctypes.POINTER(P)]
    lib.turboreg_create_ex.argtypes = [ctypes.POINTER(Params), ctypes.c_int, i32, i32, i64, ctypes.POINTER(P)]
    lib.turboreg_set_params.argtypes = [P, ctypes.POINTER(Params)]
    lib.turboreg_register.argtypes = [P, P, P, i32, ctypes.POINTER(Result)]
    lib.turboreg_ransac.argtypes = [P, P, P, i32, i32, ctypes.c_uint64, ctypes.POINTER(Result)]
    lib.turboreg_point_resolution.argtypes = [P, P, i32, ctypes.POINTER(ctypes.c_float)]
    lib.turboreg_register_batch.argtypes = [P, P, P, P, P, i32, P, P]
    lib.turboreg_destroy.argtypes = [P]
    lib.turboreg_destroy.restype = None
    lib.turboreg_status_string.argtypes = [ctypes.c_int]
    lib.turboreg_status_string.restype = ctypes.c_char_p
    lib.turboreg_get_intermediates.argtypes = [P, i32, i32, P, u64, ctypes.POINTER(u64)]
    lib.turboreg_pgs_from_adjacency.argtypes = [P, P, i32, i32]
    lib.turboreg_ranked_hypotheses.argtypes = [P, i32, i32, i32, P, ctypes.POINTER(i32)]
    lib.turboreg_split_begin.argtypes = [P, P, P, i32, i32, i32, P]
    lib.turboreg_split_buffer.argtypes = [P, i32, ctypes.POINTER(P), ctypes.POINTER(u64)]
    lib.turboreg_split_sc2.argtypes = [P, ctypes.POINTER(i64), P]
    lib.turboreg_split_search.argtypes = [P, P]
    lib.turboreg_split_merge.argtypes = [P, P, i32, P, P]
    lib.turboreg_profile_begin.argtypes = [P]
    lib.turboreg_profile_end.argtypes = [P, P, P, P, i32, ctypes.POINTER(i32)]
    lib.turboreg_set_option.argtypes = [P, ctypes.c_char_p, i64]
    lib.turboreg_set_option.restype = ctypes.c_int
    lib.turboreg_launch_count.argtypes = [P]
    lib.turboreg_launch_count.restype = i64
    lib.turboreg_workspace_bytes.argtypes = [P]
    lib.turboreg_workspace_bytes.restype = u64
    for name in ("turboreg_create", "turboreg_create_ex", "turboreg_set_params", "turboreg_register", "turboreg_register_batch",
                 "turboreg_get_intermediates", "turboreg_pgs_from_adjacency", "turboreg_profile_begin",
                 "turboreg_profile_end", "turboreg_point_resolution", "turboreg_ransac",
                 "turboreg_ranked_hypotheses", "turboreg_split_begin", "turboreg_split_buffer",
                 "turboreg_split_sc2", "turboreg_split_search", "turboreg_split_merge"):
        getattr(lib, name).restype = ctypes.c_int
    _lib = lib
    return lib


def _check(st, what):
    if st != 0:
        raise TurboRegError(st, what)


def _is_torch_cuda(x):
    return type(x).__module__.startswith("torch") and getattr(x, "is_cuda", False)


def _points(x, what):
    """Validate an (N, 3) point array (numpy or torch); returns N."""
    shape = tuple(x.shape)
    if len(shape) != 2 or shape[1] != 3:
        raise ValueError(f"{what} must have shape (N, 3), got {shape}")
    return int(shape[0])


def _nbytes(x):
    if type(x).__module__.startswith("torch"):
        return int(x.numel()) * int(x.element_size())
    return int(np.asarray(x).nbytes)


def _ptr(x, dtype=None):
    """(pointer, keepalive) for a numpy array or a torch tensor (host or CUDA)."""
    if type(x).__module__.startswith("torch"):
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        if dtype is not None and str(x.dtype) != "torch." + np.dtype(dtype).name:
            raise TypeError(f"expected {np.dtype(dtype).name} tensor, got {x.dtype}")
        return ctypes.c_void_p(x.data_ptr()), x
    a = np.ascontiguousarray(x, dtype=dtype)
    return a.ctypes.data_as(ctypes.c_void_p), a


class TurboReg:
    """One context (device workspace + stream) of the C ABI.

    ``TurboReg(tau, k1, k2, inlier_threshold, max_n=..., max_batch=...)`` then ``register(src, dst)`` or
    ``register_batch(src, dst, offsets, n)``.  Parameter meanings: include/turboreg.h.
    """

    def __init__(self, tau, k1=1000, k2=2, inlier_threshold=0.1, *, tau_base=0.0, graph_mode=0,
                 max_n=5000, max_batch=1, device=0, stage_timing=False, kernel_timing=False, hyp_errors=False,
                 rank_metric="in", max_edges=0, max_density=None, row_sums=False):
        """``max_edges``: per-pair O2 edge capacity (0 = complete graph, never overflows); ``max_density``
        (fraction of the max_n(max_n-1)/2 possible edges) is the same bound as a ratio.  Pairs with more
        edges report status EDGE_CAPACITY (include/turboreg.h, turboreg_create_ex)."""
        self._lib = library()
        flags = (F_STAGE_TIMING if stage_timing else 0) | (F_KERNEL_TIMING if kernel_timing else 0)
        flags |= (F_HYP_ERRORS if hyp_errors else 0) | {"in": 0, "mae": F_RANK_MAE, "mse": F_RANK_MSE}[rank_metric]
        flags |= F_ROW_SUMS if row_sums else 0
        self.params = Params(float(tau), float(tau_base), int(k1), int(k2), float(inlier_threshold),
                             int(graph_mode), flags)
        if max_density is not None:
            if not 0.0 < float(max_density) <= 1.0:
                raise ValueError("max_density must be in (0, 1]")
            max_edges = max(1, int(np.ceil(float(max_density) * max_n * (max_n - 1) / 2)))
        h = ctypes.c_void_p()
        _check(self._lib.turboreg_create_ex(ctypes.byref(self.params), int(device), int(max_n), int(max_batch),
                                            int(max_edges), ctypes.byref(h)), "create")
        self._h = h
        self.max_n, self.max_batch, self.device = int(max_n), int(max_batch), int(device)

    # ------------------------------------------------------------------------------------------ lifecycle
    def close(self):
        if getattr(self, "_h", None):
            self._lib.turboreg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def set_params(self, **kw):
        """Replace parameters (names of turboreg_params); on failure the context keeps its old ones."""
        new = Params.from_buffer_copy(self.params)
        for k, v in kw.items():
            if k not in dict(Params._fields_):
                raise TypeError(f"unknown parameter {k}")
            setattr(new, k, v)
        _check(self._lib.turboreg_set_params(self._h, ctypes.byref(new)), "set_params")
        self.params = new

    def set_option(self, name, value):
        """Tuning/test knobs of include/turboreg.h (sc2_path, heavy_min_rows, heavy_min_degree, heavy_cap)."""
        _check(self._lib.turboreg_set_option(self._h, name.encode(), int(value)), f"set_option({name})")

    # ------------------------------------------------------------------------------------------ compute
    def register(self, src, dst):
        """One pair (host numpy or device torch N×3 float32).  Returns a dict; status in ['status']."""
        n = _points(src, "src")
        if _points(dst, "dst") != n:
            raise ValueError("src and dst must have the same number of rows")
        ps, ks = _ptr(src, np.float32)
        pd, kd = _ptr(dst, np.float32)
        res = Result()
        st = self._lib.turboreg_register(self._h, ps, pd, n, ctypes.byref(res))
        if st not in PER_PAIR_STATUSES:
            raise TurboRegError(st, "register")
        return result_to_dict(res)

    def point_resolution(self, xyz):
        """Median nearest-neighbour distance of a point cloud (n×3 float32, host numpy or CUDA torch): the
        τ initialisation of P:322 is 0.25 × this."""
        n = _points(xyz, "xyz")
        p, keep = _ptr(xyz, np.float32)
        out = ctypes.c_float()
        _check(self._lib.turboreg_point_resolution(self._h, p, n, ctypes.byref(out)),
               "point_resolution")
        return float(out.value)

    def ransac(self, src, dst, iters, seed=0):
        """Equal-budget 3-point RANSAC baseline on one pair: ``iters`` <= K1·K2 sampled
        triples (counter-based SplitMix64 from ``seed``), fitted and scored like TurboCliques.  Returns the
        same dict as :meth:`register`."""
        n = _points(src, "src")
        if _points(dst, "dst") != n:
            raise ValueError("src and dst must have the same number of rows")
        ps, ks = _ptr(src, np.float32)
        pd, kd = _ptr(dst, np.float32)
        res = Result()
        st = self._lib.turboreg_ransac(self._h, ps, pd, n, int(iters), int(seed) & (2**64 - 1),
                                       ctypes.byref(res))
        if st not in PER_PAIR_STATUSES:
            raise TurboRegError(st, "ransac")
        return result_to_dict(res)

    def register_batch(self, src, dst, offsets, n, out=None, stream=None):
        """`batch` pairs; src/dst are (Σn)×3 float32 (host numpy or CUDA torch), offsets/n host arrays.

        ``out``: None → returns a numpy structured array (RESULT_DTYPE, blocking); or a CUDA torch uint8
        tensor of ≥ batch*104 bytes → asynchronous on ``stream`` (default: torch's current stream)."""
        offsets = np.ascontiguousarray(offsets, dtype=np.int64).reshape(-1)
        n = np.ascontiguousarray(n, dtype=np.int32).reshape(-1)
        batch = int(n.shape[0])
        # the C ABI cannot see buffer extents: every bound it relies on is checked here, before the call
        rows = _points(src, "src")
        if _points(dst, "dst") != rows:
            raise ValueError("src and dst must have the same number of rows")
        if offsets.shape[0] != batch or batch < 1:
            raise ValueError("offsets and n must be non-empty and of equal length")
        if (offsets < 0).any() or (n < 0).any():
            raise ValueError("offsets and n must be non-negative")
        if int((offsets + n).max()) > rows:
            raise ValueError(f"offsets + n exceed the {rows} rows of src/dst")
        if out is not None and _nbytes(out) < batch * RESULT_DTYPE.itemsize:
            raise ValueError(f"out holds {_nbytes(out)} bytes, needs {batch * RESULT_DTYPE.itemsize}")
        if out is not None and _is_torch_cuda(out) and int(out.device.index or 0) != self.device:
            raise ValueError(f"out is on {out.device}, the context on cuda:{self.device}")
        if _is_torch_cuda(src) and int(src.device.index or 0) != self.device:
            raise ValueError(f"src is on {src.device}, the context on cuda:{self.device}")
        ps, ks = _ptr(src, np.float32)
        pd, kd = _ptr(dst, np.float32)
        if stream is None and (_is_torch_cuda(src) or (out is not None and _is_torch_cuda(out))):
            import torch

            stream = torch.cuda.current_stream().cuda_stream
        sp = ctypes.c_void_p(int(stream)) if stream else None
        if out is None:
            host = np.zeros(batch, dtype=RESULT_DTYPE)
            st = self._lib.turboreg_register_batch(self._h, ps, pd, offsets.ctypes.data_as(ctypes.c_void_p),
                                                   n.ctypes.data_as(ctypes.c_void_p), batch,
                                                   host.ctypes.data_as(ctypes.c_void_p), sp)
            _check(st, "register_batch")
            return host
        po, ko = _ptr(out)
        st = self._lib.turboreg_register_batch(self._h, ps, pd, offsets.ctypes.data_as(ctypes.c_void_p),
                                               n.ctypes.data_as(ctypes.c_void_p), batch, po, sp)
        _check(st, "register_batch")
        return out

    def ranked_hypotheses(self, pair=0, metric="in", top_k=None):
        """The valid hypotheses of `pair` of the last call ranked by `metric` ("in" descending, "mae" / "mse"
        ascending; ties S desc, (i,j,z) asc) as a HYPOTHESIS_DTYPE array of at most `top_k` entries (all when
        None).  MAE/MSE ranking needs a context created with hyp_errors=True or an error rank_metric."""
        k = int(self.params.k1) * int(self.params.k2) if top_k is None else int(top_k)
        out = np.zeros(max(k, 1), HYPOTHESIS_DTYPE)
        cnt = ctypes.c_int32()
        _check(self._lib.turboreg_ranked_hypotheses(self._h, int(pair), METRICS[metric], k,
                                                    out.ctypes.data_as(ctypes.c_void_p), ctypes.byref(cnt)),
               "ranked_hypotheses")
        return out[: cnt.value]

    # ------------------------------------------------------------------------------------------ NEXT(1) split
    # One pair over several ranks (include/turboreg.h "NEXT(1)"); split.register_split drives the phases and the
    # exchanges over torch.distributed.  `stream`: a torch.cuda.Stream or raw handle (None = torch's current).
    @staticmethod
    def _stream_ptr(stream):
        if stream is None:
            import torch

            return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        return ctypes.c_void_p(int(getattr(stream, "cuda_stream", stream)))

    def split_begin(self, src, dst, rank, world, stream=None):
        """Phase 1; returns the pair status (0, or 2/3 when n is out of range: nothing else to do)."""
        n = _points(src, "src")
        if _points(dst, "dst") != n:
            raise ValueError("src and dst must have the same number of rows")
        ps, ks = _ptr(src, np.float32)
        pd, kd = _ptr(dst, np.float32)
        st = self._lib.turboreg_split_begin(self._h, ps, pd, n, int(rank), int(world), self._stream_ptr(stream))
        if st not in (0, 2, 3):
            raise TurboRegError(st, "split_begin")
        self._split_keep = (ks, kd)
        return int(st)

    def split_tensor(self, which, count=None):
        """Zero-copy torch view (int32 words; uint8 for SPLIT_RESULT) of a workspace buffer to exchange."""
        import torch

        ptr, nb = ctypes.c_void_p(), ctypes.c_size_t()
        _check(self._lib.turboreg_split_buffer(self._h, int(which), ctypes.byref(ptr), ctypes.byref(nb)),
               "split_buffer")
        if which == SPLIT_RESULT:
            typestr, n = "|u1", nb.value
        else:
            typestr, n = "<i4", nb.value // 4 if count is None else int(count)
            if n * 4 > nb.value:
                raise ValueError("count exceeds the buffer")

        class _Dev:
            pass

        d = _Dev()
        d.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr.value or 0, False),
                                      "version": 3, "strides": None, "stream": None}
        return torch.as_tensor(d, device=torch.device("cuda", self.device))

    def split_sc2(self, stream=None):
        """Phase 2 (after the bits all-reduce); returns E, the number of edge words to all-reduce."""
        e = ctypes.c_int64()
        _check(self._lib.turboreg_split_sc2(self._h, ctypes.byref(e), self._stream_ptr(stream)), "split_sc2")
        return int(e.value)

    def split_search(self, stream=None):
        """Phase 3 (after the edges all-reduce): this rank's record in split_tensor(SPLIT_RESULT)."""
        _check(self._lib.turboreg_split_search(self._h, self._stream_ptr(stream)), "split_search")

    def split_merge(self, parts, world, stream=None):
        """Phase 4: T* over the `world` gathered records (a CUDA uint8 tensor of world*104 bytes)."""
        if not _is_torch_cuda(parts) or _nbytes(parts) < int(world) * RESULT_DTYPE.itemsize:
            raise ValueError("parts must be a CUDA tensor of world result records")
        res = Result()
        _check(self._lib.turboreg_split_merge(self._h, ctypes.c_void_p(parts.data_ptr()), int(world),
                                              ctypes.byref(res), self._stream_ptr(stream)), "split_merge")
        return result_to_dict(res)

    # ------------------------------------------------------------------------------------------ test views
    def intermediate(self, pair, what):
        need = ctypes.c_size_t()
        _check(self._lib.turboreg_get_intermediates(self._h, int(pair), int(what), None, 0, ctypes.byref(need)),
               "get_intermediates")
        buf = np.zeros(max(need.value, 1), np.uint8)
        _check(self._lib.turboreg_get_intermediates(self._h, int(pair), int(what),
                                                    buf.ctypes.data_as(ctypes.c_void_p), buf.nbytes, None),
               "get_intermediates")
        buf = buf[: need.value]
        if what in (I_BITS, I_BITS_BASE):
            return buf.view(np.uint32)
        if what == I_SC2:
            v = buf.view(np.int32)
            n = int(round(np.sqrt(v.size)))
            return v.reshape(n, n)
        if what == I_PIVOTS:
            return buf.view(np.int32).reshape(-1, 3)
        if what == I_CLIQUES:
            return buf.view(np.int32).reshape(-1, 4)
        if what == I_HYPS:
            return buf.view(np.float32).reshape(-1, 16)
        if what == I_ERRORS:
            return buf.view(np.float64).reshape(-1, 2)
        if what == I_ROWSUM:
            return buf.view(np.int32)
        if what == I_EDGES:
            v = buf.view(np.uint32)
            n = int(self.intermediate(pair, I_STATE)["n"])
            return v[: n + 1].astype(np.int64), v[n + 1:]
        if what == I_STATE:
            s = buf.view(np.int64)
            keys = ["n", "W", "edges", "epos", "alpha", "c_gt", "need", "npiv", "nonfinite", "b1", "above",
                    "edges_base", "heavy_h", "heavy_thr", "deg_sum"]
            return {k: int(s[i]) for i, k in enumerate(keys)}
        return buf

    def bits(self, pair=0, base=False):
        """C(τ) (or C(τ_base)) of the last call as a dense uint8 [n, n] matrix."""
        st = self.intermediate(pair, I_STATE)
        n, W = st["n"], st["W"]
        words = self.intermediate(pair, I_BITS_BASE if base else I_BITS).reshape(n, W)
        return np.unpackbits(words.view(np.uint8), axis=1, bitorder="little")[:, :n]

    def pgs_from_adjacency(self, C):
        C = np.ascontiguousarray(C, dtype=np.uint8)
        n = C.shape[0]
        W = (n + 31) // 32
        padded = np.zeros((n, W * 32), np.uint8)
        padded[:, :n] = C
        words = np.packbits(padded, axis=1, bitorder="little").view(np.uint32)
        words = np.ascontiguousarray(words)
        _check(self._lib.turboreg_pgs_from_adjacency(self._h, words.ctypes.data_as(ctypes.c_void_p), n, W),
               "pgs_from_adjacency")

    # ------------------------------------------------------------------------------------------ profiling
    def profile_begin(self):
        _check(self._lib.turboreg_profile_begin(self._h), "profile_begin")

    def profile_end(self):
        cap = 32
        names = (ctypes.c_char_p * cap)()
        ms = (ctypes.c_float * cap)()
        launches = (ctypes.c_int64 * cap)()
        cnt = ctypes.c_int32()
        _check(self._lib.turboreg_profile_end(self._h, names, ms, launches, cap, ctypes.byref(cnt)), "profile_end")
        return {names[k].decode(): (float(ms[k]), int(launches[k])) for k in range(cnt.value)}

    @property
    def launch_count(self):
        return int(self._lib.turboreg_launch_count(self._h))

    @property
    def workspace_bytes(self):
        return int(self._lib.turboreg_workspace_bytes(self._h))


def result_to_dict(r):
    if isinstance(r, np.void) or (isinstance(r, np.ndarray) and r.dtype == RESULT_DTYPE):
        return {k: (r[k].copy() if np.ndim(r[k]) else r[k].item()) for k in RESULT_DTYPE.names}
    return {
        "R": np.array(r.R, np.float32).reshape(3, 3),
        "t": np.array(r.t, np.float32),
        "inlier_count": r.inlier_count,
        "clique": tuple(r.clique),
        "clique_weight": r.clique_weight,
        "num_pivots": r.num_pivots,
        "num_cliques": r.num_cliques,
        "hypotheses_evaluated": r.hypotheses_evaluated,
        "status": r.status,
        "stage_ms": tuple(r.stage_ms),
        "num_edges": r.num_edges,
    }
