"""ctypes front-end for the parity checkers.  TEST INFRASTRUCTURE ONLY.

Two checkers, both CPU:

* ``Oracle``    -- oracle/mas_oracle.c, a plain-C restatement of the
  reference's maximum-path call (parallel.cpp, reference.cpp, backtrack.hpp,
  types.cpp validation, bench.cpp generator).  Always buildable.
* ``Reference`` -- the UNMODIFIED reference engines compiled in place from
  /root/reference/proj/src by oracle/Makefile into oracle/_ref/.  Present
  only where the reference sources were available at build time (this
  container; the built .so travels to the GPU box).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
``--impl reference``) may import this module.  The product package
(paper_2409_07704_b200) never does.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libmas_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmonoalign_ref.so")
REF_SRC = "/root/reference/proj"

# include/monoalign/errors.hpp:8-30, declaration order.
ERRC_NAMES = [
    "ZeroDim", "InfeasibleLengths", "LengthsOutOfRange", "NonFinite", "SpeechTooLong",
    "ShapeMismatch", "InvalidPath", "InvalidMatrix", "InvalidConfig", "TooLarge",
    "EmptyReport", "InsufficientPoints", "IoFailure", "BadMagic", "UnsupportedVersion",
    "TruncatedFile", "DimensionOverflow",
]


def build(force: bool = False) -> None:
    """Build the C oracle, and -- when the reference sources exist -- the
    reference .so and the drop-in programs (the reference's own binding and
    test suites compiled against include/monoalign/ + libmonoalign_b200.so;
    the product library must be built first)."""
    targets = ["oracle"]
    if os.path.isdir(REF_SRC):
        targets += ["ref", "dropin"]
    if not os.path.isdir(REF_SRC) and os.path.exists(ORACLE_SO) and not force:
        return  # GPU box: use the prebuilt checkers that travelled with the repo
    import sysconfig

    import pybind11

    pyinc = f"-I{pybind11.get_include()} -I{sysconfig.get_paths()['include']}"
    ext = sysconfig.get_config_var("EXT_SUFFIX")
    subprocess.run(["make", "-s", "-C", HERE] + (["clean"] if force else []) + targets
                   + [f"PYINC={pyinc}", f"EXT={ext}"], check=True)


class _OracleError(ctypes.Structure):
    _fields_ = [("errc", ctypes.c_int32), ("item", ctypes.c_int32),
                ("i", ctypes.c_int64), ("j", ctypes.c_int64)]


_F32P = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")


def _lengths_u32(lengths, B):
    if lengths is None:
        return None
    arr = np.ascontiguousarray(np.asarray(lengths, dtype=np.int64).reshape(B, 2)).astype(np.uint32)
    return arr


class Oracle:
    """The C restatement (oracle/mas_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        lib = ctypes.CDLL(path)
        lib.oracle_align.restype = ctypes.c_int
        lib.oracle_align.argtypes = [
            ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
            ctypes.c_float, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.POINTER(_OracleError)]
        lib.oracle_generate.restype = None
        lib.oracle_generate.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64,
                                        ctypes.c_void_p]
        lib.oracle_mix_seed.restype = ctypes.c_uint64
        lib.oracle_mix_seed.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        lib.oracle_splitmix64.restype = ctypes.c_uint64
        lib.oracle_splitmix64.argtypes = [ctypes.POINTER(ctypes.c_uint64)]
        lib.oracle_validate_config.restype = ctypes.c_int
        lib.oracle_validate_config.argtypes = [ctypes.c_float, ctypes.c_int]
        lib.oracle_forward_parallel.restype = None
        lib.oracle_forward_parallel.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                                ctypes.c_ssize_t, ctypes.c_float]
        self.lib = lib

    def align(self, q, lengths=None, engine="parallel", max_neg_val=-1e32, unchecked=False,
              want_out=True, want_paths=True):
        """Returns (errc, item, (i, j), out[B,T,S] u8, paths[B,S] i32)."""
        q = np.ascontiguousarray(q, dtype=np.float32)
        if q.ndim == 2:
            q = q[None]
        B, T, S = q.shape
        if not unchecked:
            code = self.lib.oracle_validate_config(ctypes.c_float(max_neg_val), 0)
            if code >= 0:
                return code, -1, (-1, -1), None, None
        lens = _lengths_u32(lengths, B)
        out = np.zeros((B, T, S), np.uint8) if want_out else None
        paths = np.full((B, S), -1, np.int32) if want_paths else None
        err = _OracleError()
        code = self.lib.oracle_align(
            q.ctypes.data, B, T, S, None if lens is None else lens.ctypes.data,
            ctypes.c_float(max_neg_val), 1 if engine == "reference" else 0,
            None if out is None else out.ctypes.data,
            None if paths is None else paths.ctypes.data, ctypes.byref(err))
        return code, err.item, (err.i, err.j), out, paths

    def generate(self, b, t, s, seed, first_item=0):
        """bench::generate_random_batch(b, t, s, seed) restated; `first_item`
        selects the shard starting at that item of a larger batch."""
        out = np.empty((b, t, s), np.float32)
        self.lib.oracle_generate(seed, first_item * t * s, b * t * s, out.ctypes.data)
        return out

    def mix_seed(self, seed, index):
        return int(self.lib.oracle_mix_seed(seed, index))

    def splitmix64(self, state: int):
        st = ctypes.c_uint64(state)
        v = self.lib.oracle_splitmix64(ctypes.byref(st))
        return int(v), int(st.value)

    def forward_parallel(self, q, max_neg_val=-1e32):
        q = np.array(q, dtype=np.float32, copy=True, order="C")
        t, s = q.shape
        self.lib.oracle_forward_parallel(q.ctypes.data, t, s, s, ctypes.c_float(max_neg_val))
        return q


class Reference:
    """The reference engines themselves (oracle/_ref/libmonoalign_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        lib = ctypes.CDLL(path)
        lib.ref_align.restype = ctypes.c_int
        lib.ref_align.argtypes = [
            ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
            ctypes.c_int, ctypes.c_float, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
            ctypes.c_void_p, ctypes.c_char_p, ctypes.c_int]
        lib.ref_generate.restype = ctypes.c_int
        lib.ref_generate.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_uint64,
                                     ctypes.c_void_p]
        lib.ref_best_paths.restype = ctypes.c_int
        lib.ref_best_paths.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                       ctypes.POINTER(ctypes.c_double),
                                       ctypes.POINTER(ctypes.c_int), ctypes.c_void_p,
                                       ctypes.c_int]
        lib.ref_hardware_threads.restype = ctypes.c_uint
        lib.ref_forward_parallel.restype = None
        lib.ref_forward_parallel.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                             ctypes.c_int64, ctypes.c_float]
        lib.ref_forward_reference.restype = None
        lib.ref_forward_reference.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                              ctypes.c_int64, ctypes.c_float, ctypes.c_void_p]
        lib.ref_batch_create.restype = ctypes.c_void_p
        lib.ref_batch_create.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_uint64]
        lib.ref_batch_destroy.restype = None
        lib.ref_batch_destroy.argtypes = [ctypes.c_void_p]
        lib.ref_batch_time_align.restype = ctypes.c_double
        lib.ref_batch_time_align.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                             ctypes.POINTER(ctypes.c_int64)]
        lib.ref_tensor_write.restype = ctypes.c_int
        lib.ref_tensor_write.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_char_p, ctypes.c_int]
        lib.ref_tensor_read.restype = ctypes.c_int
        lib.ref_tensor_read.argtypes = [ctypes.c_char_p, ctypes.c_uint64,
                                        ctypes.POINTER(ctypes.c_int),
                                        ctypes.POINTER(ctypes.c_int64 * 3), ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_char_p, ctypes.c_int]
        self.lib = lib

    def forward_parallel(self, q, t=None, s=None, max_neg_val=-1e32):
        """parallel::forward_parallel on a copy of the 2-D item q (its [t, s] region)."""
        q = np.array(q, dtype=np.float32, copy=True, order="C")
        T, S = q.shape
        self.lib.ref_forward_parallel(q.ctypes.data, T if t is None else t, S if s is None else s,
                                      S, ctypes.c_float(max_neg_val))
        return q

    def forward_reference(self, q, max_neg_val=-1e32):
        """reference::forward_reference of the 2-D item q: its QCache as [t, s]."""
        q = np.ascontiguousarray(q, dtype=np.float32)
        T, S = q.shape
        out = np.empty((T, S), np.float32)
        self.lib.ref_forward_reference(q.ctypes.data, T, S, S, ctypes.c_float(max_neg_val),
                                       out.ctypes.data)
        return out

    def write_tensor(self, path, values, lengths=None):
        """io::write_tensor (tensor_io.cpp).  Returns (errc, message); -1 = ok."""
        v = np.ascontiguousarray(values)
        if v.ndim == 2:
            v = v[None]
        B, T, S = v.shape
        lens = None if lengths is None else np.ascontiguousarray(lengths, dtype=np.uint32)
        msg = ctypes.create_string_buffer(512)
        rc = self.lib.ref_tensor_write(os.fsencode(path), 0 if v.dtype == np.float32 else 1, B, T,
                                       S, v.ctypes.data,
                                       None if lens is None else lens.ctypes.data, msg, 512)
        return rc, msg.value.decode()

    def read_tensor(self, path, budget=1 << 30):
        """io::read_tensor.  Returns (errc, message, values, lengths)."""
        msg = ctypes.create_string_buffer(512)
        dtype = ctypes.c_int()
        dims = (ctypes.c_int64 * 3)()
        rc = self.lib.ref_tensor_read(os.fsencode(path), budget, ctypes.byref(dtype),
                                      ctypes.byref(dims), None, None, msg, 512)
        if rc != -1:
            return rc, msg.value.decode(), None, None
        vals = np.empty(tuple(dims), np.float32 if dtype.value == 0 else np.uint8)
        lens = np.empty((dims[0], 2), np.uint32)
        rc = self.lib.ref_tensor_read(os.fsencode(path), budget, ctypes.byref(dtype),
                                      ctypes.byref(dims), vals.ctypes.data, lens.ctypes.data,
                                      msg, 512)
        return rc, msg.value.decode(), vals, lens

    @staticmethod
    def available(path: str = REF_SO) -> bool:
        return os.path.exists(path)

    def align(self, q, lengths=None, engine="parallel", max_neg_val=-1e32, threads=0,
              unchecked=False, want_out=True, want_paths=False):
        """Returns (errc, message, out, paths); errc -1 on success."""
        q = np.ascontiguousarray(q, dtype=np.float32)
        if q.ndim == 2:
            q = q[None]
        B, T, S = q.shape
        lens = None
        if lengths is not None:
            lens = np.ascontiguousarray(np.asarray(lengths, dtype=np.int64).reshape(B, 2))
        out = np.zeros((B, T, S), np.uint8) if want_out else None
        paths = np.full((B, S), -1, np.int32) if want_paths else None
        msg = ctypes.create_string_buffer(1024)
        code = self.lib.ref_align(
            q.ctypes.data, B, T, S, None if lens is None else lens.ctypes.data,
            1 if engine == "reference" else 0, ctypes.c_float(max_neg_val), threads,
            1 if unchecked else 0, None if out is None else out.ctypes.data,
            None if paths is None else paths.ctypes.data, msg, len(msg))
        return code, msg.value.decode(), out, paths

    def generate(self, b, t, s, seed):
        out = np.empty((b, t, s), np.float32)
        code = self.lib.ref_generate(b, t, s, seed, out.ctypes.data)
        if code >= 0:
            raise ValueError(ERRC_NAMES[code])
        return out

    def best_paths(self, q, cap=16):
        q = np.ascontiguousarray(q, dtype=np.float32)
        t, s = q.shape
        score = ctypes.c_double()
        n = ctypes.c_int()
        paths = np.zeros((cap, s), np.int32)
        code = self.lib.ref_best_paths(q.ctypes.data, t, s, ctypes.byref(score), ctypes.byref(n),
                                       paths.ctypes.data, cap)
        if code >= 0:
            raise ValueError(ERRC_NAMES[code])
        return score.value, paths[: min(n.value, cap)], n.value

    def timed_batch(self, b, t, s, seed):
        """A pre-built generate_random_batch(b, t, s, seed) inside the
        reference library; call .time(engine, threads) -> ms per align."""
        ref = self

        class _Batch:
            def __init__(self):
                self.h = ref.lib.ref_batch_create(b, t, s, seed)
                if not self.h:
                    raise MemoryError("ref_batch_create failed")

            def time(self, engine="parallel", threads=0):
                ck = ctypes.c_int64()
                ms = ref.lib.ref_batch_time_align(self.h, 1 if engine == "reference" else 0,
                                                  threads, ctypes.byref(ck))
                if ms < 0:
                    raise RuntimeError("reference align failed")
                return ms

            def close(self):
                if self.h:
                    ref.lib.ref_batch_destroy(self.h)
                    self.h = None

        return _Batch()

    def hardware_threads(self) -> int:
        return int(self.lib.ref_hardware_threads())
