"""Python surface of the drop-in: the reference's ``monoalign`` functions.

Mirrors the pybind11 binding ``_monoalign`` (bindings/module.cpp:206-247 of
the reference) call for call -- same names, keyword arguments, defaults,
argument conversion, check order and exception types -- but every alignment
is computed by the sm_100a kernels behind the C-ABI
(include/monoalign_b200.h).  Additionally accepts torch CUDA tensors, which
stay on the device (no host copy).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _lib

__version__ = "1.0.0"  # MONOALIGN_VERSION, tests/python/test_smoke.py:9-10

_DEFAULT_MAX_NEG_VAL = float(np.float32(-1e32))  # kDefaultMaxNegVal, types.hpp:19


def _is_torch(x) -> bool:
    mod = type(x).__module__
    return mod.startswith("torch")


# ---- module.cpp:21-35 make_config ------------------------------------------
def _make_config(engine: str, max_neg_val: float, threads: int, unchecked: bool = False):
    # MasConfig defaults (mas_config_default), filled here without a C call
    cfg = _lib.MasConfig(_lib.MAS_ENGINE_PARALLEL, _DEFAULT_MAX_NEG_VAL, 0, 0, 0)
    if engine == "reference":
        cfg.engine = _lib.MAS_ENGINE_REFERENCE
    elif engine == "parallel":
        cfg.engine = _lib.MAS_ENGINE_PARALLEL
    else:
        raise ValueError("unknown engine name: " + str(engine))
    cfg.max_neg_val = float(max_neg_val)  # double -> float, module.cpp:32
    cfg.threads = int(threads)
    cfg.flags = _lib.MAS_FLAG_UNCHECKED if unchecked else 0
    return cfg


# ---- module.cpp:44-59 check_dims -------------------------------------------
def _check_dims(shape):
    if len(shape) not in (2, 3):
        raise ValueError("values must be a [T, S] or [B, T, S] array")
    was_2d = len(shape) == 2
    b = 1 if was_2d else int(shape[0])
    t = int(shape[0 if was_2d else 1])
    s = int(shape[1 if was_2d else 2])
    if b < 1 or t < 1 or s < 1:
        raise ValueError("every array dimension must be at least 1")
    return was_2d, b, t, s


# ---- module.cpp:61-84 parse_lengths ----------------------------------------
def _parse_lengths(lengths, b, t, s):
    if _is_torch(lengths):
        lengths = lengths.detach().cpu().numpy()
    arr = np.ascontiguousarray(np.asarray(lengths), dtype=np.int64)
    flat_pair = arr.ndim == 1 and arr.shape[0] == 2 and b == 1
    per_item = arr.ndim == 2 and arr.shape[0] == b and arr.shape[1] == 2
    if not flat_pair and not per_item:
        raise ValueError("lengths must have shape [B, 2] (or [2] for a single item)")
    arr = arr.reshape(b, 2)
    bad = (arr[:, 0] < 0) | (arr[:, 1] < 0) | (arr[:, 0] > t) | (arr[:, 1] > s)
    if bad.any():  # the lowest failing item, as the binding's loop reports it
        raise ValueError(f"item {int(np.argmax(bad))}: lengths must lie in [0, T] x [0, S]")
    return np.ascontiguousarray(arr.astype(np.uint32))


def _prepare(values, lengths, engine, max_neg_val, threads, unchecked):
    """batch_from_array + make_config, in the binding's order (module.cpp:120-125)."""
    if _is_torch(values):
        shape = tuple(values.shape)
    else:
        values = np.ascontiguousarray(values, dtype=np.float32)  # forcecast, module.cpp:18
        shape = values.shape
    was_2d, b, t, s = _check_dims(shape)
    lens = None if lengths is None else _parse_lengths(lengths, b, t, s)
    cfg = _make_config(engine, max_neg_val, threads, unchecked)
    return values, lens, cfg, was_2d, b, t, s


def _ptr(a, attr):
    return None if a is None else getattr(a, attr)


def _host_array(shape, dtype):
    """A numpy array in page-locked memory when it is large (the copy engine
    then writes it directly instead of through staging buffers); the pinned
    block comes from torch's caching host allocator and lives as long as the
    array."""
    nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
    if nbytes >= (1 << 20):
        try:
            import torch

            tdt = {np.uint8: torch.uint8, np.int32: torch.int32}[dtype]
            return torch.empty(shape, dtype=tdt, pin_memory=True).numpy()
        except Exception:  # no CUDA host allocator available: plain memory
            pass
    return np.empty(shape, dtype)


def _run_host(values, lens, cfg, b, t, s, want_out, want_paths, want_dur=False):
    lib = _lib.load()
    out = _host_array((b, t, s), np.uint8) if want_out else None
    paths = np.empty((b, s), np.int32) if want_paths else None
    dur = np.empty((b, t), np.int32) if want_dur else None
    err = _lib.MasError()
    rc = lib.mas_align_host_ex(
        values.ctypes.data, b, t, s, None if lens is None else lens.ctypes.data,
        ctypes.byref(cfg), None if out is None else out.ctypes.data,
        None if paths is None else paths.ctypes.data, None if dur is None else dur.ctypes.data,
        ctypes.byref(err))
    _lib.raise_for(rc, err)
    return out, paths, dur


def _run_device(values, lens, cfg, b, t, s, want_out, want_paths, want_dur=False):
    import torch

    lib = _lib.load()
    dev = values.device
    if values.dtype != torch.float32:
        values = values.to(torch.float32)
    values = values.reshape(b, t, s)
    if values.stride(2) != 1 or values.stride(0) != t * values.stride(1):
        values = values.contiguous()
    pitch = values.stride(1)
    out = torch.empty((b, t, s), dtype=torch.uint8, device=dev) if want_out else None
    paths = torch.empty((b, s), dtype=torch.int32, device=dev) if want_paths else None
    dur = torch.empty((b, t), dtype=torch.int32, device=dev) if want_dur else None
    err = _lib.MasError()

    def call():
        stream = torch.cuda.current_stream(dev)
        return lib.mas_align_device_ex(
            values.data_ptr(), pitch, b, t, s, None if lens is None else lens.ctypes.data,
            ctypes.byref(cfg), None if out is None else out.data_ptr(),
            None if paths is None else paths.data_ptr(), None if dur is None else dur.data_ptr(),
            stream.cuda_stream, ctypes.byref(err))

    if dev.index == torch.cuda.current_device():
        rc = call()  # (a device switch costs more than the rest of the wrapper)
    else:
        with torch.cuda.device(dev):
            rc = call()
    _lib.raise_for(rc, err)
    return out, paths, dur


def _align_impl(values, lengths, engine, max_neg_val, threads, unchecked, want_out, want_paths,
                want_dur=False, check=True):
    values, lens, cfg, was_2d, b, t, s = _prepare(values, lengths, engine, max_neg_val, threads,
                                                  unchecked)
    if not check:
        cfg.flags |= _lib.MAS_FLAG_NO_CHECK
    if _is_torch(values) and values.is_cuda:
        out, paths, dur = _run_device(values, lens, cfg, b, t, s, want_out, want_paths, want_dur)
    else:
        if _is_torch(values):
            values = np.ascontiguousarray(values.detach().numpy(), dtype=np.float32)
        out, paths, dur = _run_host(values, lens, cfg, b, t, s, want_out, want_paths, want_dur)
    return out, paths, dur, was_2d, lens, b, s


def align(values, lengths=None, engine="parallel", max_neg_val=_DEFAULT_MAX_NEG_VAL, threads=0,
          check=True):
    """Align a [T, S] or [B, T, S] float32 likelihood array; returns a uint8
    alignment array of the same shape. Optional lengths ([B, 2] of (t, s))
    mark each item's valid region.  (module.cpp:222-228; torch CUDA tensors
    in -> torch CUDA tensor out.)  ``check=False`` (torch CUDA input only, not
    in the reference): the call does not wait for the device's NonFinite
    scan -- it only enqueues, so a training step stays asynchronous; length /
    config errors are still raised, a non-finite likelihood is not."""
    out, _, _, was_2d, _, _, _ = _align_impl(values, lengths, engine, max_neg_val, threads, False,
                                             True, False, check=check)
    return out[0] if was_2d else out


def align_durations(values, lengths=None, engine="parallel", max_neg_val=_DEFAULT_MAX_NEG_VAL,
                    threads=0, check=True):
    """Per-token durations: the row sums of ``align``'s alignment, int32
    [B, T] ([T] for 2-D input) -- the number of speech frames spent on each
    text token, 0 past an item's text length.  Not in the reference's
    surface: the dense uint8 [B, T, S] output is
    never written, so the call moves 4.125 instead of 5.125 bytes per cell.
    Same arguments, checks and errors as ``align``."""
    _, _, dur, was_2d, _, _, _ = _align_impl(values, lengths, engine, max_neg_val, threads, False,
                                             False, False, True, check=check)
    return dur[0] if was_2d else dur


def align_paths(values, lengths=None, engine="parallel", max_neg_val=_DEFAULT_MAX_NEG_VAL,
                threads=0, check=True):
    """Like align, but returns per-frame text indices: one int32 array per
    item (a single array for 2-D input).  Each item's array has length s_b
    (path_from_matrix walks the item's valid lengths, types.cpp:161-179)."""
    _, paths, _, was_2d, lens, b, s = _align_impl(values, lengths, engine, max_neg_val, threads,
                                                  False, False, True, check=check)
    result = []
    for i in range(b):
        sb = s if lens is None else int(lens[i, 1])
        result.append(paths[i, :sb])
    return result[0] if was_2d else result


def _align_unchecked(values, lengths=None, engine="parallel", max_neg_val=_DEFAULT_MAX_NEG_VAL,
                     threads=0):
    """parallel::detail::align_unchecked / reference::detail::align_unchecked
    (parallel.hpp:29-31, reference.hpp:42-44): no validate_config, so -inf and
    -1e9 sentinels run.  Not part of the reference's Python surface; needed
    for the sentinel boundary checks."""
    out, _, _, was_2d, _, _, _ = _align_impl(values, lengths, engine, max_neg_val, threads, True,
                                             True, False)
    return out[0] if was_2d else out


# ---- MASTENS v1 tensor files (module.cpp:156-190, tensor_io.hpp) ----------
def read_tensor(path):
    """Read a tensor file; returns (values, lengths) where values is float32 or
    uint8 [B, T, S] and lengths is uint32 [B, 2].  (module.cpp:237-239;
    OSError with the reference's IoError text on a bad or truncated file.)"""
    lib = _lib.load()
    p = os.fsencode(path)
    err = _lib.MasError()
    dtype = ctypes.c_int32()
    dims = (ctypes.c_int64 * 3)()
    has_len = ctypes.c_int32()
    rc = lib.mas_io_read_header(p, _lib.MAS_IO_DEFAULT_BYTE_BUDGET, ctypes.byref(dtype),
                                ctypes.byref(dims), ctypes.byref(has_len), ctypes.byref(err))
    _lib.raise_for(rc, err)
    shape = (dims[0], dims[1], dims[2])
    values = np.empty(shape, np.float32 if dtype.value == 0 else np.uint8)
    lengths = np.empty((dims[0], 2), np.uint32)
    rc = lib.mas_io_read(p, _lib.MAS_IO_DEFAULT_BYTE_BUDGET, dtype.value, ctypes.byref(dims),
                         values.ctypes.data, lengths.ctypes.data, ctypes.byref(err))
    _lib.raise_for(rc, err)
    return values, lengths


def write_tensor(path, values, lengths=None):
    """Write a float32 (likelihood) or uint8 (alignment) array as a tensor
    file (module.cpp:169-190, 241-243): [T, S] or [B, T, S], optional [B, 2]
    lengths checked as in align; any other dtype raises ValueError."""
    if _is_torch(values):
        values = values.detach().cpu().numpy()
    values = np.asarray(values)
    if values.dtype == np.float32:
        dtype = 0
    elif values.dtype == np.uint8:
        dtype = 1
    else:
        raise ValueError("values dtype must be float32 or uint8")
    values = np.ascontiguousarray(values)
    _, b, t, s = _check_dims(values.shape)
    lens = None if lengths is None else _parse_lengths(lengths, b, t, s)
    lib = _lib.load()
    err = _lib.MasError()
    rc = lib.mas_io_write(os.fsencode(path), dtype, b, t, s, values.ctypes.data,
                          None if lens is None else lens.ctypes.data, ctypes.byref(err))
    _lib.raise_for(rc, err)


def generate_random_batch(b, t, s, seed):
    """Deterministic uniform [-5, 5] float32 batch of shape [B, T, S]
    (bench::generate_random_batch, bench.cpp:164-180), generated on the GPU
    bit-identically and returned as numpy."""
    import torch

    if b < 1 or t < 1 or s < 1:
        raise ValueError("batch dimensions must be at least 1")
    if t > s:
        raise ValueError("text length t exceeds speech length s")
    buf = generate_device(b, t, s, seed)
    return buf.cpu().numpy()


def generate_device(b, t, s, seed, first_item=0, device=None, out=None, row_pitch=None):
    """Items [first_item, first_item + b) of generate_random_batch(..., seed)
    written on the GPU into a [b, t, row_pitch] float32 tensor (a view of the
    first s columns is what the reference generates)."""
    import torch

    lib = _lib.load()
    dev = torch.device("cuda") if device is None else torch.device(device)
    pitch = s if row_pitch is None else int(row_pitch)
    if out is None:
        out = torch.empty((b, t, pitch), dtype=torch.float32, device=dev)
    with torch.cuda.device(out.device):
        stream = torch.cuda.current_stream(out.device)
        rc = lib.mas_generate_device(int(seed) & (2**64 - 1), b, t, s, int(first_item), pitch,
                                     out.data_ptr(), ctypes.c_void_p(stream.cuda_stream))
    if rc != _lib.MAS_OK:
        raise RuntimeError("mas_generate_device failed")
    return out if pitch == s else out[:, :, :s]


def forward_parallel(values, lengths=None, max_neg_val=_DEFAULT_MAX_NEG_VAL):
    """parallel::forward_parallel (reference parallel.hpp:17, parallel.cpp:95-108):
    overwrites each item's [t, s] region of ``values`` with the parallel
    engine's cumulative score table, in place, and returns ``values``.
    Bit-identical to the reference (std::max tie rule, signed zeros).  A torch
    CUDA float32 tensor is updated on its device (stream-ordered on the current
    stream); a numpy float32 C-contiguous array round-trips through the GPU and
    is written back in place.  Computed on the GPU by the forward kernel's
    score export (csrc/mas_fwd4.cu OUT 1), or forward_scores_kernel
    (csrc/mas_scores.cu) for layouts its TMA maps cannot take; there is no
    host implementation."""
    import torch

    lib = _lib.load()
    was_2d, b, t, s = _check_dims(tuple(values.shape))
    lens = None if lengths is None else _parse_lengths(lengths, b, t, s)
    lens_ptr = None if lens is None else lens.ctypes.data
    err = _lib.MasError()
    if _is_torch(values):
        if values.dtype != torch.float32 or not values.is_cuda:
            raise ValueError("values must be a float32 CUDA tensor")
        if values.stride(-1) != 1 or (not was_2d and values.stride(0) != t * values.stride(1)):
            raise ValueError("values must have unit column stride and packed items")
        pitch = values.stride(-2)
        with torch.cuda.device(values.device):
            stream = torch.cuda.current_stream(values.device)
            rc = lib.mas_forward_scores(values.data_ptr(), pitch, b, t, s, lens_ptr,
                                        float(np.float32(max_neg_val)),
                                        ctypes.c_void_p(stream.cuda_stream), ctypes.byref(err))
        _lib.raise_for(rc, err)
        return values
    if not isinstance(values, np.ndarray) or values.dtype != np.float32 or \
            not values.flags.c_contiguous or not values.flags.writeable:
        raise ValueError("values must be a writeable C-contiguous float32 array (updated in place)")
    dev = torch.empty((b, t, s), dtype=torch.float32, device="cuda")
    dev.copy_(torch.from_numpy(values.reshape(b, t, s)))
    stream = torch.cuda.current_stream(dev.device)
    rc = lib.mas_forward_scores(dev.data_ptr(), s, b, t, s, lens_ptr, float(np.float32(max_neg_val)),
                                ctypes.c_void_p(stream.cuda_stream), ctypes.byref(err))
    _lib.raise_for(rc, err)
    values.reshape(b, t, s)[...] = dev.cpu().numpy()
    return values


# ---- fused log-likelihood ---------------------------
def _gauss_inputs(z, mean, logstd):
    import torch

    for name, x in (("z", z), ("mean", mean), ("logstd", logstd)):
        if not _is_torch(x) or not x.is_cuda or x.dtype != torch.float32 or x.dim() != 3:
            raise ValueError(f"{name} must be a float32 CUDA tensor of rank 3")
    if mean.shape != logstd.shape:
        raise ValueError("mean and logstd must have the same shape [B, C, T]")
    if z.shape[0] != mean.shape[0] or z.shape[1] != mean.shape[1]:
        raise ValueError("z must be [B, C, S] with the B and C of mean / logstd")
    if not (z.device == mean.device == logstd.device):
        raise ValueError("z, mean and logstd must be on one device")
    B, C, S = (int(v) for v in z.shape)
    T = int(mean.shape[2])
    return z.contiguous(), mean.contiguous(), logstd.contiguous(), B, C, T, S


def gaussian_loglik(z, mean, logstd):
    """The prior log-likelihood matrix MAS aligns:
    q[b, i, j] = sum_c log N(z[b, c, j]; mean[b, c, i], exp(logstd[b, c, i])),
    float32 [B, T, S] on z's device, from z [B, C, S] and mean / logstd
    [B, C, T] (Glow-TTS / VITS layouts).  Computed on the tensor cores
    (tcgen05, bf16 operands of the expanded square, fp32 accumulation:
    csrc/mas_gauss.cu); the same values the fused align_gaussian uses."""
    import torch

    z, mean, logstd, B, C, T, S = _gauss_inputs(z, mean, logstd)
    lib = _lib.load()
    q = torch.empty((B, T, S), dtype=torch.float32, device=z.device)
    err = _lib.MasError()
    with torch.cuda.device(z.device):
        st = torch.cuda.current_stream(z.device)
        rc = lib.mas_gaussian_loglik_device(z.data_ptr(), mean.data_ptr(), logstd.data_ptr(), B, C,
                                            T, S, q.data_ptr(), S, ctypes.c_void_p(st.cuda_stream),
                                            ctypes.byref(err))
    _lib.raise_for(rc, err)
    return q


def align_gaussian(z, mean, logstd, lengths=None, engine="parallel",
                   max_neg_val=_DEFAULT_MAX_NEG_VAL, outputs=("alignment",), unchecked=False):
    """The maximum-path call on q = gaussian_loglik(z, mean, logstd) without
    materialising q: the forward kernel
    computes each 32-frame tile of q on the tensor cores and feeds it to the
    DP directly.  z [B, C, S], mean / logstd [B, C, T] float32 CUDA tensors;
    lengths [B, 2] of (t, s) as in align.  Returns a dict with the requested
    `outputs` among "alignment" (uint8 [B, T, S]), "paths" (int32 [B, S], -1
    past s_b) and "durations" (int32 [B, T]).  Equal, bit for bit, to
    align(gaussian_loglik(z, mean, logstd), ...) for the same arguments."""
    import torch

    z, mean, logstd, B, C, T, S = _gauss_inputs(z, mean, logstd)
    lens = None if lengths is None else _parse_lengths(lengths, B, T, S)
    cfg = _make_config(engine, max_neg_val, 0, unchecked)
    bad = set(outputs) - {"alignment", "paths", "durations"}
    if bad:
        raise ValueError(f"unknown outputs: {sorted(bad)}")
    dev = z.device
    res = {}
    if "alignment" in outputs:
        res["alignment"] = torch.empty((B, T, S), dtype=torch.uint8, device=dev)
    if "paths" in outputs:
        res["paths"] = torch.empty((B, S), dtype=torch.int32, device=dev)
    if "durations" in outputs:
        res["durations"] = torch.empty((B, T), dtype=torch.int32, device=dev)
    lib = _lib.load()
    err = _lib.MasError()
    with torch.cuda.device(dev):
        st = torch.cuda.current_stream(dev)
        rc = lib.mas_align_gaussian_device(
            z.data_ptr(), mean.data_ptr(), logstd.data_ptr(), B, C, T, S,
            None if lens is None else lens.ctypes.data, ctypes.byref(cfg),
            res["alignment"].data_ptr() if "alignment" in res else None,
            res["paths"].data_ptr() if "paths" in res else None,
            res["durations"].data_ptr() if "durations" in res else None,
            ctypes.c_void_p(st.cuda_stream), ctypes.byref(err))
    _lib.raise_for(rc, err)
    return res


class GaussianPlan:
    """Enqueue-only form of align_gaussian for training loops
    (mas_plan_create_gaussian / mas_plan_enqueue_gaussian): validation and
    the operand workspace once, then per batch the operand prep and the fused
    kernels only -- no host synchronisation, CUDA-graph capturable.  finish()
    reports the last enqueue's validation / NonFinite errors as align does.
    Texts taller than 4096 rows and NaN sentinels of the parallel engine are
    refused (ValueError / RuntimeError); align_gaussian handles them."""

    def __init__(self, b, c, t, s, lengths=None, engine="parallel",
                 max_neg_val=_DEFAULT_MAX_NEG_VAL, unchecked=False):
        lib = _lib.load()
        self._lib = lib
        self.b, self.c, self.t, self.s = b, c, t, s
        lens = None if lengths is None else _parse_lengths(lengths, b, t, s)
        self._lens = lens
        cfg = _make_config(engine, max_neg_val, 0, unchecked)
        handle = ctypes.c_void_p()
        err = _lib.MasError()
        rc = lib.mas_plan_create_gaussian(b, c, t, s, None if lens is None else lens.ctypes.data,
                                          ctypes.byref(cfg), ctypes.byref(handle),
                                          ctypes.byref(err))
        _lib.raise_for(rc, err)
        self._h = handle

    def enqueue(self, z, mean, logstd, out=None, paths=None, durations=None, stream=None):
        """z [B, C, S], mean / logstd [B, C, T] float32 CUDA tensors (the plan's
        shape); writes any of out [B,T,S] uint8, paths [B,S] int32, durations
        [B,T] int32 (device tensors)."""
        import torch

        z, mean, logstd, B, C, T, S = _gauss_inputs(z, mean, logstd)
        if (B, C, T, S) != (self.b, self.c, self.t, self.s):
            raise ValueError(f"inputs are [B={B}, C={C}, T={T}, S={S}], the plan "
                             f"[{self.b}, {self.c}, {self.t}, {self.s}]")
        err = _lib.MasError()
        st = torch.cuda.current_stream() if stream is None else stream
        rc = self._lib.mas_plan_enqueue_gaussian(
            self._h, z.data_ptr(), mean.data_ptr(), logstd.data_ptr(),
            None if out is None else out.data_ptr(), None if paths is None else paths.data_ptr(),
            None if durations is None else durations.data_ptr(), ctypes.c_void_p(st.cuda_stream),
            ctypes.byref(err))
        _lib.raise_for(rc, err)

    def finish(self, stream=None):
        import torch

        err = _lib.MasError()
        st = torch.cuda.current_stream() if stream is None else stream
        rc = self._lib.mas_plan_finish(self._h, None, ctypes.c_void_p(st.cuda_stream),
                                       ctypes.byref(err))
        _lib.raise_for(rc, err)

    def close(self):
        if getattr(self, "_h", None):
            self._lib.mas_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Plan:
    """Enqueue-only execution of the maximum-path call on device buffers
    (mas_plan_* in include/monoalign_b200.h): validation and workspace once,
    then kernels only -- what the benchmark times and a CUDA graph captures."""

    def __init__(self, b, t, s, row_pitch=None, lengths=None, engine="parallel",
                 max_neg_val=_DEFAULT_MAX_NEG_VAL, unchecked=False, pipelined=False):
        lib = _lib.load()
        self._lib = lib
        self.b, self.t, self.s = b, t, s
        self.row_pitch = s if row_pitch is None else int(row_pitch)
        lens = None if lengths is None else _parse_lengths(lengths, b, t, s)
        self._lens = lens
        cfg = _make_config(engine, max_neg_val, 0, unchecked)
        if pipelined:
            # consecutive enqueues may overlap (batch i's backtrack with batch
            # i+1's forward); give consecutive enqueues distinct outputs
            cfg.flags |= _lib.MAS_FLAG_PIPELINED
        handle = ctypes.c_void_p()
        err = _lib.MasError()
        rc = lib.mas_plan_create(b, t, s, self.row_pitch,
                                 None if lens is None else lens.ctypes.data, ctypes.byref(cfg),
                                 ctypes.byref(handle), ctypes.byref(err))
        _lib.raise_for(rc, err)
        self._h = handle

    def enqueue(self, values, out=None, paths=None, stream=None, parts=_lib.MAS_PART_ALL,
                durations=None):
        """Enqueues the kernels (`parts`: MAS_PART_FORWARD / _BACKTRACK bits)
        writing any of out [B,T,S] uint8, paths [B,S] int32, durations [B,T]
        int32 (device tensors)."""
        import torch

        err = _lib.MasError()
        st = torch.cuda.current_stream() if stream is None else stream
        rc = self._lib.mas_plan_enqueue_ex(
            self._h, parts, values.data_ptr(), None if out is None else out.data_ptr(),
            None if paths is None else paths.data_ptr(),
            None if durations is None else durations.data_ptr(), ctypes.c_void_p(st.cuda_stream),
            ctypes.byref(err))
        _lib.raise_for(rc, err)

    def finish(self, values, stream=None):
        import torch

        err = _lib.MasError()
        st = torch.cuda.current_stream() if stream is None else stream
        rc = self._lib.mas_plan_finish(self._h, values.data_ptr(),
                                       ctypes.c_void_p(st.cuda_stream), ctypes.byref(err))
        _lib.raise_for(rc, err)

    @property
    def launches(self) -> int:
        return int(self._lib.mas_plan_launches(self._h))

    @property
    def geometry(self) -> dict:
        g = (ctypes.c_int32 * 6)()
        self._lib.mas_plan_geometry(self._h, ctypes.byref(g))
        return {"rows_per_warp": g[0], "warps_per_cta": g[1], "ctas_per_item": g[2],
                "stages": g[3], "segment_cols": g[4], "max_active_clusters": g[5]}

    def close(self):
        if getattr(self, "_h", None):
            self._lib.mas_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
