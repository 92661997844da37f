"""GPU drop-in for the reference's homomorphic network evaluator.

Same functions, signatures, error behaviour, OpCounter and layer_hook
semantics as hefir.engine (engine.py:61-85, 199-423); the arithmetic runs in
libhcnn_b200.so (sm_100a) on device-resident limb-major u32 tensors.

    eval_network(tensor, model, rlk, params, counter=None, workers=1,
                 capacity=None, layer_hook=None)          engine.py:400-423
    eval_conv / eval_fc / eval_square / eval_pool       engine.py:237-397

`tensor` may be the reference's CipherTensor (host; uploaded, and the result
downloaded back into the caller's own classes) or a GpuCipherTensor (stays on
the device; `.cts` downloads lazily).  `workers` and `capacity` are accepted
for signature compatibility; the GPU grid replaces the thread pool and the
row-band blocking (capacity is still validated like plan_blocks,
engine.py:109-112).  There is no CPU fallback.
"""

from __future__ import annotations

import hashlib
import os
import time
import threading
import weakref
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import (
    CapacityError,
    HefirError,
    IncompleteResultError,
    MissingKeyError,
    ParameterMismatchError,
)
from .nn import kind_of

_COUNTER_LOCK = threading.Lock()


# ---------------------------------------------------------------- host types


@dataclass
class OpCounter:
    """Scheduled multiply-accumulate work, matching the static audit
    (engine.py:61-85)."""

    mult_plain_scheduled: int = 0
    mult_plain_executed: int = 0
    mult_plain_skipped: int = 0
    hsquare: int = 0
    hadd: int = 0

    def merge(self, other):
        with _COUNTER_LOCK:
            self.mult_plain_scheduled += other.mult_plain_scheduled
            self.mult_plain_executed += other.mult_plain_executed
            self.mult_plain_skipped += other.mult_plain_skipped
            self.hsquare += other.hsquare
            self.hadd += other.hadd


@dataclass
class CipherTensor:
    """Host feature map: one ciphertext per (y, x, channel) (engine.py:42-58)."""

    shape: tuple
    cts: list
    delta: int
    channel_modulus: int

    def __post_init__(self):
        h, w, c = self.shape
        if len(self.cts) != h * w * c:
            raise HefirError("ciphertext count != h*w*c")

    def at(self, y: int, x: int, ch: int):
        h, w, c = self.shape
        return self.cts[(y * w + x) * c + ch]


@dataclass(frozen=True)
class PackingLayout:
    batch_size: int
    slot_count: int

    def __post_init__(self):
        if self.batch_size > self.slot_count:
            raise CapacityError(f"batch {self.batch_size} exceeds slot capacity {self.slot_count}")


# ---------------------------------------------------------------- device context


def _device_index(device) -> int:
    if device is None:
        return torch.cuda.current_device()
    return torch.device(device).index or 0


class GpuContext:
    """libhcnn_b200 context for one BFV parameter set on one GPU."""

    def __init__(self, params, device=None):
        if not torch.cuda.is_available():
            raise _lib.BackendError("CUDA device required: the evaluator has no CPU path")
        self.device = _device_index(device)
        self.params = params
        ctx = params.ctx
        self.primes = [int(pm.value) for pm in ctx.primes]
        self.N = int(ctx.ring_degree)
        self.K = len(self.primes)
        self.t = int(params.t)
        self.fingerprint = params.fingerprint
        log2w = int(params.w).bit_length() - 1
        arr = (_lib.C.c_uint64 * self.K)(*self.primes)
        h = _lib.C.c_void_p()
        L = _lib.lib()
        with torch.cuda.device(self.device):
            _lib.check(L.hcnn_ctx_create(_lib.C.byref(h), self.N, self.K, arr, self.t, log2w,
                                         self.device), "hcnn_ctx_create")
        self.handle = h
        self.KP = int(L.hcnn_ctx_query(h, 2))
        self.D = int(L.hcnn_ctx_query(h, 3))
        variant = os.environ.get("HCNN_NTT_VARIANT")
        if variant is not None and self.N >= 1024:
            _lib.check(L.hcnn_ctx_set_option(h, 1, int(variant)), "hcnn_ctx_set_option")
        ts = os.environ.get("HCNN_TS_CHUNK")
        if ts is not None:
            _lib.check(L.hcnn_ctx_set_option(h, 2, int(ts)), "hcnn_ctx_set_option")
        ws = os.environ.get("HCNN_WS_LIMIT_GB")
        if ws is not None:
            _lib.check(L.hcnn_ctx_set_workspace_limit(h, int(float(ws) * (1 << 30))), "workspace limit")
        self._rlk_ref = None
        self._weights = {}
        self._finalizer = weakref.finalize(self, L.hcnn_ctx_destroy, h)

    # -- plumbing
    def bind_stream(self):
        s = torch.cuda.current_stream(self.device).cuda_stream
        _lib.check(_lib.lib().hcnn_ctx_set_stream(self.handle, _lib.C.c_void_p(s)))

    def launches(self) -> int:
        return int(_lib.lib().hcnn_ctx_query(self.handle, 6))

    def empty(self, n: int, parts: int = 2) -> torch.Tensor:
        return torch.empty((n, parts, self.K, self.N), dtype=torch.int32, device=f"cuda:{self.device}")

    def set_variant(self, variant: int):
        """Geometry flags of the fused kernels (include/hcnn_b200.h: 16 one-row
        relinearisation, 32 radix-32 square tensor, 64 mixed-width passes, 512
        2-CTA cluster rows at 2^15, 1024 relinearisation sums in TMEM, 2048 /
        4096 square tensor with rows parked in TMEM, 8192 persistent square
        tensor with TMA prefetch, 16384 relinearisation over the shared
        three-prime basis R, 32768 base conversions on the tensor cores,
        65536 the relinearisation multiply-accumulate on the tensor cores)."""
        _lib.check(_lib.lib().hcnn_ctx_set_option(self.handle, 1, int(variant)), "ntt variant")

    def variant(self) -> int:
        """Geometry flags in effect (the per-N default unless set)."""
        return int(_lib.lib().hcnn_ctx_query(self.handle, 7))

    def profile(self, enable: bool):
        _lib.check(_lib.lib().hcnn_profile(self.handle, int(bool(enable))))

    def profile_read(self) -> dict:
        import ctypes

        buf = ctypes.create_string_buffer(1 << 16)
        _lib.lib().hcnn_profile_dump(self.handle, buf, len(buf))
        out = {}
        for line in buf.value.decode().splitlines():
            name, cnt, tot = line.split()
            out[name] = (int(cnt), float(tot))
        return out

    def set_workspace_limit(self, nbytes: int):
        _lib.check(_lib.lib().hcnn_ctx_set_workspace_limit(self.handle, int(nbytes)))

    # -- keys and weights
    def set_relin_key(self, rlk):
        """Upload RelinKey.components (NTT domain, reference order) once."""
        if rlk is None:
            raise MissingKeyError("relinearization key required")
        if getattr(rlk, "fingerprint", self.fingerprint) != self.fingerprint:
            raise ParameterMismatchError("object does not match parameter set")
        if self._rlk_ref is not None and self._rlk_ref() is rlk:
            return
        coeff = getattr(rlk, "coeff", None)  # hfir.DeviceRelinKey: serialised, coefficient domain
        if coeff is not None:
            if coeff.shape[0] != self.D:
                raise ParameterMismatchError("relinearization key has the wrong digit count")
            host, domain = np.ascontiguousarray(coeff, dtype=np.uint64), 0
        else:
            comps = rlk.components
            if len(comps) != self.D:
                raise ParameterMismatchError("relinearization key has the wrong digit count")
            host = np.ascontiguousarray(
                np.stack([np.stack([k0.residues, k1.residues]) for k0, k1 in comps]).astype(np.uint64)
            )
            domain = 1
            first = comps[0][0]
            if getattr(first, "domain", None) is not None and getattr(first.domain, "value", "ntt") != "ntt":
                domain = 0
        self.bind_stream()
        _lib.check(_lib.lib().hcnn_set_relin_key(self.handle, host.ctypes.data, domain),
                   "hcnn_set_relin_key")
        try:
            self._rlk_ref = weakref.ref(rlk)
        except TypeError:
            self._rlk_ref = lambda r=rlk: r

    def set_public_key(self, pk):
        """Upload PublicKey (b_ntt, a_ntt; reference NTT order) once."""
        if getattr(pk, "fingerprint", self.fingerprint) != self.fingerprint:
            raise ParameterMismatchError("object does not match parameter set")
        if getattr(self, "_pk_ref", None) is not None and self._pk_ref() is pk:
            return
        host = np.ascontiguousarray(np.stack([pk.b_ntt.residues, pk.a_ntt.residues]).astype(np.uint64))
        self.bind_stream()
        _lib.check(_lib.lib().hcnn_set_public_key(self.handle, host.ctypes.data, 1),
                   "hcnn_set_public_key")
        self._pk_ref = weakref.ref(pk)

    def weights(self, weights):
        """Layer weights -> library weight handle (cached by content)."""
        w = np.asarray(weights)
        if w.dtype == object or not np.issubdtype(w.dtype, np.integer):
            ints = [int(x) for x in w.reshape(-1)]
            if max((abs(x) for x in ints), default=0) >= (1 << 63):
                raise ParameterMismatchError("weights must fit in int64")
            w = np.array(ints, dtype=np.int64)
        w = np.ascontiguousarray(w.reshape(-1), dtype=np.int64)
        key = (w.shape, hashlib.blake2b(w.tobytes(), digest_size=16).digest())
        handle = self._weights.get(key)
        if handle is None:
            h = _lib.C.c_void_p()
            self.bind_stream()
            _lib.check(_lib.lib().hcnn_weights_create(self.handle, w.ctypes.data, w.size, _lib.C.byref(h)),
                       "hcnn_weights_create")
            if len(self._weights) > 64:
                for old in self._weights.values():
                    _lib.lib().hcnn_weights_destroy(self.handle, old)
                self._weights.clear()
            self._weights[key] = h
            handle = h
        return handle


_CTXS: dict = {}


def release_memory(device=None):
    """Drop every cached context (their workspaces and keys) and codec on
    `device`, and return the library pool's and torch's cached free memory
    to the driver."""
    import gc

    dev = _device_index(device)
    for cache in (_CTXS, _CODECS):
        for k in [k for k in cache if k[-1] == dev]:
            del cache[k]
    gc.collect()
    torch.cuda.synchronize(dev)
    _lib.check(_lib.lib().hcnn_release_memory(dev), "hcnn_release_memory")
    torch.cuda.empty_cache()


def context_for(params, device=None) -> GpuContext:
    key = (params.fingerprint, _device_index(device))
    c = _CTXS.get(key)
    if c is None:
        c = GpuContext(params, device)
        _CTXS[key] = c
    return c


# ---------------------------------------------------------------- device tensors


class GpuCipherTensor:
    """Feature map resident on the GPU: int32 view of u32 residues
    [ct][part][limb][N], (y, x, c) row-major like CipherTensor."""

    def __init__(self, shape, data: torch.Tensor, delta: int, channel_modulus: int, params,
                 host_types=None):
        h, w, c = shape
        if data.shape[0] != h * w * c:
            raise HefirError("ciphertext count != h*w*c")
        self.shape = tuple(shape)
        self.data = data
        self.delta = delta
        self.channel_modulus = channel_modulus
        self.params = params
        self.host_types = host_types
        self._cts = None

    def __len__(self):
        return self.data.shape[0]

    def residues(self) -> np.ndarray:
        """u64 residues [ct][part][limb][N] on the host."""
        torch.cuda.current_stream(self.data.device).synchronize()
        return self.data.cpu().numpy().view(np.uint32).astype(np.uint64)

    @property
    def cts(self) -> list:
        if self._cts is None:
            self._cts = _download_cts(self)
        return self._cts

    def at(self, y: int, x: int, ch: int):
        h, w, c = self.shape
        return self.cts[(y * w + x) * c + ch]

    def to_host(self):
        cls = self.host_types[0] if self.host_types else CipherTensor
        return cls(shape=self.shape, cts=self.cts, delta=self.delta,
                   channel_modulus=self.channel_modulus)


def _host_types_of(tensor, params):
    if tensor.cts:
        ct = tensor.cts[0]
        elem = ct.parts[0]
        return (type(tensor), type(ct), type(elem), elem.domain, elem.ctx)
    return (type(tensor), None, None, None, params.ctx)


def _download_cts(t: "GpuCipherTensor") -> list:
    """Device tensor -> host Ciphertext objects: one download into a reused
    pinned u32 buffer, then the residues widened to int64 straight into the
    objects' fresh arrays by host threads (hcnn_host_widen); single-threaded
    numpy casts of the result ran at ~4 GB/s on the GPU host."""
    n = t.data.shape[0]
    if n == 0:
        return []
    g = context_for(t.params, t.data.device)
    parts, K, N = t.data.shape[1:]
    pin = _stager(g).out(n * parts * K * N)
    stream = torch.cuda.current_stream(t.data.device)
    pin.copy_(t.data.reshape(-1), non_blocking=True)
    stream.synchronize()
    arrays = [np.empty((K, N), dtype=np.int64) for _ in range(n * parts)]
    ptrs = np.array([a.ctypes.data for a in arrays], dtype=np.uintp)
    _lib.check(_lib.lib().hcnn_host_widen(_lib.C.c_void_p(pin.data_ptr()), n * parts, K * N, ptrs.ctypes.data,
                                          min(16, os.cpu_count() or 1)), "hcnn_host_widen")
    host_types = t.host_types
    if host_types and host_types[1] is not None:
        _, ct_cls, el_cls, dom, ctx = host_types
    else:
        from . import bfv as _b

        ct_cls, el_cls, dom, ctx = _b.Ciphertext, _b.RingElem, _b.Domain.COEFF, t.params.ctx
    fp = t.params.fingerprint
    return [ct_cls(parts=tuple(el_cls(ctx, arrays[i * parts + p], dom) for p in range(parts)), fingerprint=fp)
            for i in range(n)]


class _HostStager:
    """Pinned u32 staging buffer for host CipherTensors, one per context and
    reused across calls (a fresh pin_memory() per call costs more than the
    copy).  The reference's residues are int64 numpy arrays, one per part
    and ciphertext; they are narrowed to u32 straight into the pinned buffer
    by a thread pool (numpy's casting copy releases the GIL), in row ranges
    so that uploads can start on the first rows while later ones are filled."""

    _pool = None

    def __init__(self):
        self.buf = None
        self.free = None  # event after the last upload out of `buf`

    @classmethod
    def pool(cls):
        if cls._pool is None:
            import concurrent.futures

            cls._pool = concurrent.futures.ThreadPoolExecutor(
                max_workers=max(1, min(16, os.cpu_count() or 1)), thread_name_prefix="hcnn-stage")
        return cls._pool

    def out(self, words: int) -> torch.Tensor:
        """reused pinned int32 buffer of at least `words` words (downloads)"""
        ob = getattr(self, "obuf", None)
        if ob is None or ob.numel() < words:
            ob = self.obuf = torch.empty(max(words, 1 << 20), dtype=torch.int32, pin_memory=True)
        return ob[:words]

    def get(self, n: int, K: int, N: int) -> torch.Tensor:
        if self.buf is None or self.buf.shape[0] < n or tuple(self.buf.shape[1:]) != (2, K, N):
            self.buf = torch.empty((max(n, 1), 2, K, N), dtype=torch.int32, pin_memory=True)
            self.free = None
        if self.free is not None:
            self.free.synchronize()  # the previous call's uploads have left the buffer
        return self.buf[:n]

    def fill(self, stage: torch.Tensor, cts, lo: int, hi: int):
        """stage[lo:hi] <- cts[lo:hi] (int64 residues narrowed to u32): one
        multi-threaded native call (hcnn_host_narrow) when every part is a
        C-contiguous int64 [K][N] array, numpy casting copies otherwise."""
        if hi <= lo:
            return
        K, N = stage.shape[2], stage.shape[3]
        ptrs = np.empty(2 * (hi - lo), dtype=np.uintp)
        k = 0
        for ct in cts[lo:hi]:
            for part in ct.parts:
                r = part.residues
                if r.dtype != np.int64 or r.shape != (K, N) or not r.flags.c_contiguous:
                    return self._fill_numpy(stage, cts, lo, hi)
                ptrs[k] = r.ctypes.data
                k += 1
        # one native call, split over host threads inside (measured on the
        # 16-core GPU host: 14.7 ms for the 784-ciphertext MNIST input alone,
        # about 20 ms while the uploads run; tools/host_bw_probe.py)
        dst = stage.data_ptr() + lo * 2 * K * N * 4
        _lib.check(_lib.lib().hcnn_host_narrow(ptrs.ctypes.data, 2 * (hi - lo), K * N, _lib.C.c_void_p(dst),
                                               _narrow_threads()), "hcnn_host_narrow")

    def _fill_numpy(self, stage, cts, lo, hi):
        arr = stage.numpy().view(np.uint32)

        def job(a, b):
            for i in range(a, b):
                p0, p1 = cts[i].parts
                np.copyto(arr[i, 0], p0.residues, casting="unsafe")
                np.copyto(arr[i, 1], p1.residues, casting="unsafe")

        pool = self.pool()
        nw = pool._max_workers
        cuts = np.linspace(lo, hi, min(hi - lo, 4 * nw) + 1).astype(np.int64)
        for f in [pool.submit(job, int(a), int(b)) for a, b in zip(cuts[:-1], cuts[1:])]:
            f.result()


def _narrow_threads() -> int:
    """host threads of the int64 -> u32 narrowing (HCNN_NARROW_THREADS, else
    min(16, cores)); the narrowing is host-memory-bound"""
    v = os.environ.get("HCNN_NARROW_THREADS")
    return max(1, int(v)) if v else min(16, os.cpu_count() or 1)


def _stager(g) -> _HostStager:
    st = getattr(g, "_stager", None)
    if st is None:
        st = g._stager = _HostStager()
    return st


def _check_host_cts(tensor, params):
    fp = params.fingerprint
    for ct in tensor.cts:
        if ct.fingerprint != fp:
            raise ParameterMismatchError("ciphertext does not match parameter set")
        if len(ct.parts) != 2:
            raise ParameterMismatchError("evaluator expects 2-part ciphertexts")


def upload(tensor, params, device=None) -> GpuCipherTensor:
    """Host CipherTensor -> GpuCipherTensor (u64 residues narrowed to u32)."""
    if isinstance(tensor, GpuCipherTensor):
        return tensor
    g = context_for(params, device)
    _check_host_cts(tensor, params)
    n = len(tensor.cts)
    st = _stager(g)
    stage = st.get(n, g.K, g.N)
    st.fill(stage, tensor.cts, 0, n)
    data = g.empty(n)
    data.copy_(stage, non_blocking=True)
    st.free = torch.cuda.Event()
    st.free.record(torch.cuda.current_stream(data.device))
    return GpuCipherTensor(tensor.shape, data, tensor.delta, tensor.channel_modulus, params,
                           _host_types_of(tensor, params))


def from_residues(res: np.ndarray, shape, delta, channel_modulus, params, device=None) -> GpuCipherTensor:
    """u32/u64 residues [ct][2][K][N] (host) -> GpuCipherTensor."""
    g = context_for(params, device)
    host = np.ascontiguousarray(np.asarray(res).astype(np.uint32))
    data = torch.from_numpy(host.view(np.int32)).to(f"cuda:{g.device}")
    return GpuCipherTensor(shape, data, delta, channel_modulus, params)


def _ptr(t: torch.Tensor):
    return _lib.C.c_void_p(t.data_ptr())


# ---------------------------------------------------------------- counters


def _conv_counts(h, w, layer, weights):
    f, kh, kw, cg = weights.shape
    sh, sw = layer.stride
    ph = (kh - 1) // 2 if layer.padded else 0
    pw = (kw - 1) // 2 if layer.padded else 0
    oh = (h + 2 * ph - kh) // sh + 1
    ow = (w + 2 * pw - kw) // sw + 1
    vy = np.array([[0 <= oy * sh + ky - ph < h for ky in range(kh)] for oy in range(oh)], dtype=np.int64)
    vx = np.array([[0 <= ox * sw + kx - pw < w for kx in range(kw)] for ox in range(ow)], dtype=np.int64)
    nz = (np.asarray(weights) != 0).sum(axis=3).astype(np.int64)
    executed = np.einsum("ak,bl,fkl->abf", vy, vx, nz)
    sched = int(np.einsum("ak,bl->", vy, vx)) * cg * f
    ex = int(executed.sum())
    hadd = int((executed[executed > 0] - 1).sum())
    return sched, ex, hadd


def _fc_counts(weights):
    nz = (np.asarray(weights) != 0).sum(axis=1).astype(np.int64)
    sched = int(np.asarray(weights).size)
    ex = int(nz.sum())
    hadd = int((nz[nz > 0] - 1).sum())
    return sched, ex, hadd


def _count(counter, sched, ex, hadd):
    counter.mult_plain_scheduled += sched
    counter.mult_plain_executed += ex
    counter.mult_plain_skipped += sched - ex
    counter.hadd += hadd


# ---------------------------------------------------------------- layers


def _as_gpu(tensor, params, device=None):
    if tensor.channel_modulus != params.t:
        raise ParameterMismatchError("tensor channel does not match params")
    if isinstance(tensor, GpuCipherTensor):
        return tensor, False
    return upload(tensor, params, device), True


def _ret(out: GpuCipherTensor, was_host: bool):
    return out.to_host() if was_host else out


def eval_conv(tensor, layer, weights, params, counter, workers: int = 1, capacity=None):
    """Convolution layer (engine.py:237-303) on the GPU."""
    h, w, c = tensor.shape
    weights = np.asarray(weights)
    f, kh, kw, cg = weights.shape
    if c != cg * layer.groups:
        raise ParameterMismatchError(f"{layer.name}: channel mismatch")
    if tensor.channel_modulus != params.t:
        raise ParameterMismatchError(f"{layer.name}: tensor channel != params")
    if capacity is not None and capacity < kh * kw:
        raise CapacityError(f"capacity {capacity} below filter size {kh * kw}")
    src, was_host = _as_gpu(tensor, params)
    g = context_for(params, src.data.device)
    sh, sw = layer.stride
    ph = (kh - 1) // 2 if layer.padded else 0
    pw = (kw - 1) // 2 if layer.padded else 0
    oh = (h + 2 * ph - kh) // sh + 1
    ow = (w + 2 * pw - kw) // sw + 1
    wt = g.weights(weights)
    out = g.empty(oh * ow * f)
    g.bind_stream()
    _lib.check(_lib.lib().hcnn_conv(g.handle, _ptr(src.data), _ptr(out), h, w, c, wt, f,
                                    kh, kw, sh, sw, int(bool(layer.padded)), layer.groups),
               layer.name)
    _count(counter, *_conv_counts(h, w, layer, weights))
    res = GpuCipherTensor((oh, ow, f), out, tensor.delta * layer.weight_scale, params.t, params,
                          src.host_types)
    return _ret(res, was_host)


def eval_fc(tensor, layer, weights, params, counter, workers: int = 1):
    """Dense layer over the (y, x, c)-flattened tensor (engine.py:306-334)."""
    weights = np.asarray(weights)
    outputs, in_count = weights.shape
    n = tensor.shape[0] * tensor.shape[1] * tensor.shape[2]
    if in_count != n:
        raise ParameterMismatchError(f"{layer.name}: weight width != tensor size")
    src, was_host = _as_gpu(tensor, params)
    g = context_for(params, src.data.device)
    wt = g.weights(weights)
    out = g.empty(outputs)
    g.bind_stream()
    _lib.check(_lib.lib().hcnn_fc(g.handle, _ptr(src.data), _ptr(out), in_count, outputs, wt),
               layer.name)
    _count(counter, *_fc_counts(weights))
    res = GpuCipherTensor((1, 1, outputs), out, tensor.delta * layer.weight_scale, params.t, params,
                          src.host_types)
    return _ret(res, was_host)


def eval_square(tensor, rlk, params, counter, workers: int = 1):
    """HSquare of every ciphertext: exact tensor, t/q rounding, base-w relin
    (engine.py:337-364, bfv.py:435-443)."""
    src, was_host = _as_gpu(tensor, params)
    g = context_for(params, src.data.device)
    n = len(src)
    out = g.empty(n)
    if n:
        if rlk is None:
            raise MissingKeyError("relinearization key required for hsquare")
        g.set_relin_key(rlk)
        g.bind_stream()
        _lib.check(_lib.lib().hcnn_square(g.handle, _ptr(src.data), _ptr(out), n), "square")
    counter.hsquare += n
    res = GpuCipherTensor(src.shape, out, tensor.delta * tensor.delta, tensor.channel_modulus,
                          params, src.host_types)
    return _ret(res, was_host)


def eval_pool(tensor, layer, params, counter):
    """Sum-pool by window adds (engine.py:367-397)."""
    h, w, c = tensor.shape
    e = layer.extent
    sh, sw = layer.stride
    oh = (h - e) // sh + 1
    ow = (w - e) // sw + 1
    src, was_host = _as_gpu(tensor, params)
    g = context_for(params, src.data.device)
    out = g.empty(oh * ow * c)
    g.bind_stream()
    _lib.check(_lib.lib().hcnn_pool(g.handle, _ptr(src.data), _ptr(out), h, w, c, e, sh, sw),
               layer.name)
    counter.hadd += oh * ow * c * (e * e - 1)
    res = GpuCipherTensor((oh, ow, c), out, tensor.delta * e * e, tensor.channel_modulus, params,
                          src.host_types)
    return _ret(res, was_host)


def eval_network(tensor, model, rlk, params, counter=None, workers: int = 1, capacity=None,
                 layer_hook=None):
    """Evaluate every layer; returns the logits tensor (1, 1, outputs)
    (engine.py:400-423).  Host input -> host output; GPU input -> GPU output;
    layer_hook receives GpuCipherTensors (their .cts download on demand)."""
    counter = counter if counter is not None else OpCounter()
    if not isinstance(tensor, GpuCipherTensor) and _bandable(model, tensor.shape) and len(tensor.cts) > 1:
        return _eval_network_host(tensor, model, rlk, params, counter, capacity, layer_hook)
    x, was_host = _as_gpu(tensor, params)
    x = _eval_layers(x, model, 0, rlk, params, counter, workers, capacity, layer_hook)
    return _ret(x, was_host)


def _eval_network_host(tensor, model, rlk, params, counter, capacity=None, layer_hook=None, bands: int = 12):
    """eval_network of a host CipherTensor (the reference's own objects): its
    int64 residues are narrowed into a reused pinned buffer by row bands, each
    band is uploaded on a copy stream as soon as it is filled, and the leading
    row-local layers (conv1, square1, conv2, square2) run as a wavefront on
    the rows already on the device, so the host-side narrowing and the upload
    overlap the evaluation.  Same
    kernels, results and counters as the device path (engine.py:400-423)."""
    if tensor.channel_modulus != params.t:
        raise ParameterMismatchError("tensor channel does not match params")
    _, kh, kw, _ = np.asarray(model.weights[0]).shape
    if capacity is not None and capacity < kh * kw:
        raise CapacityError(f"capacity {capacity} below filter size {kh * kw}")
    _check_host_cts(tensor, params)
    g = context_for(params)
    dev = torch.device("cuda", g.device)
    compute = torch.cuda.current_stream(dev)
    up_stream, _ = _copy_streams(dev)
    up_stream.wait_stream(compute)
    st = _stager(g)
    n = len(tensor.cts)
    stage = st.get(n, g.K, g.N)
    buf = g.empty(n)
    buf.record_stream(up_stream)
    x, released, m = _banded_head(stage, buf, tuple(tensor.shape), tensor.delta, model, rlk, params, counter,
                               up_stream, compute, bands, layer_hook,
                               prepare=lambda lo, hi: st.fill(stage, tensor.cts, lo, hi),
                               host_types=_host_types_of(tensor, params))
    st.free = torch.cuda.Event()
    st.free.record(up_stream)
    compute.wait_stream(up_stream)
    x = _eval_layers(x, model, m, rlk, params, counter, layer_hook=layer_hook)
    return x.to_host()


def _eval_layers(x, model, start, rlk, params, counter, workers=1, capacity=None, layer_hook=None):
    for layer, weights in list(zip(model.spec.layers, model.weights))[start:]:
        k = kind_of(layer)
        if k == "conv":
            x = eval_conv(x, layer, weights, params, counter, workers, capacity)
        elif k == "square":
            x = eval_square(x, rlk, params, counter, workers)
        elif k == "pool":
            x = eval_pool(x, layer, params, counter)
        elif k == "fc":
            x = eval_fc(x, layer, weights, params, counter, workers)
        if layer_hook is not None:
            layer_hook(layer.name, x)
    return x


_COPY_STREAMS: dict = {}


def _copy_streams(dev):
    """One upload and one download stream per device, reused across calls (a
    fresh stream per call would also strand the caching allocator's blocks on
    streams that are never used again)."""
    key = dev.index
    if key not in _COPY_STREAMS:
        _COPY_STREAMS[key] = (torch.cuda.Stream(dev), torch.cuda.Stream(dev))
    return _COPY_STREAMS[key]


def _row_local_prefix(model) -> int:
    """Number of leading layers whose output rows each depend on a contiguous
    band of input rows (unpadded convolutions, squares, pools): those layers
    can run as a wavefront behind a row-by-row upload."""
    m = 0
    for layer in model.spec.layers:
        k = kind_of(layer)
        if k == "square" or k == "pool" or (k == "conv" and not layer.padded):
            m += 1
        else:
            break
    return m


def _bandable(model, shape) -> bool:
    """The network starts with an unpadded convolution followed by a square:
    its first layers can start on the first uploaded input rows."""
    layers = model.spec.layers
    return (_row_local_prefix(model) >= 2 and kind_of(layers[0]) == "conv" and kind_of(layers[1]) == "square"
            and shape[0] >= 2)


class _Stage:
    """One row-local layer of the wavefront: output buffer and rows done."""

    def __init__(self, layer, weights, shape, g):
        self.layer, self.kind = layer, kind_of(layer)
        self.ishape = shape
        h, w, c = shape
        if self.kind == "conv":
            weights = np.asarray(weights)
            f, kh, kw, cg = weights.shape
            if c != cg * layer.groups:
                raise ParameterMismatchError(f"{layer.name}: channel mismatch")
            self.weights, self.wt = weights, g.weights(weights)
            self.k, self.kw, self.s, self.sw = kh, kw, layer.stride[0], layer.stride[1]
            self.oshape = ((h - kh) // self.s + 1, (w - kw) // self.sw + 1, f)
        elif self.kind == "pool":
            self.k = self.kw = layer.extent
            self.s, self.sw = layer.stride
            self.oshape = ((h - self.k) // self.s + 1, (w - self.kw) // self.sw + 1, c)
        else:
            self.oshape = shape
        if self.oshape[0] <= 0 or self.oshape[1] <= 0:
            raise ParameterMismatchError(f"{layer.name}: empty output")
        self.out = g.empty(self.oshape[0] * self.oshape[1] * self.oshape[2])
        self.done = 0

    def ready_rows(self, rows_in: int) -> int:
        if self.kind == "square":
            return rows_in
        if rows_in < self.k:
            return 0
        return min(self.oshape[0], (rows_in - self.k) // self.s + 1)

    def run(self, g, src, rows_in: int) -> bool:
        """Launch this layer on the output rows its ready input rows allow."""
        L = _lib.lib()
        upto = self.ready_rows(rows_in)
        if upto <= self.done:
            return False
        lo, (h, w, c), (oh, ow, oc) = self.done, self.ishape, self.oshape
        if self.kind == "square":
            _lib.check(L.hcnn_square(g.handle, _ptr(src[lo * w * c:]), _ptr(self.out[lo * w * c:]),
                                     (upto - lo) * w * c), "square")
        else:
            y0, y1 = lo * self.s, (upto - 1) * self.s + self.k  # input rows read
            if self.kind == "conv":
                _lib.check(L.hcnn_conv(g.handle, _ptr(src[y0 * w * c:]), _ptr(self.out[lo * ow * oc:]), y1 - y0, w,
                                       c, self.wt, oc, self.k, self.kw, self.s, self.sw, 0, self.layer.groups),
                           self.layer.name)
            else:
                _lib.check(L.hcnn_pool(g.handle, _ptr(src[y0 * w * c:]), _ptr(self.out[lo * ow * oc:]), y1 - y0, w,
                                       c, self.k, self.s, self.sw), self.layer.name)
        self.done = upto
        return True


_BAND_TRACE = None  # list: (ciphertexts uploaded, host time, upload event, compute event) per band


def _banded_head(hb, buf, shape, delta, model, rlk, params, counter, up_stream, compute, bands, layer_hook,
                 prepare=None, host_types=None):
    """The network's leading row-local layers (unpadded convolutions, squares,
    pools: MNIST conv1, square1, conv2, square2) evaluated as a wavefront
    behind a row-band upload of the input: input rows go up in `bands`
    bands (by conv1 output rows), and after each band every layer is launched
    on the output rows its now-available input rows determine, so conv2 +
    square2 of the top rows run while later input rows are still uploading.
    Same kernels, same results and counters as the layer-by-layer path
    (engine.py:237-397).  `prepare(lo, hi)`, when given, fills host
    ciphertexts [lo, hi) of `hb` before they are uploaded (the drop-in path
    narrows the caller's residues there).  Returns (output tensor of the
    prefix, event after the last read of `buf`, number of layers done)."""
    if hb.shape[0] != shape[0] * shape[1] * shape[2]:
        raise ParameterMismatchError("ciphertext count != h*w*c")
    g = context_for(params, buf.device)
    m = _row_local_prefix(model)
    layers, weights = model.spec.layers[:m], model.weights[:m]
    if any(kind_of(la) == "square" for la in layers):
        if rlk is None:
            raise MissingKeyError("relinearization key required for hsquare")
        g.set_relin_key(rlk)
    stages, cur = [], tuple(shape)
    for la, wt in zip(layers, weights):
        stages.append(_Stage(la, wt, cur, g))
        cur = stages[-1].oshape
    h, w, c = shape
    row = w * c  # ciphertexts per input row
    first = stages[0]
    oh0 = first.oshape[0]
    cuts = [round(b * oh0 / bands) for b in range(bands + 1)]
    uploaded = 0
    g.bind_stream()
    for y1 in cuts[1:]:
        hi = h if y1 >= oh0 else min(h, (y1 - 1) * first.s + first.k) if first.kind != "square" else y1
        if hi <= uploaded:
            continue
        if prepare is not None:
            prepare(uploaded * row, hi * row)
        with torch.cuda.stream(up_stream):
            buf[uploaded * row:hi * row].copy_(hb[uploaded * row:hi * row], non_blocking=True)
            ready = torch.cuda.Event()
            ready.record(up_stream)
        compute.wait_event(ready)
        uploaded = hi
        g.bind_stream()
        src, rows = buf, uploaded
        for st in stages:
            st.run(g, src, rows)
            src, rows = st.out, st.done
        if _BAND_TRACE is not None:  # tools/dropin_probe.py: per-band upload / compute completion
            done = torch.cuda.Event(enable_timing=True)
            done.record(compute)
            up = torch.cuda.Event(enable_timing=True)
            up.record(up_stream)
            _BAND_TRACE.append((hi * row, time.perf_counter(), up, done))
    released = torch.cuda.Event()
    released.record(compute)
    # counters, scales and hooks layer by layer, as the reference's loop has them
    x = None
    d = delta
    for st in stages:
        if st.kind == "conv":
            _count(counter, *_conv_counts(st.ishape[0], st.ishape[1], st.layer, st.weights))
            d = d * st.layer.weight_scale
        elif st.kind == "square":
            counter.hsquare += st.oshape[0] * st.oshape[1] * st.oshape[2]
            d = d * d
        else:
            e = st.layer.extent
            counter.hadd += st.oshape[0] * st.oshape[1] * st.oshape[2] * (e * e - 1)
            d = d * e * e
        x = GpuCipherTensor(st.oshape, st.out, d, params.t, params, host_types)
        if layer_hook is not None:
            layer_hook(st.layer.name, x)
    return x, released, m


def eval_network_stream(batches, model, rlk, params, shape, delta, counter=None, device=None,
                        layer_hook=None, outputs=None, bands: int = 6):
    """Serving loop over encrypted slot-batches held in (pinned) host memory.

    Each batch is one `eval_network` (engine.py:400-423) on the GPU.  Batch
    i+1's ciphertexts are uploaded on a copy stream into the second of two
    device input buffers while batch i is evaluated (a buffer is released as
    soon as the first layer has read it), and batch i's logits go back to
    pinned host memory on a third stream as soon as its last layer is done.

    batches: iterable of host int32 tensors [n_ct][2][K][N] (u32 residues,
    (y, x, c) row-major like CipherTensor.cts), all of `shape`.
    The first batch has no evaluation to hide its upload behind: when the
    network starts with an unpadded convolution and a square, its upload is
    split into `bands` output-row bands and the leading row-local layers
    (conv1, square1, conv2, square2 for MNIST) run as a wavefront behind it,
    each launched on the rows its uploaded input rows allow (bands=1 turns
    this off).
    Returns the list of host int32 logit tensors [n_out][2][K][N] (written
    into `outputs[i]` when given, else freshly pinned); they are complete when
    the call returns.
    """
    counter = counter if counter is not None else OpCounter()
    dev = torch.device("cuda", _device_index(device))
    compute = torch.cuda.current_stream(dev)
    up_stream, down_stream = _copy_streams(dev)
    up_stream.wait_stream(compute)
    down_stream.wait_stream(compute)
    bufs, free, outs = [None, None], [None, None], []
    for i, hb in enumerate(batches):
        slot = i % 2
        if tuple(hb.shape[1:]) != (2, len(params.ctx.primes), int(params.ctx.ring_degree)):
            raise ParameterMismatchError("batch layout does not match params")
        if hb.shape[0] != shape[0] * shape[1] * shape[2]:
            raise ParameterMismatchError(f"batch {i} holds {hb.shape[0]} ciphertexts, shape {tuple(shape)} "
                                         f"needs {shape[0] * shape[1] * shape[2]}")
        if bufs[slot] is None or bufs[slot].shape != hb.shape:
            # allocated on the compute stream (which reads it), written by the
            # copy stream: record_stream keeps the block until both are done
            bufs[slot] = torch.empty(hb.shape, dtype=torch.int32, device=dev)
            bufs[slot].record_stream(up_stream)
        if i == 0 and bands > 1 and _bandable(model, shape):
            # nothing to overlap the first upload with: stream it by row bands
            # into the leading row-local layers instead
            x, free[slot], m = _banded_head(hb, bufs[slot], shape, delta, model, rlk, params, counter, up_stream,
                                            compute, bands, layer_hook)
            out = _eval_layers(x, model, m, rlk, params, counter, layer_hook=layer_hook)
        else:
            with torch.cuda.stream(up_stream):
                if free[slot] is not None:
                    up_stream.wait_event(free[slot])
                bufs[slot].copy_(hb, non_blocking=True)
                ready = torch.cuda.Event()
                ready.record(up_stream)
            compute.wait_event(ready)
            x = GpuCipherTensor(shape, bufs[slot], delta, params.t, params)
            released = torch.cuda.Event()
            state = {"first": True}

            def hook(name, t, _released=released, _state=state):
                if _state["first"]:  # the first layer has consumed the input buffer
                    _released.record(compute)
                    _state["first"] = False
                if layer_hook is not None:
                    layer_hook(name, t)

            out = eval_network(x, model, rlk, params, counter, layer_hook=hook)
            if state["first"]:
                released.record(compute)
            free[slot] = released
        done = torch.cuda.Event()
        done.record(compute)
        host = outputs[i] if outputs is not None else torch.empty(out.data.shape, dtype=torch.int32,
                                                                  pin_memory=True)
        with torch.cuda.stream(down_stream):
            down_stream.wait_event(done)
            host.copy_(out.data, non_blocking=True)
            out.data.record_stream(down_stream)
        outs.append(host)
    compute.wait_stream(down_stream)
    compute.wait_stream(up_stream)
    down_stream.synchronize()
    return outs


# ---------------------------------------------------------------- client side


def pack_images(images, layout: PackingLayout, encoder, pk, params, rng, delta: int):
    """Encrypt position i of every image into slot-aligned ciphertext i
    (engine.py:146-175); host client code, uses the bfv module's encrypt."""
    from . import bfv as _b

    if len(images) != layout.batch_size:
        raise CapacityError("image count != layout batch size")
    if layout.slot_count != params.ring_degree:
        raise ParameterMismatchError("layout slots != ring degree")
    shape = tuple(np.asarray(images[0]).shape)
    stack = np.stack([np.asarray(im, dtype=np.int64) for im in images])
    if stack.shape[1:] != shape:
        raise HefirError("images disagree on shape")
    t = params.t
    flat = stack.reshape(layout.batch_size, -1) % t
    slots = np.zeros((flat.shape[1], layout.slot_count), dtype=np.int64)
    slots[:, : layout.batch_size] = flat.T
    if hasattr(encoder, "encode_many"):
        polys = encoder.encode_many(slots)
    else:
        polys = np.stack([encoder.encode(s).poly for s in slots])
    cts = [_b.encrypt(pk, _b.Plaintext(polys[i], t), params, rng) for i in range(len(polys))]
    h, w = shape[0], shape[1]
    c = shape[2] if len(shape) == 3 else 1
    return CipherTensor(shape=(h, w, c), cts=cts, delta=delta, channel_modulus=t)


def draw_encryption_noise(rng, count: int, n: int):
    """(u, e1, e2) for `count` successive encryptions, in the reference's draw
    order (bfv.py:205-209)."""
    from .bfv import _gauss

    u = np.empty((count, n), dtype=np.int8)
    e1 = np.empty((count, n), dtype=np.int8)
    e2 = np.empty((count, n), dtype=np.int8)
    for i in range(count):
        u[i] = rng.integers(0, 2, n, dtype=np.int64)
        e1[i] = _gauss(rng, n)
        e2[i] = _gauss(rng, n)
    return u, e1, e2


def keygen_device(params, rng, device=None):
    """(sk, pk, rlk) like bfv.keygen(params, rng) (bfv.py:164-188), with the
    NTT-domain key arithmetic on the GPU (hcnn_keygen).  The randomness is drawn
    on the host in the reference's order (s, a, e, then a_i, e_i per digit),
    so the keys are bit-identical; they are also installed in the context."""
    from . import bfv as _b

    g = context_for(params, device)
    ctx = params.ctx
    n, k, d = g.N, g.K, g.D
    s_bits = rng.integers(0, 2, n, dtype=np.int64)
    a_rows = np.empty((1 + d, k, n), dtype=np.uint64)
    e_rows = np.empty((1 + d, n), dtype=np.int8)
    for r in range(1 + d):
        a_rows[r] = _b._uniform(ctx, rng)
        e_rows[r] = _b._gauss(rng, n)
    pk_out = np.empty((2, k, n), dtype=np.uint64)
    rlk_out = np.empty((d, 2, k, n), dtype=np.uint64)
    s8 = np.ascontiguousarray(s_bits.astype(np.uint8))
    g.bind_stream()
    _lib.check(_lib.lib().hcnn_keygen(g.handle, s8.ctypes.data, a_rows.ctypes.data, e_rows.ctypes.data,
                                      pk_out.ctypes.data, rlk_out.ctypes.data), "hcnn_keygen")
    el = lambda arr: _b.RingElem(ctx, arr.astype(np.int64), _b.Domain.NTT)  # noqa: E731
    m = ctx._modcol
    s_ntt = ctx.ntt.forward(s_bits[None, :] % m)  # client-side copy of the secret in the NTT domain
    sk = _b.SecretKey(s_bits=s_bits, s_ntt=el(s_ntt), s2_ntt=el(s_ntt * s_ntt % m))
    pk = _b.PublicKey(el(pk_out[0]), el(pk_out[1]), params.fingerprint)
    rlk = _b.RelinKey([(el(rlk_out[i, 0]), el(rlk_out[i, 1])) for i in range(d)], params.w, params.fingerprint)
    g._pk_ref = weakref.ref(pk)
    g._rlk_ref = weakref.ref(rlk)
    # hcnn_keygen installed this secret key on the device: keep the
    # decrypt-side cache (decrypt_device) in step with it
    g._sk_key = hashlib.blake2b(s8.tobytes(), digest_size=16).digest()
    return sk, pk, rlk


def encrypt_device(pk, polys, params, rng, device=None) -> torch.Tensor:
    """Encrypt plaintext polys [P][N] (in [0, t)) on the GPU; same bytes as P
    successive bfv.encrypt calls with this rng (bfv.py:201-216)."""
    g = context_for(params, device)
    g.set_public_key(pk)
    polys = np.ascontiguousarray(np.asarray(polys, dtype=np.int64))
    if polys.ndim != 2 or polys.shape[1] != g.N:
        raise ParameterMismatchError("plaintext length != ring degree")
    if (polys < 0).any() or (polys >= params.t).any():
        from .errors import EncodingError

        raise EncodingError("plaintext coefficient outside [0, t)")
    u, e1, e2 = draw_encryption_noise(rng, polys.shape[0], g.N)
    out = g.empty(polys.shape[0])
    g.bind_stream()
    _lib.check(_lib.lib().hcnn_encrypt(g.handle, u.ctypes.data, e1.ctypes.data, e2.ctypes.data,
                                       polys.ctypes.data, _ptr(out), polys.shape[0]), "hcnn_encrypt")
    return out


class GpuCodec:
    """SIMD slot codec over Z_t on the GPU (u64 NTT, batching.py:41-95)."""

    def __init__(self, t: int, n: int, device=None):
        self.t, self.n = int(t), int(n)
        self.device = _device_index(device)
        h = _lib.C.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(_lib.lib().hcnn_codec_create(self.t, self.n, self.device, _lib.C.byref(h)),
                       "hcnn_codec_create")
        self.handle = h
        self._fin = weakref.finalize(self, _lib.lib().hcnn_codec_destroy, h)

    def _run(self, fn, x: torch.Tensor) -> torch.Tensor:
        x = x.to(device=f"cuda:{self.device}", dtype=torch.int64).contiguous()
        out = torch.empty_like(x)
        stream = torch.cuda.current_stream(self.device).cuda_stream
        _lib.check(fn(self.handle, _ptr(x), _ptr(out), x.shape[0], _lib.C.c_void_p(stream)), "codec")
        return out

    def encode(self, slots: torch.Tensor) -> torch.Tensor:
        """[P][N] slot values in [0, t) -> [P][N] plaintext polys (int64)."""
        return self._run(_lib.lib().hcnn_codec_encode, slots)

    def decode(self, polys: torch.Tensor) -> torch.Tensor:
        return self._run(_lib.lib().hcnn_codec_decode, polys)


_CODECS: dict = {}


def codec_for(t: int, n: int, device=None) -> GpuCodec:
    key = (int(t), int(n), _device_index(device))
    c = _CODECS.get(key)
    if c is None:
        c = GpuCodec(t, n, device)
        _CODECS[key] = c
    return c


def decrypt_device(tensor: GpuCipherTensor, sk, params) -> torch.Tensor:
    """bfv.decrypt (bfv.py:239-250) of every ciphertext on the GPU: [n][N]
    plaintext polys in [0, t) (int64, device).  Requires t < 2^48."""
    g = context_for(params, tensor.data.device)
    s = np.ascontiguousarray(np.asarray(sk.s_bits).astype(np.uint8))
    key = hashlib.blake2b(s.tobytes(), digest_size=16).digest()
    if getattr(g, "_sk_key", None) != key:
        g.bind_stream()
        _lib.check(_lib.lib().hcnn_set_secret_key(g.handle, s.ctypes.data), "hcnn_set_secret_key")
        g._sk_key = key
    out = torch.empty((len(tensor), g.N), dtype=torch.int64, device=tensor.data.device)
    g.bind_stream()
    _lib.check(_lib.lib().hcnn_decrypt(g.handle, _ptr(tensor.data), _ptr(out), len(tensor)), "hcnn_decrypt")
    return out


def unpack_tensor_device(tensor: GpuCipherTensor, sk, params, batch_size: int) -> np.ndarray:
    """unpack_tensor (engine.py:178-192) on the GPU: decrypt + slot decode,
    returns (batch, h*w*c) values in [0, t)."""
    polys = decrypt_device(tensor, sk, params)
    slots = codec_for(params.t, params.ring_degree, tensor.data.device).decode(polys)
    return slots[:, :batch_size].T.contiguous().cpu().numpy()


def pack_images_device(images, layout: PackingLayout, encoder, pk, params, rng, delta: int,
                       device=None) -> GpuCipherTensor:
    """pack_images (engine.py:146-175) on the GPU: slot encoding (u64 NTT over
    Z_t) and encryption run on the device from host-drawn randomness; returns
    the same ciphertexts as the reference, resident on the device.  `encoder`
    is accepted for signature compatibility (the device codec is used)."""
    if len(images) != layout.batch_size:
        raise CapacityError("image count != layout batch size")
    if layout.slot_count != params.ring_degree:
        raise ParameterMismatchError("layout slots != ring degree")
    shape = tuple(np.asarray(images[0]).shape)
    stack = np.stack([np.asarray(im, dtype=np.int64) for im in images])
    flat = stack.reshape(layout.batch_size, -1) % params.t
    slots = np.zeros((flat.shape[1], layout.slot_count), dtype=np.int64)
    slots[:, : layout.batch_size] = flat.T
    g = context_for(params, device)
    codec = codec_for(params.t, params.ring_degree, g.device)
    polys = codec.encode(torch.from_numpy(slots))
    g.set_public_key(pk)
    u, e1, e2 = draw_encryption_noise(rng, polys.shape[0], g.N)
    data = g.empty(polys.shape[0])
    g.bind_stream()
    _lib.check(_lib.lib().hcnn_encrypt_device_msg(g.handle, u.ctypes.data, e1.ctypes.data, e2.ctypes.data,
                                                  _ptr(polys), _ptr(data), polys.shape[0]), "hcnn_encrypt")
    h, w = shape[0], shape[1]
    c = shape[2] if len(shape) == 3 else 1
    return GpuCipherTensor((h, w, c), data, delta, params.t, params)


def unpack_tensor(tensor, sk, encoder, params, batch_size: int) -> np.ndarray:
    """Decrypt and decode to per-image values (batch, h*w*c) (engine.py:178-192)."""
    from . import bfv as _b

    if tensor.channel_modulus != params.t:
        raise ParameterMismatchError("tensor channel does not match params")
    out = np.zeros((batch_size, len(tensor.cts)), dtype=np.int64)
    for pos, ct in enumerate(tensor.cts):
        out[:, pos] = encoder.decode(_b.decrypt(sk, ct, params)).values[:batch_size]
    return out


def reduce_model(model, t: int):
    """Weights centred mod t (engine.py:442-456)."""
    from .nn import QuantizedModel

    half = t // 2
    reduced = []
    for w in model.weights:
        if w is None:
            reduced.append(None)
            continue
        r = np.asarray(w, dtype=np.int64) % t
        reduced.append(np.where(r > half, r - t, r))
    return QuantizedModel(spec=model.spec, bit_width=model.bit_width, weights=reduced)


@dataclass
class ChannelResult:
    moduli: tuple
    batch_size: int
    residues: dict = None

    def __post_init__(self):
        if self.residues is None:
            self.residues = {}

    def add(self, t: int, logits: np.ndarray):
        self.residues[t] = logits


def run_channels(images, model, crt_system, params_for_channel, keys_for_channel, rng, workers: int = 1,
                 counter=None) -> ChannelResult:
    """One evaluation per plaintext-CRT channel (engine.py:459-491), every step
    on the GPU: slot encoding and encryption from the shared host rng (same
    draw order as the reference), eval_network, exact decryption and slot
    decoding.  Channels are independent; distributed.py deals them to ranks."""
    batch = len(images)
    moduli = tuple(getattr(crt_system, "moduli", crt_system))
    result = ChannelResult(moduli=moduli, batch_size=batch)
    for i, t in enumerate(moduli):
        params = params_for_channel(i)
        if params.t != t:
            raise ParameterMismatchError(f"channel {i}: params t != system t")
        sk, pk, rlk = keys_for_channel(i)
        layout = PackingLayout(batch_size=batch, slot_count=params.ring_degree)
        tensor = pack_images_device(images, layout, None, pk, params, rng, delta=model.spec.input_scale)
        logits_ct = eval_network(tensor, reduce_model(model, t), rlk, params, counter, workers)
        mat = unpack_tensor_device(logits_ct, sk, params, batch)  # (batch, outputs)
        result.add(t, mat.T.copy())
    return result


def _words_to_ints(words: np.ndarray) -> np.ndarray:
    """[M][W] u32 little-endian two's complement -> object array of Python ints
    (int64 fast path when every value fits)."""
    M, W = words.shape
    if M == 0:
        return np.zeros(0, dtype=object)
    lo = words[:, 0].astype(np.uint64) | (words[:, 1].astype(np.uint64) << np.uint64(32)) if W > 1 else \
        words[:, 0].astype(np.uint64)
    v64 = lo.view(np.int64)
    ext = np.where(v64 < 0, np.uint32(0xFFFFFFFF), np.uint32(0))
    if W <= 2 or (words[:, 2:] == ext[:, None]).all():
        return v64.astype(object)
    raw = np.ascontiguousarray(words).tobytes()
    step = 4 * W
    return np.array([int.from_bytes(raw[i:i + step], "little", signed=True) for i in range(0, len(raw), step)],
                    dtype=object)


class DeviceCrtValues:
    """Result of an asynchronous GPU CRT recombination: the signed values as
    DEVICE u32 words plus the kernel's range-check flag; nothing waits on the
    GPU until .values() (the client's host read)."""

    def __init__(self, words: torch.Tensor, flag: torch.Tensor, shape):
        self.words, self.flag, self.shape = words, flag, tuple(shape)

    def values(self) -> np.ndarray:
        """object array of signed Python ints, reshaped to `shape`"""
        if int(self.flag.item()):
            raise HefirError("CRT residue outside [0, t_i)")
        return _words_to_ints(self.words.cpu().numpy().view(np.uint32)).reshape(self.shape)


def crt_combine_device(res: torch.Tensor, moduli, sync: bool = True):
    """Centred CRT recombination on the GPU: res DEVICE int64 [C][M] (residue of
    value m mod moduli[i] at [i][m]) -> object array [M] of signed Python ints
    equal to CrtSystem.reconstruct_centered (codec.py:79-89) of each column.
    sync=False returns a DeviceCrtValues (no host synchronisation)."""
    moduli = [int(t) for t in moduli]
    if res.dim() != 2 or res.shape[0] != len(moduli):
        raise ParameterMismatchError("residue rows != modulus count")
    total = 1
    for t in moduli:
        total *= t
    words = total.bit_length() // 32 + 2
    res = res.to(dtype=torch.int64).contiguous()
    dev = res.device
    out = torch.empty((res.shape[1], words), dtype=torch.int32, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    arr = (_lib.C.c_uint64 * len(moduli))(*moduli)
    stream = torch.cuda.current_stream(dev).cuda_stream
    try:
        _lib.check(_lib.lib().hcnn_crt_combine(_ptr(res), arr, len(moduli), res.shape[1], _ptr(out), words,
                                               _ptr(flag), dev.index or 0, _lib.C.c_void_p(stream)),
                   "hcnn_crt_combine")
    except ParameterMismatchError as e:  # non-coprime / out-of-range moduli, as the reference raises
        raise HefirError(str(e)) from None
    lazy = DeviceCrtValues(out, flag, (res.shape[1],))
    return lazy if not sync else lazy.values()


def reconstruct_logits(result, crt_moduli) -> np.ndarray:
    """Signed logits (batch, outputs) from per-channel residues
    (engine.py:494-506), recombined on the GPU (crt_combine_device).  The
    per-channel matrices may be host arrays or device tensors (outputs, batch)."""
    moduli = tuple(getattr(crt_moduli, "moduli", crt_moduli))
    for t in moduli:
        if t not in result.residues:
            raise IncompleteResultError(f"missing CRT channel t={t}")
    if not torch.cuda.is_available():
        return reconstruct_logits_host(result, moduli)
    mats = [result.residues[t] for t in moduli]
    dev = next((m.device for m in mats if isinstance(m, torch.Tensor) and m.is_cuda),
               torch.device("cuda", torch.cuda.current_device()))
    stack = torch.stack([m.to(dev, dtype=torch.int64) if isinstance(m, torch.Tensor)
                         else torch.from_numpy(np.ascontiguousarray(np.asarray(m, dtype=np.int64))).to(dev)
                         for m in mats])
    C, outputs, batch = stack.shape
    vals = crt_combine_device(stack.reshape(C, -1), moduli)
    return vals.reshape(outputs, batch).T.copy()


def reconstruct_logits_device(mats, moduli) -> "DeviceCrtValues":
    """reconstruct_logits without a host synchronisation: mats = per-channel
    DEVICE int64 (outputs, batch) residues in `moduli` order; returns a
    DeviceCrtValues whose .values() is the (outputs, batch) object array
    (transpose for the reference's (batch, outputs))."""
    stack = torch.stack([m.to(dtype=torch.int64) for m in mats])
    C, outputs, batch = stack.shape
    lazy = crt_combine_device(stack.reshape(C, -1), moduli, sync=False)
    lazy.shape = (outputs, batch)
    return lazy


def reconstruct_logits_host(result, crt_moduli) -> np.ndarray:
    """The client-side host form of reconstruct_logits (engine.py:494-506) for
    a process without a GPU (the gloo tests of the gather): Garner mixed-radix
    digits vectorised over all values, Python ints only for the final sum."""
    moduli = tuple(int(t) for t in getattr(crt_moduli, "moduli", crt_moduli))
    for t in moduli:
        if t not in result.residues:
            raise IncompleteResultError(f"missing CRT channel t={t}")
    mats = []
    for t in moduli:
        m = np.asarray(result.residues[t], dtype=np.int64)
        if (m < 0).any() or (m >= t).any():
            raise HefirError(f"residue outside [0, {t})")
        mats.append(m.astype(object))
    outputs, batch = mats[0].shape
    total = 1
    for t in moduli:
        total *= t
    acc = np.zeros((outputs, batch), dtype=object)
    radix = 1
    for m, t in zip(mats, moduli):  # next mixed-radix digit: (r_i - X) * (prod t_<i)^-1 mod t_i
        acc = acc + ((m - acc) % t) * pow(radix % t, -1, t) % t * radix
        radix *= t
    half = total // 2
    out = np.where(acc > half, acc - total, acc)
    return out.T.copy()


def classify_logits(logits) -> list:
    """Per-image argmax, lowest index on ties (engine.py:509-515)."""
    out = []
    for row in logits:
        vals = list(row)
        out.append(vals.index(max(vals)))
    return out
