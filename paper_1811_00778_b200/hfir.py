"""HFIR files (the reference's bit-exact binary format, serial.py:30-229)
read into and written from device-resident ciphertext tensors.

The reference writes every element in the coefficient domain as u64 LE,
position-major then prime (serial.py:87-97), behind a header of magic,
version, kind, N, primes and t (serial.py:44-72).  Here the headers are
parsed / written on the host and the element bodies move in one copy each
way; the (N, K) <-> (K, N) transposition and the u64 <-> u32 narrowing run on
the GPU (hcnn_hfir_pack / hcnn_hfir_unpack).  Files are byte-identical to
serial.dump_cipher_tensor's; the readers raise the same error classes with
the same byte offsets as serial.load_* (FormatError, ParameterMismatchError).

    dump_cipher_tensor_device(tensor, params, fresh=None) -> bytes   serial.py:206-216
    load_cipher_tensor_device(data, params, device=None)  -> GpuCipherTensor  serial.py:219-229
    load_relin_key_device(data, params)                   -> DeviceRelinKey  serial.py:171-187
"""

from __future__ import annotations

import io
import struct

import numpy as np
import torch

from . import _lib
from .engine import GpuCipherTensor, _ptr, context_for
from .errors import FormatError, ParameterMismatchError

MAGIC = b"HFIR"
VERSION = 1
KIND_SECRET_KEY = 1
KIND_PUBLIC_KEY = 2
KIND_RELIN_KEY = 3
KIND_CIPHERTEXT = 4
KIND_CIPHER_TENSOR = 5


def _primes(params):
    return [int(pm.value) for pm in params.ctx.primes]


def header_bytes(kind: int, params) -> bytes:
    """serial._write_header (serial.py:44-50)."""
    primes = _primes(params)
    out = [MAGIC, struct.pack("<HB", VERSION, kind), struct.pack("<IH", params.ring_degree, len(primes))]
    out += [struct.pack("<Q", p) for p in primes]
    out.append(struct.pack("<Q", params.t))
    return b"".join(out)


def _read_exact(buf: io.BytesIO, count: int) -> bytes:
    data = buf.read(count)
    if len(data) != count:
        raise FormatError("truncated file", offset=buf.tell())
    return data


def read_header(buf: io.BytesIO):
    """serial.read_header (serial.py:60-72): (kind, n, primes, t)."""
    magic = _read_exact(buf, 4)
    if magic != MAGIC:
        raise FormatError(f"bad magic {magic!r}", offset=0)
    version, kind = struct.unpack("<HB", _read_exact(buf, 3))
    if version != VERSION:
        raise FormatError(f"unsupported format version {version}", offset=4)
    n, count = struct.unpack("<IH", _read_exact(buf, 6))
    primes = [struct.unpack("<Q", _read_exact(buf, 8))[0] for _ in range(count)]
    t = struct.unpack("<Q", _read_exact(buf, 8))[0]
    return kind, n, primes, t


def _check_header_params(params, n, primes, t):
    """serial._check_header_params (serial.py:75-84)."""
    if n != params.ring_degree or list(primes) != _primes(params) or t != params.t:
        raise ParameterMismatchError(
            f"file parameters (N={n}, t={t}) do not match the active set "
            f"(N={params.ring_degree}, t={params.t})"
        )


def _bodies_to_device(g, raw: np.ndarray, rows: int) -> torch.Tensor:
    """raw: rows * N * K u64 (HFIR order) -> device [rows][K][N] u32."""
    dev = torch.from_numpy(raw.view(np.int64)).to(f"cuda:{g.device}")
    out = torch.empty((rows, g.K, g.N), dtype=torch.int32, device=f"cuda:{g.device}")
    g.bind_stream()
    _lib.check(_lib.lib().hcnn_hfir_unpack(g.handle, _ptr(dev), rows, _ptr(out)), "hcnn_hfir_unpack")
    return out


def _device_to_bodies(g, rows_t: torch.Tensor, rows: int) -> np.ndarray:
    """device [rows][K][N] u32 -> host rows * N * K u64 (HFIR order)."""
    dev = torch.empty(rows * g.N * g.K, dtype=torch.int64, device=rows_t.device)
    g.bind_stream()
    _lib.check(_lib.lib().hcnn_hfir_pack(g.handle, _ptr(rows_t), rows, _ptr(dev)), "hcnn_hfir_pack")
    return dev.cpu().numpy().view(np.uint64)


# ---------------------------------------------------------------- tensors


def dump_cipher_tensor_device(tensor: GpuCipherTensor, params, fresh=None) -> bytes:
    """serial.dump_cipher_tensor (serial.py:206-216) of a device tensor of
    2-part ciphertexts; fresh: per-ciphertext is_fresh flags (default False,
    as for every evaluated ciphertext)."""
    g = context_for(params, tensor.data.device)
    count = len(tensor)
    h, w, c = tensor.shape
    delta = int(tensor.delta)
    delta_bytes = delta.to_bytes((delta.bit_length() + 7) // 8 or 1, "big")
    head = (header_bytes(KIND_CIPHER_TENSOR, params) + struct.pack("<IIIH", h, w, c, len(delta_bytes))
            + delta_bytes + struct.pack("<I", count))
    body = 2 * g.N * g.K * 8
    stride = 2 + body
    out = np.empty(len(head) + count * stride, dtype=np.uint8)
    out[: len(head)] = np.frombuffer(head, dtype=np.uint8)
    if count:
        cts = out[len(head):].reshape(count, stride)
        cts[:, 0] = 2
        cts[:, 1] = 0 if fresh is None else np.asarray(fresh, dtype=np.uint8)
        bodies = _device_to_bodies(g, tensor.data.reshape(count * 2, g.K, g.N), count * 2)
        cts[:, 2:] = bodies.view(np.uint8).reshape(count, body)
    return out.tobytes()


def load_cipher_tensor_device(data: bytes, params, device=None) -> GpuCipherTensor:
    """serial.load_cipher_tensor (serial.py:219-229) straight into device
    memory; `.fresh` holds the per-ciphertext is_fresh flags.  Device tensors
    hold 2-part ciphertexts: a 3-part one raises FormatError at its offset."""
    buf = io.BytesIO(data)
    kind, n, primes, t = read_header(buf)
    if kind != KIND_CIPHER_TENSOR:
        raise FormatError(f"expected cipher tensor, got kind {kind}", offset=6)
    _check_header_params(params, n, primes, t)
    h, w, c, delta_len = struct.unpack("<IIIH", _read_exact(buf, 14))
    delta = int.from_bytes(_read_exact(buf, delta_len), "big")
    (count,) = struct.unpack("<I", _read_exact(buf, 4))
    g = context_for(params, device)
    base = buf.tell()
    body = 2 * g.N * g.K * 8
    stride = 2 + body
    arr = np.frombuffer(data, dtype=np.uint8)
    for i in range(count):  # headers first: the same errors, at the same offsets
        off = base + i * stride
        if off + 2 > len(arr):
            raise FormatError("truncated file", offset=len(arr))
        parts = int(arr[off])
        if parts not in (2, 3):
            raise FormatError(f"ciphertext with {parts} parts", offset=off + 2)
        if parts != 2:
            raise FormatError("device tensors hold 2-part ciphertexts", offset=off + 2)
        if off + stride > len(arr):
            raise FormatError("truncated file", offset=len(arr))
    fresh = np.zeros(count, dtype=bool)
    if count:
        view = np.lib.stride_tricks.as_strided(arr[base:], shape=(count, stride), strides=(stride, 1))
        fresh = view[:, 1].astype(bool)
        raw = np.ascontiguousarray(view[:, 2:]).reshape(-1).view("<u8")
        rows = _bodies_to_device(g, raw, count * 2)
        out = rows.reshape(count, 2, g.K, g.N)
    else:
        out = torch.empty((0, 2, g.K, g.N), dtype=torch.int32, device=f"cuda:{g.device}")
    res = GpuCipherTensor((h, w, c), out, delta, t, params)
    res.fresh = fresh
    return res


# ---------------------------------------------------------------- keys


class DeviceRelinKey:
    """A relinearisation key read from HFIR (coefficient domain, serial.py:
    161-168) for the GPU evaluator: uploaded as is and transformed on the
    device (the reference NTT-transforms every component on the host at load,
    serial.py:184-185).  Usable wherever an rlk is expected (eval_square,
    eval_network)."""

    def __init__(self, coeff: np.ndarray, base: int, fingerprint: str):
        self.coeff = coeff  # u64 [D][2][K][N]
        self.base = base
        self.fingerprint = fingerprint

    @property
    def components(self):
        return [None] * self.coeff.shape[0]


def load_relin_key_device(data: bytes, params) -> DeviceRelinKey:
    """serial.load_relin_key (serial.py:171-187) without the host NTT."""
    buf = io.BytesIO(data)
    kind, n, primes, t = read_header(buf)
    if kind != KIND_RELIN_KEY:
        raise FormatError(f"expected relin key, got kind {kind}", offset=6)
    _check_header_params(params, n, primes, t)
    base, count = struct.unpack("<QH", _read_exact(buf, 10))
    if base != params.w:
        raise ParameterMismatchError(f"relin base {base} does not match parameter set base {params.w}")
    k, nn = len(primes), n
    need = count * 2 * nn * k * 8
    start = buf.tell()
    if len(data) - start < need:
        raise FormatError("truncated file", offset=len(data))
    body = np.frombuffer(data, dtype="<u8", count=count * 2 * nn * k, offset=start)
    coeff = np.ascontiguousarray(body.reshape(count, 2, nn, k).transpose(0, 1, 3, 2)).astype(np.uint64)
    return DeviceRelinKey(coeff, base, params.fingerprint)
