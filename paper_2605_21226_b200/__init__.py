"""B200-native OCTOPUS KV-cache codec hot path (arXiv 2605.21226).

Python mirror of the reference C++ API (/root/reference/proj/include/octoquant)
over the C ABI in ``include/octoquant_b200.h``.  Names, argument meaning and
error behaviour follow the reference:

==========================  =================================================
reference (C++)             here
==========================  =================================================
CodecConfig / validate      :class:`CodecConfig` / ``.validate()``
default_bit_split           :func:`default_bit_split`
Rounding, parse_rounding    :data:`ROUNDINGS`, :func:`parse_rounding`
xi_book / rho_book          :func:`xi_book`, :func:`rho_book`
Encoder(cfg[, Books])       :class:`Encoder` (device tables on the current GPU)
Encoder::encode             :meth:`Encoder.compress` (batched, bit-exact)
Encoder::decode             :meth:`Encoder.decode`
pack_keys / unpack_keys     :func:`pack_keys`, :func:`unpack_keys`
attention_decode            :func:`attention_decode` (batched GQA, K and V
                            compressed, split-K) + :class:`KVCache`
std::invalid_argument       :class:`ValueError`
FormatError                 :class:`FormatError`
==========================  =================================================

PyTorch is used only for device memory and streams.  There is no CPU compute
path: every data-path call launches the sm_100a kernels in
``liboctoquant_b200.so`` and fails loudly when the library or a GPU is absent.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

__all__ = [
    "AttentionPipeline", "CodecConfig", "Encoder", "FormatError", "KVCache", "ROUNDINGS",
    "attention_decode",
    "attention_decode_dense",
    "attention_partials", "attention_combine", "default_bit_split",
    "effective_bits_per_coord", "lib", "pack_keys", "parse_rounding", "record_bytes", "rho_book",
    "unpack_keys", "xi_book",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboctoquant_b200.so")

ROUNDINGS = ("scalar", "local2x2", "local3x3", "full")
ROLE_K, ROLE_V = 0, 1
_DTYPES = {"float32": 0, "float64": 1, "float16": 2, "bfloat16": 3}


class FormatError(RuntimeError):
    """Corrupt codes or wire data (octoquant::FormatError, io.hpp:17-20)."""


class _Config(C.Structure):
    _fields_ = [("dim", C.c_uint32), ("b_dir", C.c_uint8), ("b_nrm", C.c_uint8),
                ("rounding", C.c_uint8), ("qjl", C.c_uint8), ("rotation_seed", C.c_uint64),
                ("qjl_seed", C.c_uint64)]


class _Shape(C.Structure):
    _fields_ = [("B", C.c_int32), ("Hq", C.c_int32), ("Hkv", C.c_int32), ("T", C.c_uint64),
                ("cap_tokens", C.c_uint64), ("seq_lens", C.c_void_p)]


_lib = None


def lib():
    """Load liboctoquant_b200.so (built in-tree by ``make``); raise if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `make` (or __graft_entry__.build()); "
                          "there is no CPU fallback")
    L = C.CDLL(LIB_PATH)
    vp, sz, u64, i32 = C.c_void_p, C.c_size_t, C.c_uint64, C.c_int
    cfgp = C.POINTER(_Config)
    dp = C.POINTER(C.c_double)
    L.oq_last_error.restype = C.c_char_p
    L.oq_version.restype = C.c_char_p
    sigs = {
        "oq_config_validate": ([cfgp], i32),
        "oq_default_bit_split": ([i32, C.POINTER(i32), C.POINTER(i32)], i32),
        "oq_parse_rounding": ([C.c_char_p, C.POINTER(i32)], i32),
        "oq_effective_bits_per_coord": ([cfgp], C.c_double),
        "oq_record_bytes": ([cfgp], sz),
        "oq_xi_book": ([i32, dp, dp], i32),
        "oq_rho_book": ([C.c_uint32, i32, dp, dp], i32),
        "oq_codec_create": ([cfgp, C.POINTER(vp)], i32),
        "oq_codec_create_custom": ([cfgp, dp, i32, dp, i32, C.POINTER(vp)], i32),
        "oq_codec_destroy": ([vp], None),
        "oq_compress": ([vp, vp, i32, sz, vp, vp], i32),
        "oq_compress_ex": ([vp, vp, i32, sz, vp, vp, vp], i32),
        "oq_attention_sharded_workspace_bytes": ([vp, vp, C.POINTER(_Shape), i32, i32], sz),
        "oq_attention_decode_sharded": ([vp, vp, C.POINTER(_Shape), vp, vp, vp, C.c_uint64,
                                         C.c_uint64, vp, i32, vp, i32, vp, sz, vp], i32),
        "oq_nccl_get_unique_id": ([vp], i32),
        "oq_nccl_comm_init_rank": ([C.POINTER(vp), i32, vp, i32], i32),
        "oq_nccl_comm_destroy": ([vp], i32),
        "oq_nccl_comm_info": ([vp, C.POINTER(i32), C.POINTER(i32)], i32),
        "oq_attention_p2p_exchange_bytes": ([vp, C.POINTER(_Shape), i32], sz),
        "oq_attention_decode_p2p": ([vp, vp, C.POINTER(_Shape), vp, vp, vp, u64, u64, i32, i32,
                                     C.POINTER(vp), C.c_uint32, i32, vp, vp, sz, vp], i32),
        "oq_ipc_handle": ([vp, vp], i32),
        "oq_ipc_open": ([vp, C.POINTER(vp)], i32),
        "oq_ipc_close": ([vp], i32),
        "oq_device_alloc": ([sz, C.POINTER(vp)], i32),
        "oq_device_free": ([vp], i32),
        "oq_device_memset": ([vp, i32, sz], i32),
        "oq_cache_append": ([vp, i32, vp, i32, C.c_uint64, vp, C.c_int64, vp, vp, C.c_uint64, vp],
                            i32),
        "oq_cache_append_kv": ([vp, vp, vp, vp, i32, C.c_uint64, vp, C.c_int64, vp, vp, vp, vp,
                                C.c_uint64, vp], i32),
        "oq_decode": ([vp, vp, sz, vp, vp], i32),
        "oq_wire_header": ([cfgp, u64, C.c_char_p], i32),
        "oq_wire_parse_header": ([C.c_char_p, sz, cfgp, C.POINTER(u64)], i32),
        "oq_validate_records": ([vp, vp, sz, vp], i32),
        "oq_cache_tile_bytes": ([vp, i32], sz),
        "oq_cache_bytes": ([vp, i32, u64], sz),
        "oq_cache_pack": ([vp, i32, vp, u64, u64, u64, vp, u64, vp], i32),
        "oq_attention_workspace_bytes": ([vp, vp, C.POINTER(_Shape), i32], sz),
        "oq_attention_decode": ([vp, vp, C.POINTER(_Shape), vp, vp, vp, vp, i32, vp, sz, vp],
                                i32),
        "oq_attention_partials": ([vp, vp, C.POINTER(_Shape), vp, vp, vp, u64, u64, vp, i32, vp,
                                   sz, vp], i32),
        "oq_attention_combine": ([vp, vp, i32, i32, sz, sz, i32, vp, vp], i32),
        "oq_scores": ([vp, vp, i32, vp, sz, vp, vp], i32),
        "oq_attention_dense_workspace_bytes": ([i32, i32, i32], sz),
        "oq_attention_decode_dense": ([vp, vp, i32, vp, sz, vp, i32, i32, vp, vp, sz, vp], i32),
        "oq_dir_table": ([dp, i32, dp], i32),
        "oq_prepare_f64": ([vp, vp, sz, vp, vp, vp], i32),
        "oq_reconstruct_rotated": ([vp, vp, sz, vp, vp], i32),
        "oq_decode_f64": ([vp, vp, sz, vp, vp], i32),
        "oq_score_prepared": ([vp, vp, vp, sz, vp, sz, vp, vp], i32),
        "oq_attention_f64_workspace_bytes": ([vp, sz, sz], sz),
        "oq_attention_decode_f64": ([vp, vp, sz, vp, sz, vp, i32, i32, vp, vp, sz, vp], i32),
        "oq_timing_enable": ([i32], None),
        "oq_timing_collect": ([C.c_char_p, C.POINTER(C.c_double), C.POINTER(i32)], i32),
    }
    for name, (args, res) in sigs.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def _check(status):
    if status == 0:
        return
    msg = lib().oq_last_error().decode()
    if status == 1:
        raise ValueError(msg)
    if status == 2:
        raise FormatError(msg)
    if status == 4:
        raise NotImplementedError(msg)
    raise RuntimeError(f"CUDA error: {msg}")


def _stream(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _ptr(t):
    return C.c_void_p(t.data_ptr())


def timing(enable=True):
    """Enable CUDA-event timing of the hot kernels (clears previous marks)."""
    lib().oq_timing_enable(1 if enable else 0)


def timing_collect(name):
    """(total_ms, launches) of the timed launches named `name`."""
    t = C.c_double()
    n = C.c_int()
    _check(lib().oq_timing_collect(name.encode(), C.byref(t), C.byref(n)))
    return t.value, n.value


@dataclass
class CodecConfig:
    """CodecConfig (codec.hpp:54-73), same fields and defaults."""
    dim: int = 128
    b_dir: int = 3
    b_nrm: int = 1
    rounding: str = "local3x3"
    rotation_seed: int = 0
    qjl: bool = False
    qjl_seed: int = 1

    def n_tri(self):
        return (self.dim + 2) // 3

    def _c(self):
        if self.rounding not in ROUNDINGS:
            raise ValueError(f"unknown rounding mode: {self.rounding}")
        return _Config(self.dim, self.b_dir, self.b_nrm, ROUNDINGS.index(self.rounding),
                       1 if self.qjl else 0, self.rotation_seed, self.qjl_seed)

    def validate(self):
        c = self._c()
        _check(lib().oq_config_validate(C.byref(c)))

    @staticmethod
    def for_bits(b, **kw):
        bd, bn = default_bit_split(b)
        return CodecConfig(b_dir=bd, b_nrm=bn, **kw)


def default_bit_split(b):
    """codec.hpp:77-80: (b_dir, b_nrm) = (b + 1, b - 1)."""
    bd, bn = C.c_int(), C.c_int()
    _check(lib().oq_default_bit_split(int(b), C.byref(bd), C.byref(bn)))
    return bd.value, bn.value


def parse_rounding(name):
    r = C.c_int()
    _check(lib().oq_parse_rounding(name.encode(), C.byref(r)))
    return ROUNDINGS[r.value]


def effective_bits_per_coord(cfg: CodecConfig):
    c = cfg._c()
    return lib().oq_effective_bits_per_coord(C.byref(c))


def record_bytes(cfg: CodecConfig):
    c = cfg._c()
    return lib().oq_record_bytes(C.byref(c))


def _book(fn, *args, bits):
    c = np.empty(1 << bits)
    b = np.empty(max(1, (1 << bits) - 1))
    _check(fn(*args, bits, c.ctypes.data_as(C.POINTER(C.c_double)),
              b.ctypes.data_as(C.POINTER(C.c_double))))
    return c, b[: (1 << bits) - 1]


def xi_book(bits):
    """books.hpp:69-74 -> (centroids, boundaries), bit-identical fp64."""
    return _book(lib().oq_xi_book, bits=bits)


def rho_book(dim, bits):
    """books.hpp:86-95 -> (centroids, boundaries), bit-identical fp64."""
    return _book(lib().oq_rho_book, dim, bits=bits)


class Encoder:
    """Encoder(cfg) / Encoder(cfg, Books::custom(xi, rho)) on the current GPU."""

    def __init__(self, cfg: CodecConfig, books=None):
        self.cfg = cfg
        c = cfg._c()
        h = C.c_void_p()
        if books is None:
            _check(lib().oq_codec_create(C.byref(c), C.byref(h)))
        else:
            xc = np.ascontiguousarray(books[0], np.float64)
            rc = np.ascontiguousarray(books[1], np.float64)
            xb = int(np.log2(len(xc)))
            rb = int(np.log2(len(rc)))
            if (1 << xb) != len(xc) or (1 << rb) != len(rc):
                raise ValueError("custom books must have 2^bits centroids")
            dp = C.POINTER(C.c_double)
            _check(lib().oq_codec_create_custom(C.byref(c), xc.ctypes.data_as(dp), xb,
                                                rc.ctypes.data_as(dp), rb, C.byref(h)))
        self._h = h
        self.record_bytes = record_bytes(cfg)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.oq_codec_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def config(self):
        return self.cfg

    def compress(self, x, out=None, stream=None, flagged=None):
        """Encoder::encode over rows of a CUDA tensor -> uint8 [n, record_bytes].

        flagged: optional CUDA int32 tensor of one element that receives how
        many keys the certified fp32 pass sent to the exact fp64 path."""
        import torch
        if not x.is_cuda:
            raise ValueError("compress expects a CUDA tensor (there is no CPU path)")
        if x.shape[-1] != self.cfg.dim:
            raise ValueError("key dimension mismatch")
        x = x.contiguous()
        n = x.numel() // self.cfg.dim
        dt = _DTYPES.get(str(x.dtype).replace("torch.", ""))
        if dt is None:
            raise ValueError(f"unsupported dtype {x.dtype}")
        if out is None:
            out = torch.empty((n, self.record_bytes), dtype=torch.uint8, device=x.device)
        fl = None if flagged is None else _ptr(flagged)
        _check(lib().oq_compress_ex(self._h, _ptr(x), dt, n, _ptr(out), fl, _stream(stream)))
        return out

    def decode(self, records, out=None, stream=None):
        """Encoder::decode of OCTO records -> float32 [n, dim]."""
        import torch
        if not records.is_cuda:
            raise ValueError("decode expects a CUDA tensor (there is no CPU path)")
        records = records.contiguous()
        n = records.numel() // self.record_bytes
        if n * self.record_bytes != records.numel():
            raise FormatError("code stream length mismatch")
        if out is None:
            out = torch.empty((n, self.cfg.dim), dtype=torch.float32, device=records.device)
        _check(lib().oq_decode(self._h, _ptr(records), n, _ptr(out), _stream(stream)))
        return out

    def validate_records(self, records, stream=None):
        """unpack_keys padding checks on device; raises FormatError."""
        n = records.numel() // self.record_bytes
        _check(lib().oq_validate_records(self._h, _ptr(records.contiguous()), n,
                                         _stream(stream)))

    # -- single-key convenience mirrors (host fp64 in, like the reference) -----
    def encode(self, k):
        """Encoder::encode(span<const double>) -> one OCTO record (bytes)."""
        import torch
        k = np.asarray(k, np.float64)
        if k.shape != (self.cfg.dim,):
            raise ValueError("key dimension mismatch")
        t = torch.from_numpy(k.copy()).cuda().reshape(1, -1)
        return bytes(self.compress(t).cpu().numpy().tobytes())

    def scores(self, q, records, stream=None):
        """Encoder::score(prepare(q), k) for q [nq, dim] x records [n] -> [nq, n] fp32."""
        import torch
        q = q.contiguous().float().reshape(-1, self.cfg.dim)
        records = records.contiguous()
        n = records.numel() // self.record_bytes
        out = torch.empty((q.shape[0], n), dtype=torch.float32, device=q.device)
        _check(lib().oq_scores(self._h, _ptr(q), q.shape[0], _ptr(records), n, _ptr(out),
                               _stream(stream)))
        return out

    def tile_bytes(self, role):
        return lib().oq_cache_tile_bytes(self._h, role)

    # -- the per-key reference API in exact fp64 (bit-identical) --------------
    def prepare(self, q, stream=None):
        """Encoder::prepare (codec.hpp:282-292) for q [nq, dim]: (rot, sketch)
        float64 CUDA tensors (sketch None without QJL), bit-identical."""
        import torch
        q = q.contiguous().to(torch.float64).reshape(-1, self.cfg.dim)
        rot = torch.empty_like(q)
        sk = torch.empty_like(q) if self.cfg.qjl else None
        _check(lib().oq_prepare_f64(self._h, _ptr(q), q.shape[0], _ptr(rot),
                                    None if sk is None else _ptr(sk), _stream(stream)))
        return rot, sk

    def reconstruct_rotated(self, records, stream=None):
        """Encoder::reconstruct_rotated (codec.hpp:252-266): float64 [n, dim]."""
        import torch
        records = records.contiguous()
        n = records.numel() // self.record_bytes
        out = torch.empty((n, self.cfg.dim), dtype=torch.float64, device=records.device)
        _check(lib().oq_reconstruct_rotated(self._h, _ptr(records), n, _ptr(out),
                                            _stream(stream)))
        return out

    def decode_exact(self, records, stream=None):
        """Encoder::decode (codec.hpp:268-275) in exact fp64: float64 [n, dim]."""
        import torch
        records = records.contiguous()
        n = records.numel() // self.record_bytes
        out = torch.empty((n, self.cfg.dim), dtype=torch.float64, device=records.device)
        _check(lib().oq_decode_f64(self._h, _ptr(records), n, _ptr(out), _stream(stream)))
        return out

    def score_prepared(self, rot, sketch, records, stream=None):
        """Encoder::score(prepared, k) (codec.hpp:295-311): float64 [nq, n]."""
        import torch
        records = records.contiguous()
        n = records.numel() // self.record_bytes
        rot = rot.contiguous().to(torch.float64)
        out = torch.empty((rot.shape[0], n), dtype=torch.float64, device=records.device)
        sk = None if sketch is None else _ptr(sketch.contiguous().to(torch.float64))
        _check(lib().oq_score_prepared(self._h, _ptr(rot), sk, rot.shape[0], _ptr(records), n,
                                       _ptr(out), _stream(stream)))
        return out

    def attention_exact(self, q, records, values, n_splits=1, stream=None):
        """attention_decode(enc, q, keys, values, n_splits) in fp64 on the GPU
        (attention.hpp:50-73): q [nq, dim], values [n, vdim] -> [nq, vdim]."""
        import torch
        q = q.contiguous().to(torch.float64).reshape(-1, self.cfg.dim)
        values = values.contiguous().to(torch.float64)
        records = records.contiguous()
        n = records.numel() // self.record_bytes
        if values.shape[0] != n:
            raise ValueError("values/cache length mismatch")
        L = lib()
        wsb = L.oq_attention_f64_workspace_bytes(self._h, q.shape[0], n)
        ws = torch.empty(max(wsb, 8), dtype=torch.uint8, device=q.device)
        out = torch.empty((q.shape[0], values.shape[1]), dtype=torch.float64, device=q.device)
        _check(L.oq_attention_decode_f64(self._h, _ptr(q), q.shape[0], _ptr(records), n,
                                         _ptr(values), values.shape[1], n_splits, _ptr(out),
                                         _ptr(ws), ws.numel(), _stream(stream)))
        return out


def pack_keys(cfg: CodecConfig, records):
    """pack_keys (codec.hpp:364-396): 20-byte OCTO header + records."""
    c = cfg._c()
    rb = record_bytes(cfg)
    if hasattr(records, "cpu"):
        records = records.cpu().numpy()
    records = np.ascontiguousarray(records, np.uint8).reshape(-1)
    if records.size % rb:
        raise ValueError("key shape does not match config")
    hdr = C.create_string_buffer(20)
    _check(lib().oq_wire_header(C.byref(c), records.size // rb, hdr))
    return hdr.raw + records.tobytes()


def unpack_keys(blob: bytes, device="cuda"):
    """unpack_keys (codec.hpp:410-465) -> (CodecConfig, uint8 records tensor).

    Header and payload size are checked on the host, padding bits on the GPU.
    """
    import torch
    c = _Config()
    cnt = C.c_uint64()
    _check(lib().oq_wire_parse_header(blob, len(blob), C.byref(c), C.byref(cnt)))
    cfg = CodecConfig(dim=c.dim, b_dir=c.b_dir, b_nrm=c.b_nrm, qjl=bool(c.qjl),
                      qjl_seed=1 if c.qjl else 1)
    rb = record_bytes(cfg)
    recs = torch.frombuffer(bytearray(blob[20:]), dtype=torch.uint8).reshape(-1, rb) \
        if cnt.value else torch.empty((0, rb), dtype=torch.uint8)
    recs = recs.to(device)
    if cnt.value:
        enc = Encoder(cfg)
        enc.validate_records(recs)
    return cfg, recs


class KVCache:
    """Compressed K/V cache in the attention tile formats.

    Streams are (batch, kv head) pairs; each holds ``cap_tokens`` tokens in
    32-token tiles (K and V tile formats differ; see attention.cu).
    """

    def __init__(self, enc_k: Encoder, enc_v: Encoder, B, Hkv, cap_tokens, device="cuda"):
        import torch
        self.enc_k, self.enc_v = enc_k, enc_v
        self.B, self.Hkv, self.cap = B, Hkv, int(cap_tokens)
        kt, vt = enc_k.tile_bytes(ROLE_K), enc_v.tile_bytes(ROLE_V)
        if kt == 0 or vt == 0:
            raise NotImplementedError("attention tiles need dim 128 and 2*b_dir+b_nrm in {7, 10, 13} (b = 2, 3, 4 at the default split)")
        ntiles = (self.cap + 31) // 32
        self.k = torch.zeros(B * Hkv * ntiles * kt, dtype=torch.uint8, device=device)
        self.v = torch.zeros(B * Hkv * ntiles * vt, dtype=torch.uint8, device=device)
        self.tokens = 0

    def pack(self, k_records, v_records, n_tokens, rec_stride=None, stream=None):
        """Fill from OCTO records [B*Hkv, rec_stride, rb] (first n_tokens each)."""
        rs = rec_stride if rec_stride is not None else n_tokens
        n = self.B * self.Hkv
        _check(lib().oq_cache_pack(self.enc_k.handle, ROLE_K, _ptr(k_records), n, n_tokens, rs,
                                   _ptr(self.k), self.cap, _stream(stream)))
        _check(lib().oq_cache_pack(self.enc_v.handle, ROLE_V, _ptr(v_records), n, n_tokens, rs,
                                   _ptr(self.v), self.cap, _stream(stream)))
        self.tokens = n_tokens

    def append(self, k, v, pos=None, stream=None, records=None):
        """Decode step: compress one new key and value per stream (k, v: CUDA
        [B, Hkv, dim]) and write them at token ``pos`` (an int, or a CUDA int64
        tensor [B*Hkv] of per-stream positions; default: ``self.tokens``).
        K and V go through ONE fused launch (``oq_cache_append_kv``).
        records: optional (k_records, v_records) uint8 CUDA tensors
        [B*Hkv, record_bytes] that also receive the OCTO records."""
        import torch
        n = self.B * self.Hkv
        p = self.tokens if pos is None else pos
        L = lib()
        k = k.contiguous().reshape(n, self.enc_k.cfg.dim)
        v = v.contiguous().reshape(n, self.enc_v.cfg.dim)
        if v.dtype != k.dtype:
            v = v.to(k.dtype)
        dt = _DTYPES.get(str(k.dtype).replace("torch.", ""))
        if dt is None:
            raise ValueError(f"unsupported dtype {k.dtype}")
        if isinstance(p, int):
            pd, ps = None, p
        else:
            pos_t = p.contiguous().to(torch.int64)
            pd, ps = _ptr(pos_t), 0
        rk, rv = (None, None) if records is None else (_ptr(records[0]), _ptr(records[1]))
        _check(L.oq_cache_append_kv(self.enc_k.handle, self.enc_v.handle, _ptr(k), _ptr(v), dt, n,
                                    pd, ps, rk, rv, _ptr(self.k), _ptr(self.v), self.cap,
                                    _stream(stream)))
        if isinstance(p, int):
            self.tokens = max(self.tokens, p + 1)

    def nbytes_per_token(self):
        return (self.enc_k.tile_bytes(ROLE_K) + self.enc_v.tile_bytes(ROLE_V)) / 32.0


def default_splits(B, Hkv, Hq, T, num_sms=None):
    """Split-K count for the persistent attention grid (one CTA per SM).

    Work items = B*Hkv*ceil(G/8)*splits; pick the split count whose item
    count is closest to a whole number of waves over the SMs (exact when
    possible, e.g. 32 streams x 37 splits = 8 x 148), with each item at least
    16 tiles long so its merge epilogue stays amortized."""
    if num_sms is None:
        try:
            import torch
            num_sms = torch.cuda.get_device_properties(0).multi_processor_count
        except Exception:
            num_sms = 148
    hc = (Hq // Hkv + 7) // 8
    streams = B * Hkv * hc
    tiles = max(1, (T + 31) // 32)
    best, best_eff = 1, -1.0
    for s in range(1, max(1, tiles // 16) + 1):
        items = streams * s
        waves = -(-items // num_sms)
        eff = items / (waves * num_sms) - 0.002 * waves  # busy SM fraction, fewer waves
        if eff > best_eff + 1e-9:
            best, best_eff = s, eff
        if waves > 16:
            break
    return best


class _Workspace:
    """Per-(device, stream, kind) device scratch for the attention calls.

    The tile-attention workspace's first 64 KiB are arrival counters the fused
    kernel requires to be zero on entry (and leaves at zero), so one buffer is
    never shared between streams: calls on different streams would race on the
    counters and partials.  A buffer is allocated and zero-filled ON the launch
    stream (ordered before the kernel that first uses it).  A buffer that is
    outgrown is retired, never freed: a kernel still in flight or a captured
    CUDA graph may reference it."""
    buf = {}
    _retired = []

    @classmethod
    def get(cls, nbytes, device, stream, kind="tile"):
        import torch
        key = (str(device), int(stream.cuda_stream), kind)
        b = cls.buf.get(key)
        if b is None or b.numel() < nbytes:
            if b is not None:
                cls._retired.append(b)
            with torch.cuda.stream(stream):
                b = torch.zeros(max(nbytes, 1 << 20), dtype=torch.uint8, device=device)
            cls.buf[key] = b
        return b


def _launch_stream(stream, device):
    """The torch stream a call launches on (the caller's, or the current one)."""
    import torch
    return stream if stream is not None else torch.cuda.current_stream(device)


def _check_query(q, cache):
    if not q.is_cuda:
        raise ValueError("q must be a CUDA tensor (there is no CPU path)")
    if q.dim() != 3 or q.shape[0] != cache.B:
        raise ValueError("q must be [B, Hq, dim] with B matching the cache")
    if q.shape[-1] != cache.enc_k.cfg.dim:
        raise ValueError("query dimension mismatch")


def _check_seq_lens(seq_lens, B, device):
    import torch
    if seq_lens is None:
        return
    if (not seq_lens.is_cuda or seq_lens.dtype != torch.int32 or seq_lens.dim() != 1
            or seq_lens.numel() != B or seq_lens.device != device):
        raise ValueError("seq_lens must be an int32 CUDA tensor of length B on q's device")
    if not seq_lens.is_contiguous():
        raise ValueError("seq_lens must be contiguous")


def _shape(cache: KVCache, Hq, T, seq_lens):
    return _Shape(cache.B, Hq, cache.Hkv, T, cache.cap,
                  seq_lens.data_ptr() if seq_lens is not None else None)


def attention_decode(q, cache: KVCache, n_splits=None, seq_lens=None, T=None, out=None,
                     stream=None):
    """attention_decode (attention.hpp:50-73), batched GQA over compressed K and V.

    q: CUDA float32 [B, Hq, dim].  Returns [B, Hq, dim] float32.  n_splits:
    None/0 = stream-K (balanced over the SMs); k >= 1 = k contiguous chunks
    per stream, the reference's n_splits.  seq_lens: optional int32 CUDA [B].
    Everything (scratch, the fp32 copy of q, out) is allocated on the launch
    stream, ``stream`` or the current one.
    """
    import torch
    _check_query(q, cache)
    _check_seq_lens(seq_lens, cache.B, q.device)
    B, Hq, D = q.shape
    T = cache.tokens if T is None else T
    if n_splits is None:
        n_splits = 0  # stream-K: every SM gets an equal contiguous share of all tiles
    sh = _shape(cache, Hq, T, seq_lens)
    L = lib()
    ws_bytes = L.oq_attention_workspace_bytes(cache.enc_k.handle, cache.enc_v.handle,
                                              C.byref(sh), n_splits)
    st = _launch_stream(stream, q.device)
    with torch.cuda.stream(st):
        ws = _Workspace.get(ws_bytes, q.device, st)
        if out is None:
            out = torch.empty((B, Hq, D), dtype=torch.float32, device=q.device)
        q = q.contiguous().float()
        _check(L.oq_attention_decode(cache.enc_k.handle, cache.enc_v.handle, C.byref(sh),
                                     _ptr(q), _ptr(cache.k), _ptr(cache.v), _ptr(out), n_splits,
                                     _ptr(ws), ws.numel(), C.c_void_p(st.cuda_stream)))
    return out


class AttentionPipeline:
    """Serving loop for attention_decode with HOST queries and outputs.

    Each ``run(q_host, out_host)`` copies that step's queries host -> device,
    runs the fused attention and copies the output device -> host, on three
    streams with double-buffered device q / out, so step i+1's upload and step
    i's download overlap the attention kernels instead of serialising with
    them on one stream.  q_host / out_host: pinned CPU float32 [B, Hq, dim];
    out_host is complete once ``synchronize()`` (or the step's event from
    ``run``) has passed.  Every step still moves its own inputs and outputs.
    """

    def __init__(self, cache: KVCache, Hq, n_splits=0, seq_lens=None, device=None, step=None):
        """step: optional callable (q_dev, out_dev, stream) running the
        attention itself (e.g. a sequence-sharded call); default
        attention_decode over ``cache``."""
        import torch
        self.cache, self.Hq, self.n_splits, self.seq_lens = cache, Hq, n_splits, seq_lens
        self.step = step
        dev = device if device is not None else cache.k.device
        D = cache.enc_k.cfg.dim
        self.dev = dev
        self.q = [torch.empty((cache.B, Hq, D), dtype=torch.float32, device=dev) for _ in range(2)]
        self.out = [torch.empty((cache.B, Hq, D), dtype=torch.float32, device=dev)
                    for _ in range(2)]
        self.compute = torch.cuda.Stream(device=dev)
        self.h2d = torch.cuda.Stream(device=dev)
        self.d2h = torch.cuda.Stream(device=dev)
        self.q_ready = [torch.cuda.Event() for _ in range(2)]
        self.q_free = [torch.cuda.Event() for _ in range(2)]
        self.out_ready = [torch.cuda.Event() for _ in range(2)]
        self.out_free = [torch.cuda.Event() for _ in range(2)]
        self.done = [torch.cuda.Event() for _ in range(2)]
        self.i = 0
        for e in self.q_free + self.out_free:  # both buffers start free
            e.record(self.compute)

    def run(self, q_host, out_host):
        import torch
        j = self.i & 1
        self.i += 1
        with torch.cuda.stream(self.h2d):
            self.h2d.wait_event(self.q_free[j])      # step i-2's kernel has read q[j]
            self.q[j].copy_(q_host, non_blocking=True)
            self.q_ready[j].record(self.h2d)
        self.compute.wait_event(self.q_ready[j])
        self.compute.wait_event(self.out_free[j])    # step i-2's download of out[j] is done
        if self.step is not None:
            with torch.cuda.stream(self.compute):
                self.step(self.q[j], self.out[j], self.compute)
        else:
            attention_decode(self.q[j], self.cache, n_splits=self.n_splits,
                             seq_lens=self.seq_lens, out=self.out[j], stream=self.compute)
        self.q_free[j].record(self.compute)
        self.out_ready[j].record(self.compute)
        with torch.cuda.stream(self.d2h):
            self.d2h.wait_event(self.out_ready[j])
            out_host.copy_(self.out[j], non_blocking=True)
            self.out_free[j].record(self.d2h)
            self.done[j].record(self.d2h)
        return self.done[j]

    def synchronize(self):
        for s in (self.h2d, self.compute, self.d2h):
            s.synchronize()


def attention_decode_dense(enc: Encoder, q, records, values, n_splits=1, stream=None):
    """attention_decode(enc, q, keys, values, n_splits) (attention.hpp:50-73) for any
    codec config: q [nq, dim] fp32, keys as OCTO records [n], dense values
    [n, vdim] fp32 -> [nq, vdim]."""
    import torch
    if q.shape[-1] != enc.cfg.dim:
        raise ValueError("query dimension mismatch")
    st = _launch_stream(stream, q.device)
    with torch.cuda.stream(st):
        q = q.contiguous().float().reshape(-1, enc.cfg.dim)
        records = records.contiguous()
        values = values.contiguous().float()
        n = records.numel() // enc.record_bytes
        nq, vdim = q.shape[0], values.shape[-1] if values.dim() > 1 else 1
        if values.shape[0] != n:
            raise ValueError("values/cache length mismatch")
        L = lib()
        ws_bytes = L.oq_attention_dense_workspace_bytes(nq, max(1, n_splits), vdim)
        ws = _Workspace.get(ws_bytes, q.device, st, kind="dense")
        out = torch.empty((nq, vdim), dtype=torch.float32, device=q.device)
        _check(L.oq_attention_decode_dense(enc.handle, _ptr(q), nq, _ptr(records), n,
                                           _ptr(values), vdim, n_splits, _ptr(out), _ptr(ws),
                                           ws.numel(), C.c_void_p(st.cuda_stream)))
    return out


def attention_partials(q, cache: KVCache, t_begin, t_end, n_splits=None, T=None, seq_lens=None,
                       out=None, stream=None):
    """SoftmaxState of tokens [t_begin, t_end) per (b, q head): [B*Hq, 132] fp32."""
    import torch
    _check_query(q, cache)
    _check_seq_lens(seq_lens, cache.B, q.device)
    B, Hq, D = q.shape
    T = cache.tokens if T is None else T
    if n_splits is None:
        n_splits = 0
    sh = _shape(cache, Hq, T, seq_lens)
    L = lib()
    ws_bytes = L.oq_attention_workspace_bytes(cache.enc_k.handle, cache.enc_v.handle,
                                              C.byref(sh), n_splits)
    st = _launch_stream(stream, q.device)
    with torch.cuda.stream(st):
        ws = _Workspace.get(ws_bytes, q.device, st)
        if out is None:
            out = torch.empty((B * Hq, 4 + D), dtype=torch.float32, device=q.device)
        q = q.contiguous().float()
        _check(L.oq_attention_partials(cache.enc_k.handle, cache.enc_v.handle, C.byref(sh),
                                       _ptr(q), _ptr(cache.k), _ptr(cache.v), t_begin, t_end,
                                       _ptr(out), n_splits, _ptr(ws), ws.numel(),
                                       C.c_void_p(st.cuda_stream)))
    return out


class NcclComm:
    """An NCCL communicator created through the library's own NCCL loader
    (libnccl.so.2): ``uid = NcclComm.unique_id()`` on one rank, share it, then
    ``NcclComm(nranks, uid, rank)`` on every rank (one GPU each)."""

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        _check(lib().oq_nccl_get_unique_id(buf))
        return bytes(buf)

    def __init__(self, nranks: int, uid: bytes, rank: int):
        self.nranks, self.rank = nranks, rank
        self.handle = C.c_void_p()
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        _check(lib().oq_nccl_comm_init_rank(C.byref(self.handle), nranks, buf, rank))

    def info(self):
        """(rank, nranks) as NCCL reports them (ncclCommUserRank / ncclCommCount)."""
        r, n = C.c_int(), C.c_int()
        _check(lib().oq_nccl_comm_info(self.handle, C.byref(r), C.byref(n)))
        return r.value, n.value

    def close(self):
        if self.handle:
            _check(lib().oq_nccl_comm_destroy(self.handle))
            self.handle = C.c_void_p()


def attention_decode_sharded(q, cache: KVCache, t_begin, t_end, comm: NcclComm, n_splits=None,
                             T=None, out=None, stream=None):
    """Sequence-sharded attention_decode: this rank's tokens [t_begin, t_end),
    one NCCL all-gather of the partials, rank-ordered merge (identical output
    on every rank)."""
    import torch
    _check_query(q, cache)
    B, Hq, D = q.shape
    T = cache.tokens if T is None else T
    n_splits = 0 if n_splits is None else n_splits
    sh = _shape(cache, Hq, T, None)
    L = lib()
    ws_bytes = L.oq_attention_sharded_workspace_bytes(cache.enc_k.handle, cache.enc_v.handle,
                                                      C.byref(sh), n_splits, comm.nranks)
    st = _launch_stream(stream, q.device)
    with torch.cuda.stream(st):
        ws = _Workspace.get(ws_bytes, q.device, st)
        if out is None:
            out = torch.empty((B, Hq, D), dtype=torch.float32, device=q.device)
        q = q.contiguous().float()
        _check(L.oq_attention_decode_sharded(cache.enc_k.handle, cache.enc_v.handle,
                                             C.byref(sh), _ptr(q), _ptr(cache.k), _ptr(cache.v),
                                             t_begin, t_end, comm.handle, comm.nranks, _ptr(out),
                                             n_splits, _ptr(ws), ws.numel(),
                                             C.c_void_p(st.cuda_stream)))
    return out


def p2p_exchange_bytes(cache: KVCache, Hq, nranks):
    """Bytes of one rank's exchange buffer for attention_decode_p2p."""
    sh = _shape(cache, Hq, cache.cap, None)
    return lib().oq_attention_p2p_exchange_bytes(cache.enc_k.handle, C.byref(sh), nranks)


def attention_decode_p2p(q, cache: KVCache, t_begin, t_end, rank, nranks, xbufs, epoch, T=None,
                         out=None, max_ctas=0, stream=None):
    """Sequence-sharded attention_decode fused over peer memory (one launch, no
    collective library): this rank's tokens [t_begin, t_end) of ``cache``;
    ``xbufs`` = the nranks exchange buffers (device pointers as mapped in this
    process, or CUDA tensors); ``epoch`` nonzero and increasing per call.
    Every rank gets the same [B, Hq, dim] output (oq_attention_decode_p2p)."""
    import torch
    _check_query(q, cache)
    B, Hq, D = q.shape
    T = cache.tokens if T is None else T
    sh = _shape(cache, Hq, T, None)
    L = lib()
    ws_bytes = L.oq_attention_workspace_bytes(cache.enc_k.handle, cache.enc_v.handle,
                                              C.byref(sh), 0)
    st = _launch_stream(stream, q.device)
    ptrs = (C.c_void_p * nranks)(*[C.c_void_p(x.data_ptr() if hasattr(x, "data_ptr") else int(x))
                                   for x in xbufs])
    with torch.cuda.stream(st):
        ws = _Workspace.get(ws_bytes, q.device, st)
        if out is None:
            out = torch.empty((B, Hq, D), dtype=torch.float32, device=q.device)
        q = q.contiguous().float()
        _check(L.oq_attention_decode_p2p(cache.enc_k.handle, cache.enc_v.handle, C.byref(sh),
                                         _ptr(q), _ptr(cache.k), _ptr(cache.v), t_begin, t_end,
                                         rank, nranks, ptrs, epoch, max_ctas, _ptr(out), _ptr(ws),
                                         ws.numel(), C.c_void_p(st.cuda_stream)))
    return out


class P2PExchange:
    """The exchange buffers of attention_decode_p2p across one process per GPU:
    this rank's buffer comes from cudaMalloc (zero-filled), its CUDA IPC handle
    is shared through torch.distributed (``group``), and the peers' buffers are
    mapped into this process.  ``decode`` is then one fused launch per step."""

    def __init__(self, cache: KVCache, Hq, group=None):
        import torch.distributed as dist
        self.rank, self.nranks = dist.get_rank(group), dist.get_world_size(group)
        L = lib()
        nbytes = p2p_exchange_bytes(cache, Hq, self.nranks)
        own = C.c_void_p()
        _check(L.oq_device_alloc(nbytes, C.byref(own)))
        _check(L.oq_device_memset(own, 0, nbytes))
        self._own = own
        h = (C.c_uint8 * 64)()
        _check(L.oq_ipc_handle(own, h))
        handles = [None] * self.nranks
        dist.all_gather_object(handles, bytes(h), group=group)
        self.ptrs, self._opened = [], []
        for r, hb in enumerate(handles):
            if r == self.rank:
                self.ptrs.append(own.value)
                continue
            peer = C.c_void_p()
            _check(L.oq_ipc_open((C.c_uint8 * 64).from_buffer_copy(hb), C.byref(peer)))
            self.ptrs.append(peer.value)
            self._opened.append(peer)
        dist.barrier(group=group)
        self.epoch = 0

    def decode(self, q, cache: KVCache, t_begin, t_end, out=None, stream=None):
        self.epoch += 1
        return attention_decode_p2p(q, cache, t_begin, t_end, self.rank, self.nranks, self.ptrs,
                                    self.epoch, out=out, stream=stream)

    def close(self):
        L = lib()
        for peer in self._opened:
            L.oq_ipc_close(peer)
        self._opened = []
        if self._own:
            L.oq_device_free(self._own)
            self._own = None


def attention_combine(enc_v: Encoder, partials, rows, n_parts, row_stride, part_stride,
                      finalize=True, out=None, stream=None):
    """Merge partials in token order (SoftmaxState::merge) and finalize."""
    import torch
    D = enc_v.cfg.dim
    if out is None:
        out = torch.empty((rows, D if finalize else 4 + D), dtype=torch.float32,
                          device=partials.device)
    _check(lib().oq_attention_combine(enc_v.handle, _ptr(partials), rows, n_parts, row_stride,
                                      part_stride, 1 if finalize else 0, _ptr(out),
                                      _stream(stream)))
    return out
