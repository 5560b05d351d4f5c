"""ctypes bindings to the parity checkers (test infrastructure only).

* ``Oracle``  -> oracle/liboctoquant_oracle.so (C restatement)
* ``RefLib``  -> oracle/_ref/libocto_ref.so (the reference headers compiled)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg import
this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboctoquant_oracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libocto_ref.so")

_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_u8p = C.POINTER(C.c_uint8)
_u16p = C.POINTER(C.c_uint16)


def _ptr(a, t):
    return a.ctypes.data_as(t)


class OrcConfig(C.Structure):
    _fields_ = [
        ("dim", C.c_uint32),
        ("b_dir", C.c_uint8),
        ("b_nrm", C.c_uint8),
        ("rounding", C.c_uint8),
        ("qjl", C.c_uint8),
        ("rotation_seed", C.c_uint64),
        ("qjl_seed", C.c_uint64),
    ]


ROUNDING = {"scalar": 0, "local2x2": 1, "local3x3": 2, "full": 3}


def record_bytes(dim, b_dir, b_nrm, qjl):
    nt = (dim + 2) // 3
    r = 4 + (2 * nt * b_dir + 7) // 8 + (nt * b_nrm + 7) // 8
    if qjl:
        r += 2 + (dim + 7) // 8
    return r


class Oracle:
    def __init__(self, path=ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = self.L = C.CDLL(path)
        L.orc_mix64.restype = C.c_uint64
        L.orc_mix64.argtypes = [C.c_uint64]
        L.orc_stream_child.restype = C.c_uint64
        L.orc_stream_child.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_stream_at.restype = C.c_uint64
        L.orc_stream_at.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_fill_gaussian.restype = C.c_uint64
        L.orc_fill_gaussian.argtypes = [C.c_uint64, C.c_uint64, _dp, C.c_size_t]
        L.orc_gaussian_f32.argtypes = [C.c_uint64, C.c_size_t, _fp]
        L.orc_f32_to_f16.restype = C.c_uint16
        L.orc_f32_to_f16.argtypes = [C.c_float]
        L.orc_f16_to_f32.restype = C.c_float
        L.orc_f16_to_f32.argtypes = [C.c_uint16]
        L.orc_rotation_signs.argtypes = [C.c_uint32, C.c_uint64, _dp]
        L.orc_fwht.argtypes = [_dp, C.c_size_t]
        L.orc_oct_encode.argtypes = [_dp, _dp]
        L.orc_oct_decode.argtypes = [C.c_double, C.c_double, _dp]
        L.orc_xi_book.argtypes = [C.c_int, _dp, _dp]
        L.orc_rho_book.argtypes = [C.c_uint32, C.c_int, _dp, _dp]
        L.orc_quantize.restype = C.c_uint32
        L.orc_quantize.argtypes = [_dp, C.c_uint32, C.c_double]
        L.orc_encoder_new.restype = C.c_void_p
        L.orc_encoder_new.argtypes = [C.POINTER(OrcConfig)]
        L.orc_encoder_free.argtypes = [C.c_void_p]
        L.orc_record_bytes.restype = C.c_size_t
        L.orc_record_bytes.argtypes = [C.POINTER(OrcConfig)]
        L.orc_encode_record.argtypes = [C.c_void_p, _dp, _u8p]
        L.orc_encode_f32.argtypes = [C.c_void_p, _fp, C.c_size_t, _u8p, C.c_int]
        L.orc_decode_records.restype = C.c_int
        L.orc_decode_records.argtypes = [C.c_void_p, _u8p, C.c_size_t, _dp]
        L.orc_score.restype = C.c_double
        L.orc_score.argtypes = [C.c_void_p, _dp, _u8p]
        L.orc_attention.restype = C.c_int
        L.orc_attention.argtypes = [C.c_void_p, _dp, _u8p, C.c_size_t, _dp, C.c_size_t,
                                    C.c_int, _dp]
        L.orc_attention_partial.argtypes = [C.c_void_p, _dp, _u8p, C.c_size_t, C.c_size_t,
                                            _dp, C.c_size_t, _dp, _dp, _dp]
        L.orc_wire_header.argtypes = [C.POINTER(OrcConfig), C.c_uint64, _u8p]
        L.orc_unpack_check.restype = C.c_int
        L.orc_unpack_check.argtypes = [_u8p, C.c_size_t, C.POINTER(OrcConfig),
                                       C.POINTER(C.c_uint64)]
        L.orc_record_codes.restype = C.c_int
        L.orc_record_codes.argtypes = [C.POINTER(OrcConfig), _u8p, _fp, _u16p, _u16p, _u16p,
                                       _u8p]

    # -- small helpers -------------------------------------------------------
    def gaussian_f32(self, seed, n):
        out = np.empty(n, np.float32)
        self.L.orc_gaussian_f32(seed, n, _ptr(out, _fp))
        return out

    def xi_book(self, bits):
        c = np.empty(1 << bits)
        b = np.empty((1 << bits) - 1 or 1)
        assert self.L.orc_xi_book(bits, _ptr(c, _dp), _ptr(b, _dp)) == 0
        return c, b[: (1 << bits) - 1]

    def rho_book(self, dim, bits):
        c = np.empty(1 << bits)
        b = np.empty((1 << bits) - 1 or 1)
        assert self.L.orc_rho_book(dim, bits, _ptr(c, _dp), _ptr(b, _dp)) == 0
        return c, b[: (1 << bits) - 1]

    def encoder(self, **kw):
        return OracleEncoder(self, **kw)


def make_config(dim=128, b_dir=3, b_nrm=1, rounding="local3x3", rotation_seed=0, qjl=False,
                qjl_seed=1):
    return OrcConfig(dim, b_dir, b_nrm, ROUNDING[rounding] if isinstance(rounding, str)
                     else rounding, 1 if qjl else 0, rotation_seed, qjl_seed)


class OracleEncoder:
    def __init__(self, orc: Oracle, **kw):
        self.orc = orc
        self.cfg = make_config(**kw)
        self.h = orc.L.orc_encoder_new(C.byref(self.cfg))
        if not self.h:
            raise ValueError("invalid codec config")
        self.dim = self.cfg.dim
        self.rb = orc.L.orc_record_bytes(C.byref(self.cfg))

    def __del__(self):
        if getattr(self, "h", None):
            self.orc.L.orc_encoder_free(self.h)

    def encode_f32(self, x, threads=8):
        x = np.ascontiguousarray(x, np.float32).reshape(-1, self.dim)
        out = np.zeros((x.shape[0], self.rb), np.uint8)
        self.orc.L.orc_encode_f32(self.h, _ptr(x, _fp), x.shape[0], _ptr(out, _u8p), threads)
        return out

    def encode_f64(self, k):
        k = np.ascontiguousarray(k, np.float64)
        out = np.zeros(self.rb, np.uint8)
        self.orc.L.orc_encode_record(self.h, _ptr(k, _dp), _ptr(out, _u8p))
        return out

    def decode(self, recs):
        recs = np.ascontiguousarray(recs, np.uint8).reshape(-1, self.rb)
        out = np.empty((recs.shape[0], self.dim))
        rc = self.orc.L.orc_decode_records(self.h, _ptr(recs, _u8p), recs.shape[0],
                                           _ptr(out, _dp))
        if rc:
            raise ValueError("FormatError")
        return out

    def score(self, q, rec):
        q = np.ascontiguousarray(q, np.float64)
        rec = np.ascontiguousarray(rec, np.uint8)
        return self.orc.L.orc_score(self.h, _ptr(q, _dp), _ptr(rec, _u8p))

    def attention(self, q, krecs, values, n_splits=1):
        q = np.ascontiguousarray(q, np.float64)
        krecs = np.ascontiguousarray(krecs, np.uint8)
        values = np.ascontiguousarray(values, np.float64)
        out = np.empty(values.shape[1])
        rc = self.orc.L.orc_attention(self.h, _ptr(q, _dp), _ptr(krecs, _u8p),
                                      krecs.shape[0], _ptr(values, _dp), values.shape[1],
                                      n_splits, _ptr(out, _dp))
        if rc:
            raise ValueError("invalid argument")
        return out

    def partial(self, q, krecs, begin, end, values):
        q = np.ascontiguousarray(q, np.float64)
        krecs = np.ascontiguousarray(krecs, np.uint8)
        values = np.ascontiguousarray(values, np.float64)
        m = C.c_double()
        l = C.c_double()
        acc = np.empty(values.shape[1])
        self.orc.L.orc_attention_partial(self.h, _ptr(q, _dp), _ptr(krecs, _u8p), begin, end,
                                         _ptr(values, _dp), values.shape[1], C.byref(m),
                                         C.byref(l), _ptr(acc, _dp))
        return m.value, l.value, acc

    def codes(self, rec):
        nt = (self.dim + 2) // 3
        g = C.c_float()
        d = np.empty(2 * nt, np.uint16)
        n = np.empty(nt, np.uint16)
        gr = C.c_uint16()
        s = np.empty(max(1, (self.dim + 7) // 8), np.uint8)
        rec = np.ascontiguousarray(rec, np.uint8)
        rc = self.orc.L.orc_record_codes(C.byref(self.cfg), _ptr(rec, _u8p), C.byref(g),
                                         _ptr(d, _u16p), _ptr(n, _u16p), C.byref(gr),
                                         _ptr(s, _u8p))
        if rc:
            raise ValueError("FormatError")
        return g.value, d, n, gr.value, s


class RefLib:
    """The reference implementation itself (compiled headers)."""

    def __init__(self, path=REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` where "
                                    "/root/reference exists")
        L = self.L = C.CDLL(path)
        L.ref_xi_book.argtypes = [C.c_int, _dp, _dp]
        L.ref_rho_book.argtypes = [C.c_uint32, C.c_int, _dp, _dp]
        L.ref_encoder_new.restype = C.c_void_p
        L.ref_encoder_new.argtypes = [C.c_uint32, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int,
                                      C.c_uint64]
        L.ref_encoder_free.argtypes = [C.c_void_p]
        L.ref_encode_f32.argtypes = [C.c_void_p, _fp, C.c_size_t, _u8p, C.c_int]
        L.ref_decode.restype = C.c_int
        L.ref_decode.argtypes = [C.c_void_p, _u8p, C.c_size_t, _dp, C.c_int]
        L.ref_score.restype = C.c_double
        L.ref_score.argtypes = [C.c_void_p, _dp, _u8p]
        L.ref_attention.restype = C.c_int
        L.ref_attention.argtypes = [C.c_void_p, _dp, C.c_size_t, _u8p, C.c_size_t, _dp,
                                    C.c_size_t, C.c_int, _dp, C.c_int]
        L.ref_cache_new.restype = C.c_void_p
        L.ref_cache_new.argtypes = [C.c_void_p, C.c_void_p, _u8p, _u8p, C.c_size_t]
        L.ref_cache_free.argtypes = [C.c_void_p]
        L.ref_cache_attention.restype = C.c_int
        L.ref_cache_attention.argtypes = [C.c_void_p, _dp, C.c_size_t, _dp, C.c_int]
        L.ref_unpack_repack.restype = C.c_size_t
        L.ref_unpack_repack.argtypes = [_u8p, C.c_size_t, _u8p]

    def xi_book(self, bits):
        c = np.empty(1 << bits)
        b = np.empty(max(1, (1 << bits) - 1))
        self.L.ref_xi_book(bits, _ptr(c, _dp), _ptr(b, _dp))
        return c, b[: (1 << bits) - 1]

    def rho_book(self, dim, bits):
        c = np.empty(1 << bits)
        b = np.empty(max(1, (1 << bits) - 1))
        self.L.ref_rho_book(dim, bits, _ptr(c, _dp), _ptr(b, _dp))
        return c, b[: (1 << bits) - 1]

    def encoder(self, dim=128, b_dir=3, b_nrm=1, rounding="local3x3", rotation_seed=0, qjl=False,
                qjl_seed=1):
        return RefEncoder(self, dim, b_dir, b_nrm, ROUNDING[rounding], rotation_seed, qjl,
                          qjl_seed)


class RefEncoder:
    def __init__(self, lib, dim, b_dir, b_nrm, rounding, rot, qjl, qjl_seed):
        self.lib = lib
        self.h = lib.L.ref_encoder_new(dim, b_dir, b_nrm, rounding, rot, 1 if qjl else 0,
                                       qjl_seed)
        if not self.h:
            raise ValueError("invalid codec config")
        self.dim = dim
        self.rb = record_bytes(dim, b_dir, b_nrm, qjl)

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.L.ref_encoder_free(self.h)

    def encode_f32(self, x, threads=8):
        x = np.ascontiguousarray(x, np.float32).reshape(-1, self.dim)
        out = np.zeros((x.shape[0], self.rb), np.uint8)
        self.lib.L.ref_encode_f32(self.h, _ptr(x, _fp), x.shape[0], _ptr(out, _u8p), threads)
        return out

    def decode(self, recs, threads=8):
        recs = np.ascontiguousarray(recs, np.uint8).reshape(-1, self.rb)
        out = np.empty((recs.shape[0], self.dim))
        if self.lib.L.ref_decode(self.h, _ptr(recs, _u8p), recs.shape[0], _ptr(out, _dp),
                                 threads):
            raise ValueError("FormatError")
        return out

    def score(self, q, rec):
        q = np.ascontiguousarray(q, np.float64)
        rec = np.ascontiguousarray(rec, np.uint8)
        return self.lib.L.ref_score(self.h, _ptr(q, _dp), _ptr(rec, _u8p))

    def attention(self, q, krecs, values, n_splits=1, threads=8):
        q = np.ascontiguousarray(q, np.float64).reshape(-1, self.dim)
        krecs = np.ascontiguousarray(krecs, np.uint8)
        values = np.ascontiguousarray(values, np.float64)
        out = np.empty((q.shape[0], values.shape[1]))
        if self.lib.L.ref_attention(self.h, _ptr(q, _dp), q.shape[0], _ptr(krecs, _u8p),
                                    krecs.shape[0], _ptr(values, _dp), values.shape[1],
                                    n_splits, _ptr(out, _dp), threads):
            raise ValueError("invalid argument")
        return out


class RefCache:
    """A CPU-resident compressed K/V cache held as the reference's
    CompressedKey vectors (records unpacked once); attention() runs, per call,
    Encoder::decode of every V key and attention_decode per query row."""

    def __init__(self, ek: RefEncoder, ev: RefEncoder, krecs, vrecs):
        self.lib = ek.lib
        self.ek, self.ev = ek, ev  # keep the encoders alive
        self._k = np.ascontiguousarray(krecs, np.uint8)
        self._v = np.ascontiguousarray(vrecs, np.uint8)
        self.n = self._k.shape[0]
        self.h = self.lib.L.ref_cache_new(ek.h, ev.h, _ptr(self._k, _u8p), _ptr(self._v, _u8p),
                                          self.n)
        if not self.h:
            raise ValueError("FormatError")

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.L.ref_cache_free(self.h)

    def attention(self, q, threads=1):
        q = np.ascontiguousarray(q, np.float64).reshape(-1, self.ek.dim)
        out = np.empty((q.shape[0], self.ev.dim))
        if self.lib.L.ref_cache_attention(self.h, _ptr(q, _dp), q.shape[0], _ptr(out, _dp),
                                          threads):
            raise ValueError("invalid argument")
        return out
