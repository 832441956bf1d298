"""ctypes binding of the CPU oracle — TEST INFRASTRUCTURE ONLY.

The oracle (oracle/gsr_oracle.hpp) is a from-scratch CPU restatement of
/root/reference/SPEC.md and PAPER.md Alg. 1-2 / Eq. 6-7. Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this module; the product package never does.

Arrays are numpy, row-major. `dtype` selects the f32 or f64 instantiation.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libgsr_oracle.so")
_lib = None

MODE_ALG12, MODE_GSRC, MODE_REV = 0, 1, 2
NORM_NONE, NORM_ROW_MEAN, NORM_SYM = 0, 1, 2
EPI_NONE, EPI_ADD, EPI_SUB, EPI_SCATTER_ADD, EPI_SCATTER_SUB = range(5)


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code


def build():
    subprocess.check_call(["make", "-s", "-C", _HERE])


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = C.CDLL(_LIB_PATH)
        _lib.gsro_last_error.restype = C.c_char_p
        for name in ("gsro_graph_create", "gsro_graph_from_edges", "gsro_net_create_f32", "gsro_net_create_f64"):
            getattr(_lib, name).restype = C.c_void_p
        _lib.gsro_graph_e.restype = C.c_longlong
        _lib.gsro_net_num_params.restype = C.c_longlong
        _lib.gsro_work_muladds.restype = C.c_ulonglong
        _lib.gsro_mse_f32.restype = C.c_double
        _lib.gsro_mse_f64.restype = C.c_double
    return _lib


def _chk(st):
    if st != 0:
        raise OracleError(st, lib().gsro_last_error().decode())


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _sfx(dtype):
    return "f64" if np.dtype(dtype) == np.float64 else "f32"


def set_tf32(on):
    """TF32 transform mode: both operands of every block transform (and of the
    GSR-C dW product) read as TF32 by truncation, as the B200 tensor core reads
    fp32 operands (measured: scratch/tf32_probe.cu)."""
    _chk(lib().gsro_set_tf32(int(bool(on))))


def set_threads(n):
    _chk(lib().gsro_set_threads(int(n)))


def work_reset():
    lib().gsro_work_reset()


def work_muladds():
    return int(lib().gsro_work_muladds())


class Graph:
    """CsrGraph with cached transpose."""

    def __init__(self, row_ptr, col_idx, norm=NORM_NONE):
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(col_idx, dtype=np.int32)
        self.n = rp.size - 1
        self.e = ci.size
        h = lib().gsro_graph_create(C.c_longlong(self.n), C.c_longlong(self.e), _p(rp), _p(ci), int(norm))
        if not h:
            raise OracleError(1, lib().gsro_last_error().decode())
        self.h = C.c_void_p(h)
        self.norm = norm

    @classmethod
    def from_edges(cls, n, pairs, norm=NORM_NONE):
        uv = np.ascontiguousarray(np.asarray(pairs, dtype=np.int64).reshape(-1, 2))
        h = lib().gsro_graph_from_edges(C.c_longlong(n), C.c_longlong(uv.shape[0]), _p(uv), int(norm))
        if not h:
            raise OracleError(1, lib().gsro_last_error().decode())
        self = cls.__new__(cls)
        self.h = C.c_void_p(h)
        self.n = n
        self.e = int(lib().gsro_graph_e(self.h))
        self.norm = norm
        return self

    def csr(self):
        rp = np.zeros(self.n + 1, np.int64)
        ci = np.zeros(self.e, np.int32)
        lib().gsro_graph_csr(self.h, _p(rp), _p(ci))
        return rp, ci

    def csc(self):
        rp = np.zeros(self.n + 1, np.int64)
        ci = np.zeros(self.e, np.int32)
        lib().gsro_graph_csc(self.h, _p(rp), _p(ci))
        return rp, ci

    def __del__(self):
        try:
            lib().gsro_graph_destroy(self.h)
        except Exception:
            pass


def gs_topk(x, k):
    x = np.ascontiguousarray(x)
    n, w = x.shape
    vals = np.zeros((n, k), x.dtype)
    idx = np.zeros((n, k), np.int32)
    _chk(getattr(lib(), "gsro_gs_topk_" + _sfx(x.dtype))(C.c_longlong(n), w, k, _p(x), C.c_longlong(w), _p(vals), _p(idx)))
    return vals, idx


def scatter(vals, idx, width):
    vals = np.ascontiguousarray(vals)
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    n, k = vals.shape
    out = np.zeros((n, width), vals.dtype)
    _chk(getattr(lib(), "gsro_scatter_" + _sfx(vals.dtype))(C.c_longlong(n), width, k, _p(vals), _p(idx), _p(out), C.c_longlong(width)))
    return out


def gather(x, idx):
    x = np.ascontiguousarray(x)
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    n, w = x.shape
    k = idx.shape[1]
    vals = np.zeros((n, k), x.dtype)
    _chk(getattr(lib(), "gsro_gather_" + _sfx(x.dtype))(C.c_longlong(n), w, k, _p(x), C.c_longlong(w), _p(idx), _p(vals)))
    return vals


def spmm(g, x, transpose=False):
    x = np.ascontiguousarray(x)
    n, cols = x.shape
    y = np.zeros_like(x)
    _chk(getattr(lib(), "gsro_spmm_" + _sfx(x.dtype))(g.h, int(transpose), cols, _p(x), C.c_longlong(cols), _p(y), C.c_longlong(cols)))
    return y


def spmm_sparse(g, vals, idx, width, transpose=False):
    vals = np.ascontiguousarray(vals)
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    n, k = vals.shape
    y = np.zeros((n, width), vals.dtype)
    _chk(getattr(lib(), "gsro_spmm_sparse_" + _sfx(vals.dtype))(g.h, int(transpose), width, k, _p(vals), _p(idx), _p(y), C.c_longlong(width)))
    return y


def gemm(a, b, bt=False, out=None):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b, dtype=a.dtype)
    M, K = a.shape
    N = b.shape[0] if bt else b.shape[1]
    acc = out is not None
    if out is None:
        out = np.zeros((M, N), a.dtype)
    _chk(getattr(lib(), "gsro_gemm_" + _sfx(a.dtype))(C.c_longlong(M), K, N, _p(a), C.c_longlong(K), _p(b), C.c_longlong(b.shape[1]), int(bt), int(acc), _p(out), C.c_longlong(N)))
    return out


def block_fwd(g, vals, idx, W, b=None, width=None, use_weight=True, use_bias=False, epi=EPI_NONE, R=None, rvals=None, ridx=None):
    vals = np.ascontiguousarray(vals)
    dt = vals.dtype
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    n, k = vals.shape
    w = width if width is not None else W.shape[0]
    W = np.ascontiguousarray(W if W is not None else np.zeros((w, w)), dtype=dt)
    b = np.ascontiguousarray(b if b is not None else np.zeros(w), dtype=dt)
    out = np.zeros((n, w), dt)
    Rr = np.ascontiguousarray(R, dtype=dt) if R is not None else None
    rv = np.ascontiguousarray(rvals, dtype=dt) if rvals is not None else None
    ri = np.ascontiguousarray(ridx, dtype=np.int32) if ridx is not None else None
    _chk(getattr(lib(), "gsro_block_fwd_" + _sfx(dt))(g.h, w, k, _p(vals), _p(idx), _p(W), _p(b), int(use_weight), int(use_bias), int(epi),
                                                      _p(Rr), C.c_longlong(w), _p(rv), _p(ri), _p(out), C.c_longlong(w)))
    return out


def dense_block(g, x, W=None, b=None, use_weight=True, use_bias=False):
    x = np.ascontiguousarray(x)
    dt = x.dtype
    n, w = x.shape
    W = np.ascontiguousarray(W if W is not None else np.zeros((w, w)), dtype=dt)
    b = np.ascontiguousarray(b if b is not None else np.zeros(w), dtype=dt)
    out = np.zeros((n, w), dt)
    _chk(getattr(lib(), "gsro_dense_block_" + _sfx(dt))(g.h, w, _p(x), C.c_longlong(w), _p(W), _p(b), int(use_weight), int(use_bias), _p(out), C.c_longlong(w)))
    return out


def block_bwd(g, m, isrc, fvals, fidx, W, use_weight=True, use_bias=False, dW=None, db=None):
    m = np.ascontiguousarray(m)
    dt = m.dtype
    n, w = m.shape
    k = isrc.shape[1]
    isrc = np.ascontiguousarray(isrc, dtype=np.int32)
    fvals = np.ascontiguousarray(fvals, dtype=dt)
    fidx = np.ascontiguousarray(fidx, dtype=np.int32)
    W = np.ascontiguousarray(W, dtype=dt)
    dW = np.zeros((w, w), dt) if dW is None else dW
    db = np.zeros(w, dt) if db is None else db
    out = np.zeros((n, w), dt)
    _chk(getattr(lib(), "gsro_block_bwd_" + _sfx(dt))(g.h, w, k, _p(m), C.c_longlong(w), _p(isrc), _p(fvals), _p(fidx), _p(W), int(use_weight), int(use_bias),
                                                      _p(out), C.c_longlong(w), _p(dW), _p(db)))
    return out, dW, db


def mse(yhat, y, mask):
    yhat = np.ascontiguousarray(yhat)
    y = np.ascontiguousarray(y, dtype=yhat.dtype)
    mask = np.ascontiguousarray(mask, dtype=np.uint8)
    gy = np.zeros_like(yhat)
    loss = getattr(lib(), "gsro_mse_" + _sfx(yhat.dtype))(C.c_longlong(yhat.size), _p(yhat), _p(y), _p(mask), _p(gy))
    if loss < 0:
        raise OracleError(1, lib().gsro_last_error().decode())
    return loss, gy


def adam(p, g, m, v, t, lr=1e-3, b1=0.9, b2=0.999, eps=1e-8, wd=0.0):
    """In-place bias-corrected Adam step number t (1-based)."""
    dt = p.dtype
    ct = C.c_double if dt == np.float64 else C.c_float
    bc1 = 1.0 - b1 ** t
    bc2 = 1.0 - b2 ** t
    getattr(lib(), "gsro_adam_" + _sfx(dt))(C.c_longlong(p.size), _p(p), _p(g), _p(m), _p(v), ct(lr), ct(b1), ct(b2), ct(eps), ct(wd), ct(bc1), ct(bc2))


class Net:
    """GSR / GSR-C / rev-baseline network."""

    # the device's default residual-stream grid (gsrc_set_residual_quant): f32
    # nets in the grouped-reversible modes match it unless told otherwise; f64
    # verification nets (finite differences) keep plain adds
    DEVICE_QSHIFT = 20

    def __init__(self, g, mode, L, D, C_groups, k, d_in, use_weight=True, use_bias=False, index_source=0, dtype=np.float32, qshift=None):
        self.g = g
        self.dtype = np.dtype(dtype)
        self.sfx = _sfx(dtype)
        h = getattr(lib(), "gsro_net_create_" + self.sfx)(g.h, mode, L, D, C_groups, k, d_in, int(use_weight), int(use_bias), int(index_source))
        if not h:
            raise OracleError(1, lib().gsro_last_error().decode())
        self.h = C.c_void_p(h)
        self.mode, self.L, self.D, self.C, self.k, self.d_in = mode, L, D, C_groups, k, d_in
        self.n = g.n
        self.P = int(lib().gsro_net_num_params(self.h))
        if qshift is None:
            qshift = self.DEVICE_QSHIFT if (self.dtype == np.float32 and mode != MODE_ALG12) else 0
        self.set_quant(qshift)

    def set_quant(self, shift):
        """Residual-stream grid 2^-shift (exactly invertible layers); 0 = plain adds."""
        _chk(lib().gsro_net_set_quant(self.h, int(shift)))
        self.qshift = int(shift)

    def _f(self, name):
        return getattr(lib(), f"gsro_net_{name}_{self.sfx}")

    def set_params(self, p):
        p = np.ascontiguousarray(p, dtype=self.dtype)
        assert p.size == self.P
        _chk(self._f("set_params")(self.h, _p(p)))

    def params(self):
        p = np.zeros(self.P, self.dtype)
        _chk(self._f("get_params")(self.h, _p(p)))
        return p

    def grads(self):
        p = np.zeros(self.P, self.dtype)
        _chk(self._f("get_grads")(self.h, _p(p)))
        return p

    def zero_grads(self):
        _chk(self._f("zero_grads")(self.h))

    def forward(self, X0):
        X0 = np.ascontiguousarray(X0, dtype=self.dtype)
        X = np.zeros((self.n, self.D), self.dtype)
        yhat = np.zeros(self.n, self.dtype)
        _chk(self._f("forward")(self.h, _p(X0), _p(X), _p(yhat)))
        return yhat, X

    def loss_grads(self, X0, y, mask):
        X0 = np.ascontiguousarray(X0, dtype=self.dtype)
        y = np.ascontiguousarray(y, dtype=self.dtype)
        mask = np.ascontiguousarray(mask, dtype=np.uint8)
        X = np.zeros((self.n, self.D), self.dtype)
        yhat = np.zeros(self.n, self.dtype)
        loss = C.c_double(0)
        _chk(self._f("loss_grads")(self.h, _p(X0), _p(y), _p(mask), C.byref(loss), _p(yhat), _p(X)))
        return loss.value, self.grads(), yhat, X

    def layer_forward(self, l, X):
        X = np.ascontiguousarray(X, dtype=self.dtype).copy()
        _chk(self._f("layer_forward")(self.h, l, _p(X)))
        return X

    def layer_inverse(self, l, Y):
        Y = np.ascontiguousarray(Y, dtype=self.dtype).copy()
        _chk(self._f("layer_inverse")(self.h, l, _p(Y)))
        return Y

    def layer_backward(self, l, Y, G):
        Y = np.ascontiguousarray(Y, dtype=self.dtype).copy()
        G = np.ascontiguousarray(G, dtype=self.dtype).copy()
        _chk(self._f("layer_backward")(self.h, l, _p(Y), _p(G)))
        return Y, G

    def transcribe_forward(self, l, X):
        X = np.ascontiguousarray(X, dtype=self.dtype).copy()
        _chk(self._f("transcribe_forward")(self.h, l, _p(X)))
        return X

    def transcribe_backward(self, l, G):
        G = np.ascontiguousarray(G, dtype=self.dtype).copy()
        _chk(self._f("transcribe_backward")(self.h, l, _p(G)))
        return G

    def __del__(self):
        try:
            lib().gsro_net_destroy(self.h)
        except Exception:
            pass
