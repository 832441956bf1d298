"""ctypes binding of the C-ABI (include/gsr_cuda.h) — the Python host mirror.

Loads the in-tree libgsrcuda.so (built by paper_2603_27156_b200/build.py for
sm_100a). There is no fallback: if the library is missing or no CUDA device is
present, every entry point raises.

Error behaviour mirrors /root/reference/proj/include/gsr/common.hpp:13-35:
status 1 → ConfigError, 3 → ResourceError, 4 → SequencingError.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GSRC_LIB") or os.path.join(_HERE, "libgsrcuda.so")  # GSRC_LIB: an alternate build (A/B timing)

MODE_ALG12, MODE_GSRC, MODE_REV = 0, 1, 2
NORM_NONE, NORM_ROW_MEAN, NORM_SYM_DEGREE = 0, 1, 2
GEMM_FP32, GEMM_TF32 = 0, 1
EPI_NONE, EPI_ADD, EPI_SUB, EPI_SCATTER_ADD, EPI_SCATTER_SUB = range(5)


class GsrError(RuntimeError):
    code = 2


class ConfigError(GsrError):      # ConfigError / ShapeError / FormatError (common.hpp:14-25)
    code = 1


class ResourceError(GsrError):    # common.hpp:32-35
    code = 3


class SequencingError(GsrError):  # common.hpp:27-30
    code = 4


_ERRS = {1: ConfigError, 2: GsrError, 3: ResourceError, 4: SequencingError}


class ModelCfg(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("mode", "layers", "hidden", "groups", "k", "d_in", "use_weight", "use_bias",
                                       "index_source", "gemm")]


class OptimCfg(C.Structure):
    _fields_ = [("optimizer", C.c_int), ("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float),
                ("weight_decay", C.c_float), ("momentum", C.c_float)]


class MemReport(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("reserved_bytes", "active_bytes", "peak_reserved_bytes", "peak_active_bytes",
                                          "alloc_count", "reuse_count", "release_count")] + [("utilization", C.c_double)]


class Timing(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("t_forward", "t_backward", "t_copy", "t_optimizer", "t_total")]


# Every exported symbol of include/gsr_cuda.h (checked by tests/test_capi_symbols.py).
EXPORTS = [
    "gsrc_create", "gsrc_destroy", "gsrc_last_error", "gsrc_set_stream", "gsrc_synchronize", "gsrc_version",
    "gsrc_graph_upload", "gsrc_model_init", "gsrc_num_params", "gsrc_params_set", "gsrc_params_get", "gsrc_grads_get",
    "gsrc_zero_grads", "gsrc_grads_device", "gsrc_params_device", "gsrc_data_upload", "gsrc_forward", "gsrc_forward_backward",
    "gsrc_optimizer_step", "gsrc_train_step", "gsrc_activation_get", "gsrc_activation_set", "gsrc_gradient_get",
    "gsrc_gradient_set", "gsrc_set_graph_capture", "gsrc_last_timing", "gsrc_mem_stats", "gsrc_high_water_reset",
    "gsrc_kernel_launches", "gsrc_work_counter", "gsrc_work_reset", "gsrc_profile_kernels", "gsrc_layer_forward", "gsrc_layer_inverse", "gsrc_layer_backward", "gsrc_op_gs_topk",
    "gsrc_set_op_precision", "gsrc_op_spmm", "gsrc_op_spmm_sparse", "gsrc_op_block_forward", "gsrc_op_dense_block", "gsrc_op_block_backward",
    "gsrc_get_stream", "gsrc_optim_state_get", "gsrc_optim_state_set", "gsrc_comm_unique_id", "gsrc_comm_init",
    "gsrc_comm_allreduce_grads", "gsrc_comm_destroy", "gsrc_diag_masks", "gsrc_diag_mask_flips", "gsrc_set_residual_quant",
    "gsrc_get_residual_quant",
]

_lib = None


def lib():
    """Load libgsrcuda.so (raises if it was not built — no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        vp, i64, i32, f32p = C.c_void_p, C.c_int64, C.c_int, C.c_void_p
        L.gsrc_last_error.restype = C.c_char_p
        L.gsrc_last_error.argtypes = [vp]
        L.gsrc_destroy.restype = None
        L.gsrc_destroy.argtypes = [vp]
        L.gsrc_create.argtypes = [i32, C.POINTER(vp)]
        L.gsrc_graph_upload.argtypes = [vp, i64, i64, vp, vp, i32]
        L.gsrc_model_init.argtypes = [vp, C.POINTER(ModelCfg)]
        L.gsrc_num_params.argtypes = [vp, C.POINTER(i64)]
        for nm in ("gsrc_params_set", "gsrc_params_get", "gsrc_grads_get"):
            getattr(L, nm).argtypes = [vp, f32p, i64]
        L.gsrc_grads_device.argtypes = [vp, C.POINTER(vp), C.POINTER(i64)]
        L.gsrc_params_device.argtypes = [vp, C.POINTER(vp), C.POINTER(i64)]
        L.gsrc_data_upload.argtypes = [vp, vp, vp, vp]
        L.gsrc_forward.argtypes = [vp, vp]
        L.gsrc_forward_backward.argtypes = [vp, C.POINTER(C.c_double)]
        L.gsrc_optimizer_step.argtypes = [vp, C.POINTER(OptimCfg)]
        L.gsrc_train_step.argtypes = [vp, C.POINTER(OptimCfg), C.POINTER(C.c_double)]
        for nm in ("gsrc_activation_get", "gsrc_activation_set", "gsrc_gradient_get", "gsrc_gradient_set"):
            getattr(L, nm).argtypes = [vp, vp]
        L.gsrc_set_graph_capture.argtypes = [vp, i32]
        L.gsrc_set_stream.argtypes = [vp, vp]
        L.gsrc_last_timing.argtypes = [vp, C.POINTER(Timing)]
        L.gsrc_mem_stats.argtypes = [vp, C.POINTER(MemReport)]
        L.gsrc_kernel_launches.argtypes = [vp, C.POINTER(i64)]
        L.gsrc_work_counter.argtypes = [vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.gsrc_work_reset.argtypes = [vp]
        L.gsrc_profile_kernels.argtypes = [vp, i32, vp]
        for nm in ("gsrc_layer_forward", "gsrc_layer_inverse", "gsrc_layer_backward"):
            getattr(L, nm).argtypes = [vp, i32]
        L.gsrc_op_gs_topk.argtypes = [vp, i64, i32, i32, vp, vp, vp]
        L.gsrc_set_op_precision.argtypes = [vp, i32]
        L.gsrc_op_spmm.argtypes = [vp, i32, i32, vp, vp]
        L.gsrc_op_spmm_sparse.argtypes = [vp, i32, i32, i32, vp, vp, vp]
        L.gsrc_op_block_forward.argtypes = [vp, i32, i32, vp, vp, vp, vp, i32, i32, i32, vp, vp, vp, vp, i32, vp, vp]
        L.gsrc_op_dense_block.argtypes = [vp, i32, vp, vp, vp, i32, i32, vp]
        L.gsrc_op_block_backward.argtypes = [vp, i32, i32, vp, vp, vp, vp, vp, i32, i32, vp, vp, vp]
        L.gsrc_version.argtypes = [C.c_char_p, C.c_size_t]
        L.gsrc_get_stream.argtypes = [vp, C.POINTER(vp)]
        L.gsrc_optim_state_get.argtypes = [vp, vp, vp, C.POINTER(i64), i64]
        L.gsrc_optim_state_set.argtypes = [vp, vp, vp, i64, i64]
        L.gsrc_comm_unique_id.argtypes = [vp, C.c_size_t]
        L.gsrc_comm_init.argtypes = [vp, vp, i32, i32]
        L.gsrc_comm_allreduce_grads.argtypes = [vp]
        L.gsrc_comm_destroy.argtypes = [vp]
        L.gsrc_diag_masks.argtypes = [vp, i32, i32]
        L.gsrc_diag_mask_flips.argtypes = [vp, vp, C.POINTER(i64)]
        L.gsrc_set_residual_quant.argtypes = [vp, i32]
        L.gsrc_get_residual_quant.argtypes = [vp, C.POINTER(i32)]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f32(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float32)
    if shape is not None:
        a = a.reshape(shape)
    return a


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


class Context:
    """One device, one stream, one arena (SURVEY.md §8b 'Ownership'/'Threading')."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        st = lib().gsrc_create(int(device), C.byref(h))
        if st != 0:
            raise _ERRS.get(st, GsrError)(f"gsrc_create failed with status {st} (no CUDA device?)")
        self.h = h
        self.device = int(device)
        self.n = 0
        self.cfg = None
        self.P = 0

    def close(self):
        if getattr(self, "h", None):
            lib().gsrc_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _chk(self, st):
        if st != 0:
            raise _ERRS.get(st, GsrError)(lib().gsrc_last_error(self.h).decode())

    # ---- setup ---------------------------------------------------------------
    def set_stream(self, stream_ptr: int | None):
        """Bind to a caller's stream; None = the context-owned stream. Handle 0
        (the legacy default stream) is rejected: the C-ABI reads NULL as "own
        stream", which would silently lose the ordering the caller asked for."""
        if stream_ptr == 0:
            raise ConfigError("set_stream(0): the legacy default stream cannot be bound; use a torch.cuda.Stream "
                              "or None (context-owned stream, see stream_ptr())")
        self._chk(lib().gsrc_set_stream(self.h, C.c_void_p(stream_ptr)))

    def stream_ptr(self) -> int:
        """cudaStream_t every call enqueues on (wrap with torch.cuda.ExternalStream to order torch work with it)."""
        s = C.c_void_p()
        self._chk(lib().gsrc_get_stream(self.h, C.byref(s)))
        return s.value or 0

    def graph_upload(self, row_ptr, col_idx, norm=NORM_ROW_MEAN):
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        ci = _i32(col_idx)
        self._chk(lib().gsrc_graph_upload(self.h, rp.size - 1, ci.size, _p(rp), _p(ci), int(norm)))
        self.n = rp.size - 1

    def model_init(self, mode, layers, hidden, groups, k, d_in, use_weight=True, use_bias=False, index_source=0, gemm=GEMM_FP32):
        cfg = ModelCfg(int(mode), int(layers), int(hidden), int(groups), int(k), int(d_in), int(use_weight), int(use_bias),
                       int(index_source), int(gemm))
        self._chk(lib().gsrc_model_init(self.h, C.byref(cfg)))
        P = C.c_int64()
        self._chk(lib().gsrc_num_params(self.h, C.byref(P)))
        self.P = P.value
        self.cfg = dict(mode=mode, layers=layers, hidden=hidden, groups=2 if mode == MODE_ALG12 else groups, k=k, d_in=d_in,
                        use_weight=use_weight, use_bias=use_bias, index_source=index_source, gemm=gemm)

    def set_params(self, p):
        p = _f32(p)
        self._chk(lib().gsrc_params_set(self.h, _p(p), p.size))

    def params(self):
        p = np.zeros(self.P, np.float32)
        self._chk(lib().gsrc_params_get(self.h, _p(p), p.size))
        return p

    def grads(self):
        g = np.zeros(self.P, np.float32)
        self._chk(lib().gsrc_grads_get(self.h, _p(g), g.size))
        return g

    def zero_grads(self):
        self._chk(lib().gsrc_zero_grads(self.h))

    def grads_device(self):
        p, n = C.c_void_p(), C.c_int64()
        self._chk(lib().gsrc_grads_device(self.h, C.byref(p), C.byref(n)))
        return p.value, n.value

    def grads_tensor(self):
        """torch view (no copy) of the flat device gradient buffer, for the DP all-reduce."""
        from .dp import device_grads_tensor
        return device_grads_tensor(self, self.device)

    def params_device(self):
        p, n = C.c_void_p(), C.c_int64()
        self._chk(lib().gsrc_params_device(self.h, C.byref(p), C.byref(n)))
        return p.value, n.value

    def data_upload(self, x0, y, mask):
        """Host arrays (numpy, or raw pointers for pinned buffers)."""
        if isinstance(x0, int):
            self._chk(lib().gsrc_data_upload(self.h, C.c_void_p(x0), C.c_void_p(y), C.c_void_p(mask)))
            return
        x0 = _f32(x0)
        y = _f32(y)
        m = np.ascontiguousarray(mask, dtype=np.uint8)
        self._chk(lib().gsrc_data_upload(self.h, _p(x0), _p(y), _p(m)))

    # ---- step ------------------------------------------------------------------
    def forward(self):
        yh = np.zeros(self.n, np.float32)
        self._chk(lib().gsrc_forward(self.h, _p(yh)))
        return yh

    def forward_backward(self):
        loss = C.c_double()
        self._chk(lib().gsrc_forward_backward(self.h, C.byref(loss)))
        return loss.value

    def optimizer_step(self, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0, optimizer=0, momentum=0.0):
        o = OptimCfg(int(optimizer), lr, beta1, beta2, eps, weight_decay, momentum)
        self._chk(lib().gsrc_optimizer_step(self.h, C.byref(o)))

    def train_step(self, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0, optimizer=0, momentum=0.0):
        o = OptimCfg(int(optimizer), lr, beta1, beta2, eps, weight_decay, momentum)
        loss = C.c_double()
        self._chk(lib().gsrc_train_step(self.h, C.byref(o), C.byref(loss)))
        return loss.value

    def set_graph_capture(self, enable=True):
        self._chk(lib().gsrc_set_graph_capture(self.h, int(enable)))

    def activation(self):
        X = np.zeros((self.n, self.cfg["hidden"]), np.float32)
        self._chk(lib().gsrc_activation_get(self.h, _p(X)))
        return X

    def set_activation(self, X):
        X = _f32(X)
        self._chk(lib().gsrc_activation_set(self.h, _p(X)))

    def gradient(self):
        G = np.zeros((self.n, self.cfg["hidden"]), np.float32)
        self._chk(lib().gsrc_gradient_get(self.h, _p(G)))
        return G

    def set_gradient(self, G):
        G = _f32(G)
        self._chk(lib().gsrc_gradient_set(self.h, _p(G)))

    def layer_forward(self, l):
        self._chk(lib().gsrc_layer_forward(self.h, int(l)))

    def layer_inverse(self, l):
        self._chk(lib().gsrc_layer_inverse(self.h, int(l)))

    def layer_backward(self, l):
        self._chk(lib().gsrc_layer_backward(self.h, int(l)))

    def last_timing(self):
        t = Timing()
        self._chk(lib().gsrc_last_timing(self.h, C.byref(t)))
        return {f: getattr(t, f) for f, _ in Timing._fields_}

    def mem_stats(self):
        m = MemReport()
        self._chk(lib().gsrc_mem_stats(self.h, C.byref(m)))
        return {f: getattr(m, f) for f, _ in MemReport._fields_}

    def high_water_reset(self):
        self._chk(lib().gsrc_high_water_reset(self.h))

    def work_counter(self):
        """WorkCounter: (scalar_mul_adds, rows_touched) since create / work_reset()."""
        ma, rows = C.c_uint64(), C.c_uint64()
        self._chk(lib().gsrc_work_counter(self.h, C.byref(ma), C.byref(rows)))
        return ma.value, rows.value

    def work_reset(self):
        self._chk(lib().gsrc_work_reset(self.h))

    def kernel_launches(self):
        n = C.c_int64()
        self._chk(lib().gsrc_kernel_launches(self.h, C.byref(n)))
        return n.value

    KERNEL_CLASSES = ("fused_block_fwd", "block_bwd_recompute", "block_bwd_input", "gs_groupsum")

    def profile_kernels(self, reps=20):
        """Live CUDA-event timing of each kernel class over all C blocks (device state preserved)."""
        Cg = self.cfg["groups"]
        out = np.zeros(16 + 3 * Cg, np.float64)
        self._chk(lib().gsrc_profile_kernels(self.h, int(reps), _p(out)))
        res = {}
        for c, name in enumerate(self.KERNEL_CLASSES):
            ms, byts, per_step, flops = out[4 * c:4 * c + 4]
            res[name] = dict(ms=float(ms), bytes=float(byts), launches_per_step=float(per_step), flops=float(flops))
            if c < 3:
                res[name]["ms_per_block"] = [float(x) for x in out[16 + c * Cg:16 + (c + 1) * Cg]]
        return res

    # ---- optimizer state / data parallelism / diagnostics -------------------------
    def optim_state(self):
        m = np.zeros(self.P, np.float32)
        v = np.zeros(self.P, np.float32)
        t = C.c_int64()
        self._chk(lib().gsrc_optim_state_get(self.h, _p(m), _p(v), C.byref(t), self.P))
        return m, v, t.value

    def set_optim_state(self, m, v, step):
        m, v = _f32(m), _f32(v)
        self._chk(lib().gsrc_optim_state_set(self.h, _p(m), _p(v), int(step), self.P))

    @staticmethod
    def comm_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        st = lib().gsrc_comm_unique_id(buf, 128)
        if st != 0:
            raise _ERRS.get(st, GsrError)("gsrc_comm_unique_id failed (NCCL unavailable?)")
        return buf.raw

    def comm_init(self, unique_id: bytes, nranks: int, rank: int):
        buf = C.create_string_buffer(bytes(unique_id), 128)
        self._chk(lib().gsrc_comm_init(self.h, buf, int(nranks), int(rank)))

    def comm_allreduce_grads(self):
        self._chk(lib().gsrc_comm_allreduce_grads(self.h))

    def comm_destroy(self):
        self._chk(lib().gsrc_comm_destroy(self.h))

    def set_residual_quant(self, shift: int):
        """Residual-stream grid 2^-shift (exactly invertible layers; 0 = plain fp32 adds)."""
        self._chk(lib().gsrc_set_residual_quant(self.h, int(shift)))

    def residual_quant(self) -> int:
        s = C.c_int()
        self._chk(lib().gsrc_get_residual_quant(self.h, C.byref(s)))
        return s.value

    def diag_masks(self, enable=True, row_stride=1):
        self._chk(lib().gsrc_diag_masks(self.h, int(enable), int(row_stride)))

    def mask_flips(self):
        """(layers × groups) counts of sampled rows whose backward-recomputed GS mask differs from the forward's, and the sample size."""
        L, Cg = self.cfg["layers"], self.cfg["groups"]
        f = np.zeros(L * Cg, np.int64)
        rows = C.c_int64()
        self._chk(lib().gsrc_diag_mask_flips(self.h, _p(f), C.byref(rows)))
        return f.reshape(L, Cg), rows.value

    # ---- op-level parity entry points (SPEC op names) ----------------------------
    def set_op_precision(self, gemm):
        self._chk(lib().gsrc_set_op_precision(self.h, int(gemm)))

    def gs_topk(self, x, k):
        x = _f32(x)
        n, w = x.shape
        vals = np.zeros((n, k), np.float32)
        idx = np.zeros((n, k), np.int32)
        self._chk(lib().gsrc_op_gs_topk(self.h, n, w, int(k), _p(x), _p(vals), _p(idx)))
        return vals, idx

    def spmm(self, x, transpose=False):
        x = _f32(x)
        y = np.zeros_like(x)
        self._chk(lib().gsrc_op_spmm(self.h, int(transpose), x.shape[1], _p(x), _p(y)))
        return y

    def spmm_sparse(self, vals, idx, width, transpose=False):
        vals = _f32(vals)
        idx = _i32(idx)
        y = np.zeros((vals.shape[0], width), np.float32)
        self._chk(lib().gsrc_op_spmm_sparse(self.h, int(transpose), int(width), vals.shape[1], _p(vals), _p(idx), _p(y)))
        return y

    def block_forward(self, vals, idx, W=None, b=None, width=None, use_weight=True, use_bias=False, epi=EPI_NONE, R=None,
                      rvals=None, ridx=None, gs_k=0):
        vals = _f32(vals)
        idx = _i32(idx)
        n, k = vals.shape
        w = width if width is not None else W.shape[0]
        W = _f32(W) if W is not None else None
        b = _f32(b) if b is not None else None
        R = _f32(R) if R is not None else None
        rv = _f32(rvals) if rvals is not None else None
        ri = _i32(ridx) if ridx is not None else None
        out = np.zeros((n, w), np.float32)
        gv = np.zeros((n, max(gs_k, 1)), np.float32)
        gi = np.zeros((n, max(gs_k, 1)), np.int32)
        self._chk(lib().gsrc_op_block_forward(self.h, int(w), int(k), _p(vals), _p(idx), _p(W), _p(b), int(use_weight), int(use_bias),
                                              int(epi), _p(R), _p(rv), _p(ri), _p(out), int(gs_k), _p(gv), _p(gi)))
        if gs_k:
            return out, gv, gi
        return out

    def dense_block(self, x, W=None, b=None, use_weight=True, use_bias=False):
        x = _f32(x)
        n, w = x.shape
        out = np.zeros((n, w), np.float32)
        self._chk(lib().gsrc_op_dense_block(self.h, int(w), _p(x), _p(_f32(W) if W is not None else None),
                                            _p(_f32(b) if b is not None else None), int(use_weight), int(use_bias), _p(out)))
        return out

    def block_backward(self, m, isrc, fvals, fidx, W, use_weight=True, use_bias=False):
        m = _f32(m)
        n, w = m.shape
        k = isrc.shape[1]
        out = np.zeros((n, w), np.float32)
        dW = np.zeros((w, w), np.float32)
        db = np.zeros(w, np.float32)
        self._chk(lib().gsrc_op_block_backward(self.h, int(w), int(k), _p(m), _p(_i32(isrc)), _p(_f32(fvals)), _p(_i32(fidx)),
                                               _p(_f32(W)), int(use_weight), int(use_bias), _p(out), _p(dW), _p(db)))
        return out, dW, db


def version():
    buf = C.create_string_buffer(64)
    lib().gsrc_version(buf, 64)
    return buf.value.decode()
