"""ctypes binding of libsppo.so (include/sppo.h) — argument marshalling only.

Every compute step runs in the CUDA kernels behind the C ABI; this module turns
torch tensors into device pointers, Python lists into C arrays and non-OK
statuses into exceptions.  It never computes anything itself and there is no
fallback: if the native library is missing, importing it raises.

Names follow the C ABI: sppo_attn_fwd -> Context.attn_fwd, etc.
"""

from __future__ import annotations

import ctypes as C
import math
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsppo.so")

SPPO_BF16, SPPO_FP32 = 0, 1
SPPO_FIRST, SPPO_LAST = 1, 2
SPPO_COPY_NO_ORDER, SPPO_COPY_DEFER_WAIT = 1, 2

STATUS = {0: "SPPO_OK", 1: "SPPO_E_ARG", 2: "SPPO_E_SHAPE", 3: "SPPO_E_ALIGN", 4: "SPPO_E_STATE",
          5: "SPPO_E_NOT_RESIDENT", 6: "SPPO_E_OOM", 7: "SPPO_E_CUDA", 8: "SPPO_E_UNSUPPORTED"}

# every symbol include/sppo.h declares
EXPORTS = ("sppo_ctx_create", "sppo_ctx_destroy", "sppo_ctx_sync", "sppo_last_error", "sppo_version",
           "sppo_attn_fwd", "sppo_attn_fwd_chunks", "sppo_attn_bwd", "sppo_host_alloc", "sppo_host_free", "sppo_kv_offload",
           "sppo_kv_prefetch", "sppo_partition_equal", "sppo_partition_balanced", "sppo_partition_balanced_lin", "sppo_causal_pairs",
           "sppo_offload_alpha",
           "sppo_finalize", "sppo_ctx_streams", "sppo_ctx_numa_node")
# every symbol include/sppo_layer.h declares (per-chunk transformer layer)
LAYER_EXPORTS = ("sppo_gemm", "sppo_layernorm_fwd", "sppo_layernorm_bwd", "sppo_col_reduce")
# every symbol include/sppo_pipeline.h declares (subsequence pipeline plan)
PIPELINE_EXPORTS = ("sppo_msp_phases", "sppo_pipeline_bubble", "sppo_pipeline_makespan")
SPPO_MSP_LEFT, SPPO_MSP_STEADY, SPPO_MSP_RIGHT = 0, 1, 2
SPPO_EPI_STORE, SPPO_EPI_GELU, SPPO_EPI_DGELU, SPPO_EPI_ACC_F32 = 0, 1, 2, 3


class SppoError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


class _Layout(C.Structure):
    _fields_ = [("heads", C.c_int32), ("head_dim", C.c_int32), ("dtype", C.c_int32), ("num_chunks", C.c_int32),
                ("offsets", C.POINTER(C.c_int64)), ("scale", C.c_float)]


class _KvSet(C.Structure):
    _fields_ = [("n", C.c_int32), ("ids", C.POINTER(C.c_int32)), ("k", C.POINTER(C.c_void_p)),
                ("v", C.POINTER(C.c_void_p))]


class _FwdState(C.Structure):
    _fields_ = [("o_acc", C.c_void_p), ("m", C.c_void_p), ("l", C.c_void_p)]


class _BwdArgs(C.Structure):
    _fields_ = [("o", C.c_void_p), ("lse", C.c_void_p), ("dout", C.c_void_p), ("delta", C.c_void_p),
                ("dq_acc", C.c_void_p), ("dk_acc", C.POINTER(C.c_void_p)), ("dv_acc", C.POINTER(C.c_void_p)),
                ("dq", C.c_void_p), ("dk", C.c_void_p), ("dv", C.c_void_p)]


class _GemmArgs(C.Structure):
    _fields_ = [("M", C.c_int64), ("N", C.c_int64), ("K", C.c_int64), ("a_mn", C.c_int32), ("b_mn", C.c_int32),
                ("a_parts", C.c_int32), ("a", C.c_void_p * 3), ("b", C.c_void_p), ("epilogue", C.c_int32),
                ("bias", C.c_void_p), ("residual", C.c_void_p), ("aux_in", C.c_void_p), ("aux_out", C.c_void_p),
                ("c_parts", C.c_int32), ("c", C.c_void_p * 3)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run __graft_entry__.build() (no CPU fallback exists)")
    lib = C.CDLL(LIB_PATH)
    i32, vp, sz = C.c_int32, C.c_void_p, C.c_size_t
    sig = {
        "sppo_ctx_create": ([C.c_int, C.POINTER(vp)], i32),
        "sppo_ctx_destroy": ([vp], i32),
        "sppo_ctx_sync": ([vp], i32),
        "sppo_last_error": ([], C.c_char_p),
        "sppo_version": ([], i32),
        "sppo_attn_fwd": ([vp, C.POINTER(_Layout), i32, vp, C.POINTER(_KvSet), i32, C.POINTER(_FwdState), vp, vp, vp],
                          i32),
        "sppo_attn_fwd_chunks": ([vp, C.POINTER(_Layout), i32, i32, C.POINTER(vp), C.POINTER(_KvSet), C.POINTER(vp),
                                  C.POINTER(vp), vp], i32),
        "sppo_attn_bwd": ([vp, C.POINTER(_Layout), i32, vp, C.POINTER(_KvSet), C.POINTER(_BwdArgs), i32, vp], i32),
        "sppo_host_alloc": ([vp, sz, C.POINTER(vp)], i32),
        "sppo_host_free": ([vp, vp], i32),
        "sppo_kv_offload": ([vp, i32, vp, vp, sz, C.c_double, vp, vp, C.POINTER(sz)], i32),
        "sppo_kv_prefetch": ([vp, i32, vp, vp, sz, vp, vp, i32], i32),
        "sppo_partition_equal": ([C.c_int64, i32, C.POINTER(C.c_int64)], i32),
        "sppo_partition_balanced": ([C.c_int64, i32, C.POINTER(C.c_int64)], i32),
        "sppo_partition_balanced_lin": ([C.c_int64, i32, C.c_int64, C.POINTER(C.c_int64)], i32),
        "sppo_causal_pairs": ([C.POINTER(C.c_int64), i32, C.POINTER(C.c_int64)], i32),
        "sppo_offload_alpha": ([C.POINTER(C.c_double), C.POINTER(C.c_double), i32, C.c_double,
                                C.POINTER(C.c_double)], i32),
        "sppo_finalize": ([vp, vp, vp, sz, i32, vp], i32),
        "sppo_ctx_streams": ([vp, C.POINTER(vp), C.POINTER(vp)], i32),
        "sppo_ctx_numa_node": ([vp, C.POINTER(i32)], i32),
        "sppo_gemm": ([vp, C.POINTER(_GemmArgs), vp], i32),
        "sppo_msp_phases": ([i32, i32, i32, C.POINTER(C.c_int8), C.POINTER(i32), C.POINTER(i32)], i32),
        "sppo_pipeline_bubble": ([i32, i32, C.POINTER(C.c_double)], i32),
        "sppo_pipeline_makespan": ([i32, i32, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                    C.POINTER(C.c_double)], i32),
        "sppo_layernorm_fwd": ([vp, vp, vp, vp, C.c_int64, i32, C.c_float, vp, vp, vp, vp], i32),
        "sppo_layernorm_bwd": ([vp, vp, vp, vp, vp, vp, vp, C.c_int64, i32, vp, vp], i32),
        "sppo_col_reduce": ([vp, i32, C.POINTER(vp), vp, vp, vp, C.c_int64, i32, vp, vp, vp], i32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes, fn.restype = args, res
    return lib


_lib = _load()


def lib():
    return _lib


def _check(st: int):
    if st != 0:
        raise SppoError(st, _lib.sppo_last_error().decode(errors="replace"))


def _ptr(t):
    """Device/host pointer of a tensor (or int / None) — marshalling only."""
    if t is None:
        return None
    if isinstance(t, int):
        return t
    if not t.is_contiguous():
        raise ValueError("tensors passed to the C ABI must be contiguous")
    return t.data_ptr()


def _stream(s):
    if s is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(s, int):
        return s
    return s.cuda_stream


def _event(e):
    if e is None:
        return None
    if isinstance(e, int):
        return e
    if not e.cuda_event:  # torch creates the CUDA event lazily, on first record
        import torch
        e.record(torch.cuda.current_stream())
    return e.cuda_event


# ------------------------------------------------------------------ plan helpers
def partition_equal(S: int, N: int):
    out = (C.c_int64 * (N + 1))()
    _check(_lib.sppo_partition_equal(S, N, out))
    return list(out)


def partition_balanced(S: int, N: int, lin: int = 0):
    out = (C.c_int64 * (N + 1))()
    if lin:
        _check(_lib.sppo_partition_balanced_lin(S, N, int(lin), out))
    else:
        _check(_lib.sppo_partition_balanced(S, N, out))
    return list(out)


def causal_pairs(offsets) -> int:
    arr = (C.c_int64 * len(offsets))(*offsets)
    out = C.c_int64()
    _check(_lib.sppo_causal_pairs(arr, len(offsets) - 1, C.byref(out)))
    return out.value


def offload_alpha(A, m_threshold, last: float = 1.0):
    """m_threshold: scalar (the paper's constant M_threshold) or per-chunk list."""
    n = len(A)
    thr = list(m_threshold) if hasattr(m_threshold, "__len__") else [m_threshold] * n
    a = (C.c_double * n)(*A)
    m = (C.c_double * n)(*thr)
    out = (C.c_double * n)()
    _check(_lib.sppo_offload_alpha(a, m, n, last, out))
    return list(out)


def msp_phases(pp: int, n: int, stage: int):
    """sppo_msp_phases -> dict(left, steady, right ids; left_sp, right_sp stage lists)."""
    ph = (C.c_int8 * n)()
    ls, rs = (C.c_int32 * 2)(), (C.c_int32 * 2)()
    _check(_lib.sppo_msp_phases(pp, n, stage, ph, ls, rs))
    ids = {k: [x for x in range(n) if ph[x] == c] for k, c in (("left", 0), ("steady", 1), ("right", 2))}
    ids["left_sp"] = list(range(ls[0], ls[1] + 1))
    ids["right_sp"] = list(range(rs[0], rs[1] + 1))
    return ids


def pipeline_bubble(pp: int, n: int) -> float:
    out = C.c_double()
    _check(_lib.sppo_pipeline_bubble(pp, n, C.byref(out)))
    return out.value


def pipeline_makespan(pp: int, t_fwd, t_bwd) -> float:
    n = len(t_fwd)
    out = C.c_double()
    _check(_lib.sppo_pipeline_makespan(pp, n, (C.c_double * n)(*t_fwd), (C.c_double * n)(*t_bwd), C.byref(out)))
    return out.value


class Layout:
    """sppo_layout: heads on this device, head_dim, dtype, chunk offsets."""

    def __init__(self, heads: int, head_dim: int, offsets, dtype: int = SPPO_BF16, scale: float = 0.0):
        self.offsets = [int(x) for x in offsets]
        self._off = (C.c_int64 * len(self.offsets))(*self.offsets)
        self.c = _Layout(heads, head_dim, dtype, len(self.offsets) - 1, self._off, scale)
        self.heads, self.head_dim, self.dtype = heads, head_dim, dtype
        self.num_chunks = len(self.offsets) - 1
        self.scale = scale if scale else 1.0 / math.sqrt(head_dim)

    def chunk_len(self, i: int) -> int:
        return self.offsets[i + 1] - self.offsets[i]


def _kvset(ids, ks, vs):
    n = len(ids)
    kv = _KvSet(n, (C.c_int32 * n)(*ids), (C.c_void_p * n)(*[_ptr(k) for k in ks]),
                (C.c_void_p * n)(*[_ptr(v) for v in vs]))
    return kv


class Context:
    """sppo_ctx: one per (device, host thread)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _check(_lib.sppo_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device

    def close(self):
        if self.h:
            _check(_lib.sppo_ctx_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def sync(self):
        _check(_lib.sppo_ctx_sync(self.h))

    def copy_streams(self):
        """(d2h, h2d) cudaStream_t handles of the ctx (sppo_ctx_streams)."""
        a, b = C.c_void_p(), C.c_void_p()
        _check(_lib.sppo_ctx_streams(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def numa_node(self) -> int:
        """NUMA node of this ctx's GPU used by host_alloc (sppo_ctx_numa_node; -1 unknown)."""
        n = C.c_int32()
        _check(_lib.sppo_ctx_numa_node(self.h, C.byref(n)))
        return n.value

    # -------------------------------------------------------------- attention
    def attn_fwd(self, layout: Layout, chunk: int, q, kv_ids, ks, vs, flags=SPPO_FIRST | SPPO_LAST, state=None,
                 o=None, lse=None, stream=None):
        kv = _kvset(kv_ids, ks, vs)
        st = None
        if state is not None:
            st = _FwdState(_ptr(state[0]), _ptr(state[1]), _ptr(state[2]))
        _check(_lib.sppo_attn_fwd(self.h, C.byref(layout.c), chunk, _ptr(q), C.byref(kv), flags,
                                  C.byref(st) if st is not None else None, _ptr(o), _ptr(lse), _stream(stream)))

    def attn_fwd_chunks(self, layout: Layout, i0: int, i1: int, qs, ks, vs, os_, lses, stream=None):
        """sppo_attn_fwd_chunks: chunks i0..i1-1 in one launch (ks, vs: chunks 0..i1-1)."""
        n = i1 - i0
        kv = _kvset(list(range(len(ks))), ks, vs)  # the C side checks they are exactly 0..i1-1
        _check(_lib.sppo_attn_fwd_chunks(self.h, C.byref(layout.c), i0, i1,
                                         (C.c_void_p * n)(*[_ptr(t) for t in qs]), C.byref(kv),
                                         (C.c_void_p * n)(*[_ptr(t) for t in os_]),
                                         (C.c_void_p * n)(*[_ptr(t) for t in lses]), _stream(stream)))

    def attn_bwd(self, layout: Layout, chunk: int, q, kv_ids, ks, vs, o, lse, dout, delta, dq_acc, dk_accs,
                 dv_accs, dq=None, dk=None, dv=None, flags=SPPO_FIRST | SPPO_LAST, stream=None):
        kv = _kvset(kv_ids, ks, vs)
        n = len(kv_ids)
        args = _BwdArgs(_ptr(o), _ptr(lse), _ptr(dout), _ptr(delta), _ptr(dq_acc),
                        (C.c_void_p * n)(*[_ptr(t) for t in dk_accs]), (C.c_void_p * n)(*[_ptr(t) for t in dv_accs]),
                        _ptr(dq), _ptr(dk), _ptr(dv))
        _check(_lib.sppo_attn_bwd(self.h, C.byref(layout.c), chunk, _ptr(q), C.byref(kv), C.byref(args), flags,
                                  _stream(stream)))

    def finalize(self, src, dst, dtype: int = SPPO_BF16, stream=None):
        """a7: dst(dtype) = src(fp32) over src.numel() elements (sppo_finalize)."""
        _check(_lib.sppo_finalize(self.h, _ptr(src), _ptr(dst), src.numel(), dtype, _stream(stream)))

    # -------------------------------------------------------------- host arena / copies
    def host_alloc(self, nbytes: int) -> int:
        p = C.c_void_p()
        _check(_lib.sppo_host_alloc(self.h, nbytes, C.byref(p)))
        return p.value

    def host_free(self, ptr: int):
        _check(_lib.sppo_host_free(self.h, ptr))

    def kv_offload(self, chunk: int, dev, host: int, nbytes: int, alpha: float = 1.0, producer=None, done=None) -> int:
        copied = C.c_size_t()
        _check(_lib.sppo_kv_offload(self.h, chunk, _ptr(dev), host, nbytes, alpha, _stream(producer), _event(done),
                                    C.byref(copied)))
        return copied.value

    def kv_prefetch(self, chunk: int, host: int, dev, nbytes: int, consumer=None, done=None, flags: int = 0):
        _check(_lib.sppo_kv_prefetch(self.h, chunk, host, _ptr(dev), nbytes, _stream(consumer), _event(done), flags))

    # -------------------------------------------------------------- transformer layer (sppo_layer.h)
    def gemm(self, M: int, N: int, K: int, a, b, c, a_mn: int = 0, b_mn: int = 0, epilogue: int = SPPO_EPI_STORE,
             bias=None, residual=None, aux_in=None, aux_out=None, stream=None):
        """sppo_gemm.  ``a`` / ``c``: one tensor or a list of up to 3 (split along the contiguous dim)."""
        al = list(a) if isinstance(a, (list, tuple)) else [a]
        cl = list(c) if isinstance(c, (list, tuple)) else [c]
        g = _GemmArgs(M, N, K, a_mn, b_mn, len(al), (C.c_void_p * 3)(*[_ptr(t) for t in al]), _ptr(b), epilogue,
                      _ptr(bias), _ptr(residual), _ptr(aux_in), _ptr(aux_out), len(cl),
                      (C.c_void_p * 3)(*[_ptr(t) for t in cl]))
        _check(_lib.sppo_gemm(self.h, C.byref(g), _stream(stream)))

    def layernorm_fwd(self, x, gamma, beta, y, mean, rstd, eps: float = 1e-5, stream=None):
        rows, cols = x.shape
        _check(_lib.sppo_layernorm_fwd(self.h, _ptr(x), _ptr(gamma), _ptr(beta), rows, cols, eps, _ptr(y),
                                       _ptr(mean), _ptr(rstd), _stream(stream)))

    def layernorm_bwd(self, dy, x, gamma, mean, rstd, dx, dres=None, stream=None):
        rows, cols = x.shape
        _check(_lib.sppo_layernorm_bwd(self.h, _ptr(dy), _ptr(x), _ptr(gamma), _ptr(mean), _ptr(rstd), _ptr(dres),
                                       rows, cols, _ptr(dx), _stream(stream)))

    def col_reduce(self, dy, rows: int, cols: int, sum_acc, x=None, mean=None, rstd=None, prod_acc=None,
                   stream=None):
        dl = list(dy) if isinstance(dy, (list, tuple)) else [dy]
        arr = (C.c_void_p * len(dl))(*[_ptr(t) for t in dl])
        _check(_lib.sppo_col_reduce(self.h, len(dl), arr, _ptr(x), _ptr(mean), _ptr(rstd), rows, cols,
                                    _ptr(sum_acc), _ptr(prod_acc), _stream(stream)))
