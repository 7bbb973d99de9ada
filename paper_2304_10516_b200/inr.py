"""Thin ctypes binding of libinr.so (include/inr.h): argument marshalling only.

Every function here has the name of the C entry point it wraps and does no
computation of its own; all work runs in the sm_100a kernels of libinr.so.
Device buffers are passed as integer device pointers (e.g. a torch CUDA
tensor's ``data_ptr()``), streams as integer ``cudaStream_t`` handles (e.g.
``torch.cuda.current_stream().cuda_stream``).  A missing library raises
ImportError: there is no CPU fallback.
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("INR_LIB_PATH") or os.path.join(_HERE, "lib", "libinr.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "inr.h")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libinr.so not built at {LIB_PATH}: run __graft_entry__.build() "
                      "(make -C paper_2304_10516_b200); there is no CPU fallback")
_lib = ctypes.CDLL(LIB_PATH)

# ---- status codes / enums (inr.h)
INR_OK, INR_ERR_INVALID_ARG, INR_ERR_DOMAIN, INR_ERR_NONFINITE = 0, 1, 2, 3
INR_ERR_OOM, INR_ERR_CUDA, INR_ERR_STATE, INR_ERR_UNSUPPORTED = 4, 5, 6, 7
INR_PREC_FP32, INR_PREC_FP16_MLP = 0, 1
INR_REDUCE_ATOMIC, INR_REDUCE_DETERMINISTIC = 0, 1
CACHE_HOST_RESIDENT, CACHE_FP16 = 1, 2
STATUS_NAMES = {0: "OK", 1: "INVALID_ARG", 2: "DOMAIN", 3: "NONFINITE", 4: "OOM", 5: "CUDA", 6: "STATE",
                7: "UNSUPPORTED"}


class InrError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class inr_config(ctypes.Structure):
    _fields_ = [("levels", ctypes.c_int32), ("features", ctypes.c_int32), ("log2_table_size", ctypes.c_int32),
                ("base_resolution", ctypes.c_int32), ("per_level_scale", ctypes.c_float),
                ("mlp_width", ctypes.c_int32), ("mlp_hidden_layers", ctypes.c_int32), ("out_dim", ctypes.c_int32),
                ("mlp_bias", ctypes.c_int32), ("precision", ctypes.c_int32), ("reduction", ctypes.c_int32),
                ("seed", ctypes.c_uint64)]


class inr_block(ctypes.Structure):
    _fields_ = [("origin", ctypes.c_int64 * 3), ("n", ctypes.c_int32 * 3), ("global_dims", ctypes.c_int64 * 3)]


class inr_fit_opts(ctypes.Structure):
    _fields_ = [("lambda_", ctypes.c_double), ("boundary_batch", ctypes.c_int32), ("lr0", ctypes.c_double),
                ("lr_decay", ctypes.c_double), ("lr_step", ctypes.c_int32), ("beta1", ctypes.c_double),
                ("beta2", ctypes.c_double), ("eps", ctypes.c_double), ("vmin", ctypes.c_double),
                ("vmax", ctypes.c_double), ("target_psnr", ctypes.c_double), ("check_interval", ctypes.c_int32),
                ("vmin_c", ctypes.c_double * 3), ("vmax_c", ctypes.c_double * 3), ("sparse_adam", ctypes.c_int32),
                ("split_step", ctypes.c_int32)]

    def set_range(self, lo, hi):
        """Scalar range (scalar fields) or per-channel sequences (vector fields)."""
        if hasattr(lo, "__len__"):
            for c in range(len(lo)):
                self.vmin_c[c], self.vmax_c[c] = float(lo[c]), float(hi[c])
            self.vmin, self.vmax = float(lo[0]), float(hi[0])
        else:
            self.vmin, self.vmax = float(lo), float(hi)


class inr_fit_report(ctypes.Structure):
    _fields_ = [("steps_taken", ctypes.c_int32), ("reached_target", ctypes.c_int32),
                ("constant_field", ctypes.c_int32), ("loss_uniform", ctypes.c_double),
                ("loss_boundary", ctypes.c_double), ("probe_psnr", ctypes.c_double)]


class inr_camera(ctypes.Structure):
    _fields_ = [("eye", ctypes.c_double * 3), ("look", ctypes.c_double * 3), ("up", ctypes.c_double * 3),
                ("fovy_deg", ctypes.c_double), ("width", ctypes.c_int32), ("height", ctypes.c_int32)]


class inr_transfer_fn(ctypes.Structure):
    _fields_ = [("npoints", ctypes.c_int32), ("s", ctypes.c_float * 16), ("rgba", (ctypes.c_float * 4) * 16),
                ("vmin", ctypes.c_double), ("vmax", ctypes.c_double), ("base_step", ctypes.c_double)]


def make_camera(eye, look, up, fovy, width, height):
    return inr_camera((ctypes.c_double * 3)(*eye), (ctypes.c_double * 3)(*look), (ctypes.c_double * 3)(*up),
                      float(fovy), int(width), int(height))


def make_tf(points, rgba, vmin, vmax, base_step=1.0):
    t = inr_transfer_fn()
    t.npoints = len(points)
    for i, (sv, c) in enumerate(zip(points, rgba)):
        t.s[i] = sv
        for k in range(4):
            t.rgba[i][k] = c[k]
    t.vmin, t.vmax, t.base_step = float(vmin), float(vmax), float(base_step)
    return t


class inr_view(ctypes.Structure):
    _fields_ = [("base", ctypes.c_void_p), ("lo", ctypes.c_int64 * 3), ("dims", ctypes.c_int32 * 3),
                ("stride", ctypes.c_int64 * 3), ("channels", ctypes.c_int32)]


_P = ctypes.c_void_p
_I32, _I64, _U64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
_PP = ctypes.POINTER(ctypes.c_void_p)
_SIG = {
    "inr_last_error": (ctypes.c_char_p, []),
    "inr_create": (_I32, [ctypes.POINTER(inr_config), ctypes.POINTER(inr_block), ctypes.c_int, _PP]),
    "inr_reset": (_I32, [_P, _U64]),
    "inr_destroy": (_I32, [_P]),
    "inr_reset_optimizer": (_I32, [_P]),
    "inr_state_bytes": (_I32, [_P, ctypes.POINTER(_I64)]),
    "inr_export_state": (_I32, [_P, _P, _P]),
    "inr_import_state": (_I32, [_P, _P, _P]),
    "inr_set_mesh": (_I32, [_P, ctypes.POINTER(ctypes.c_void_p)]),
    "inr_param_count": (_I32, [_P, ctypes.POINTER(_I64)]),
    "inr_param_bytes": (_I32, [_P, ctypes.POINTER(_I64)]),
    "inr_steps": (_I32, [_P, ctypes.POINTER(_I64)]),
    "inr_fit_opts_default": (None, [ctypes.POINTER(inr_fit_opts)]),
    "inr_fit": (_I32, [_P, ctypes.POINTER(inr_view), _I32, _I32, ctypes.POINTER(inr_fit_opts),
                       ctypes.POINTER(inr_fit_report), _P]),
    "inr_fit_group": (_I32, [_PP, ctypes.POINTER(inr_view), _I32, _I32, _I32, ctypes.POINTER(inr_fit_opts),
                             ctypes.POINTER(inr_fit_report), _P]),
    "inr_fit_losses": (_I32, [_PP, _I32, _P, _P]),
    "inr_decode": (_I32, [_P, _P, _I64, _P, _I32, _P]),
    "inr_decode_group": (_I32, [_PP, _I32, _P, _I64, _P, _I32, _P]),
    "inr_decode_grid": (_I32, [_P, ctypes.POINTER(_I32), _P, ctypes.POINTER(_I64), _P, _P, _P]),
    "inr_decode_grid_part": (_I32, [_P, ctypes.POINTER(_I32), ctypes.POINTER(_I32), _P, ctypes.POINTER(_I64), _P,
                                    _P, _P]),
    "inr_value_range": (_I32, [ctypes.POINTER(inr_view), _P, _P]),
    "cache_create": (_I32, [_I32, _I32, ctypes.c_int, _PP]),
    "cache_destroy": (_I32, [_P]),
    "cache_insert": (_I32, [_P, _I64, _PP, _I32, ctypes.POINTER(_I64), _P]),
    "cache_evict": (_I32, [_P, ctypes.POINTER(_I64)]),
    "cache_size": (_I32, [_P, ctypes.POINTER(_I32)]),
    "cache_bytes": (_I32, [_P, ctypes.POINTER(_I64)]),
    "cache_get": (_I32, [_P, _I32, ctypes.POINTER(_I64), ctypes.POINTER(_PP), ctypes.POINTER(_I32)]),
    "inr_trace_grids": (_I32, [ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_double), _I32,
                               ctypes.POINTER(_I64), ctypes.c_double, _P, _I32, ctypes.c_double, _I32, _P, _P, _P,
                               _P]),
    "inr_pathlines": (_I32, [_P, _I32, _P, _I32, ctypes.c_double, _I32, _P, _P, _P, _P]),
    "inr_renderer_create": (_I32, [_PP, _I32, _I32, ctypes.c_double, _P, _PP]),
    "inr_renderer_destroy": (_I32, [_P]),
    "inr_render": (_I32, [_P, ctypes.POINTER(inr_camera), ctypes.POINTER(inr_transfer_fn),
                          ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double), ctypes.c_double,
                          ctypes.c_double, _I32, _P, _P]),
    "inr_render_stats": (_I32, [_P, ctypes.POINTER(_I64), ctypes.POINTER(_I64), ctypes.POINTER(_I32)]),
    "inr_composite": (_I32, [_P, _I32, _I64, ctypes.POINTER(ctypes.c_float), _P, _P]),
    "inr_ipc_handle": (_I32, [_P, ctypes.c_char_p, ctypes.POINTER(_I64)]),
    "inr_ipc_open": (_I32, [ctypes.c_char_p, _I64, ctypes.c_int, ctypes.POINTER(_P), ctypes.POINTER(_P)]),
    "inr_ipc_close": (_I32, [_P]),
    "inr_get_params": (_I32, [_P, _P, _I64]),
    "inr_set_params": (_I32, [_P, _P, _I64]),
    "inr_get_grads": (_I32, [_P, _P, _I64]),
    "inr_get_adam_state": (_I32, [_P, _P, _P, _I64]),
    "inr_debug_encode": (_I32, [_P, _P, _I64, _P, _P, _P]),
    "inr_debug_forward": (_I32, [_P, _P, _I64, _P, _P]),
    "inr_kernel_launches": (_I64, []),
    "inr_profile_enable": (_I32, [_I32]),
    "inr_profile_read": (_I32, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_I64)]),
    "inr_profile_span": (_I32, [ctypes.POINTER(ctypes.c_double)]),
}
for _name, (_res, _args) in _SIG.items():
    if not hasattr(_lib, _name) and os.environ.get("INR_LIB_PATH"):
        continue  # an older diagnostic build
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args

lib = _lib


def inr_last_error():
    return _lib.inr_last_error().decode()


def _check(status):
    if status != INR_OK:
        raise InrError(status, inr_last_error())


def _ptrs(handles):
    arr = (ctypes.c_void_p * len(handles))(*[h.value if isinstance(h, ctypes.c_void_p) else h for h in handles])
    return ctypes.cast(arr, _PP), arr


def make_config(levels=16, features=2, log2_table_size=19, base_resolution=4, per_level_scale=2.0, mlp_width=64,
                mlp_hidden_layers=3, out_dim=1, mlp_bias=1, precision=INR_PREC_FP32, reduction=INR_REDUCE_ATOMIC,
                seed=0x230410516):
    return inr_config(levels, features, log2_table_size, base_resolution, per_level_scale, mlp_width,
                      mlp_hidden_layers, out_dim, mlp_bias, precision, reduction, seed)


def make_block(origin, n, global_dims):
    return inr_block((ctypes.c_int64 * 3)(*origin), (ctypes.c_int32 * 3)(*n), (ctypes.c_int64 * 3)(*global_dims))


def make_view(base_ptr, lo, dims, stride, channels=1):
    """Strides in elements per node; a vector field (channels = 3) stores channel c at +c."""
    return inr_view(base_ptr, (ctypes.c_int64 * 3)(*lo), (ctypes.c_int32 * 3)(*dims), (ctypes.c_int64 * 3)(*stride),
                    channels)


def inr_fit_opts_default():
    o = inr_fit_opts()
    _lib.inr_fit_opts_default(ctypes.byref(o))
    return o


# ---- models
def inr_create(cfg, block, device=0):
    h = ctypes.c_void_p()
    _check(_lib.inr_create(ctypes.byref(cfg), ctypes.byref(block), device, ctypes.byref(h)))
    return h


def inr_reset(m, seed):
    _check(_lib.inr_reset(m, seed))


def inr_reset_optimizer(m):
    _check(_lib.inr_reset_optimizer(m))


def inr_set_mesh(m, coords):
    """coords: three float64 arrays of the global node coordinates per axis (x, y, z), or None (uniform)."""
    if coords is None:
        _check(_lib.inr_set_mesh(m, None))
        return
    import numpy as _np
    arrs = [_np.ascontiguousarray(c, dtype=_np.float64) for c in coords]
    ptrs = (ctypes.c_void_p * 3)(*[a.ctypes.data for a in arrs])
    _check(_lib.inr_set_mesh(m, ptrs))


def inr_state_bytes(m):
    n = _I64()
    _check(_lib.inr_state_bytes(m, ctypes.byref(n)))
    return n.value


def inr_export_state(m, dst_ptr, stream=0):
    _check(_lib.inr_export_state(m, dst_ptr, stream))


def inr_import_state(m, src_ptr, stream=0):
    _check(_lib.inr_import_state(m, src_ptr, stream))


def inr_destroy(m):
    _check(_lib.inr_destroy(m))


def inr_param_count(m):
    n = _I64()
    _check(_lib.inr_param_count(m, ctypes.byref(n)))
    return n.value


def inr_param_bytes(m):
    n = _I64()
    _check(_lib.inr_param_bytes(m, ctypes.byref(n)))
    return n.value


def inr_steps(m):
    n = _I64()
    _check(_lib.inr_steps(m, ctypes.byref(n)))
    return n.value


def inr_fit(m, view, steps, batch, opts, stream=0, report=True):
    rep = inr_fit_report() if report else None
    _check(_lib.inr_fit(m, ctypes.byref(view), steps, batch, ctypes.byref(opts),
                        ctypes.byref(rep) if rep is not None else None, stream))
    return rep


def inr_fit_group(models, views, steps, batch, opts, stream=0, report=True):
    if len(views) != len(models):
        raise ValueError(f"{len(models)} models but {len(views)} views")
    pp, keep = _ptrs(models)
    va = (inr_view * len(views))(*views)
    reps = (inr_fit_report * len(models))() if report else None
    _check(_lib.inr_fit_group(pp, va, len(models), steps, batch, ctypes.byref(opts), reps, stream))
    return list(reps) if reps is not None else None


def inr_fit_losses(models, out_ptr, stream=0):
    """Enqueue the (L1_u, L1_b, nonfinite) report of every model's last step into out (3 doubles per model)."""
    pp, keep = _ptrs(models)
    _check(_lib.inr_fit_losses(pp, len(models), out_ptr, stream))


def inr_decode(m, xyz_ptr, q, out_ptr, strict=0, stream=0):
    _check(_lib.inr_decode(m, xyz_ptr, q, out_ptr, strict, stream))


def inr_decode_group(models, xyz_ptr, q, out_ptr, strict=0, stream=0):
    pp, keep = _ptrs(models)
    _check(_lib.inr_decode_group(pp, len(models), xyz_ptr, q, out_ptr, strict, stream))


def inr_decode_grid(m, res, out_ptr, out_stride=None, ref_ptr=None, sse_ptr=None, stream=0, count=None):
    for name, t in (("res", res), ("out_stride", out_stride), ("count", count)):
        if t is not None and len(t) != 3:
            raise ValueError(f"{name} must have 3 entries (x, y, z), got {len(t)}")
    r = (_I32 * 3)(*res)
    s = (_I64 * 3)(*out_stride) if out_stride is not None else None
    if count is None:
        _check(_lib.inr_decode_grid(m, r, out_ptr, s, ref_ptr, sse_ptr, stream))
    else:
        _check(_lib.inr_decode_grid_part(m, r, (_I32 * 3)(*count), out_ptr, s, ref_ptr, sse_ptr, stream))


def inr_value_range(view, minmax_ptr, stream=0):
    _check(_lib.inr_value_range(ctypes.byref(view), minmax_ptr, stream))


# ---- pathlines (NEXT-2)
INR_PATH_WINDOW_EXHAUSTED, INR_PATH_OUT_OF_DOMAIN, INR_PATH_MAX_STEPS = 0, 1, 2
INR_WINDOW_REVERSE, INR_WINDOW_NEGATE = 1, 2


def inr_trace_grids(grid_ptrs, times, dims, sign, seeds_ptr, nseeds, dt, max_steps, vert_ptr, counts_ptr,
                    reasons_ptr, stream=0):
    g = (ctypes.c_void_p * len(grid_ptrs))(*grid_ptrs)
    t = (ctypes.c_double * len(times))(*[float(v) for v in times])
    _check(_lib.inr_trace_grids(ctypes.cast(g, _PP), t, len(grid_ptrs), (_I64 * 3)(*dims), float(sign), seeds_ptr,
                                nseeds, float(dt), max_steps, vert_ptr, counts_ptr, reasons_ptr, stream))


def inr_pathlines(cache, window_ops, seeds_ptr, nseeds, dt, max_steps, vert_ptr, counts_ptr, reasons_ptr, stream=0):
    _check(_lib.inr_pathlines(cache, window_ops, seeds_ptr, nseeds, float(dt), max_steps, vert_ptr, counts_ptr,
                              reasons_ptr, stream))


# ---- volume rendering (NEXT-3)
def inr_renderer_create(models, cells=16, pad=0.0, stream=0):
    pp, keep = _ptrs(models)
    h = ctypes.c_void_p()
    _check(_lib.inr_renderer_create(pp, len(models), cells, float(pad), stream, ctypes.byref(h)))
    return h


def inr_renderer_destroy(r):
    _check(_lib.inr_renderer_destroy(r))


def inr_render(r, cam, tf, lo, hi, step, frag_ptr, stop_alpha=0.99, use_macrocells=1, stream=0):
    _check(_lib.inr_render(r, ctypes.byref(cam), ctypes.byref(tf), (ctypes.c_double * 3)(*lo),
                           (ctypes.c_double * 3)(*hi), float(step), float(stop_alpha), int(use_macrocells), frag_ptr,
                           stream))


def inr_render_stats(r):
    e, s, w = _I64(), _I64(), _I32()
    _check(_lib.inr_render_stats(r, ctypes.byref(e), ctypes.byref(s), ctypes.byref(w)))
    return e.value, s.value, w.value


def inr_composite(frag_ptr, nfrag, npixels, bg, img_ptr, stream=0):
    _check(_lib.inr_composite(frag_ptr, nfrag, npixels, (ctypes.c_float * 3)(*bg), img_ptr, stream))


# ---- peer memory (fused decode + gather)
def inr_ipc_handle(ptr):
    """(64-byte handle, offset) of the device allocation holding ptr."""
    h = ctypes.create_string_buffer(64)
    off = _I64()
    _check(_lib.inr_ipc_handle(ptr, h, ctypes.byref(off)))
    return h.raw, off.value


def inr_ipc_open(handle, offset, device):
    """Map another process's allocation: (pointer, base for inr_ipc_close)."""
    p, b = ctypes.c_void_p(), ctypes.c_void_p()
    _check(_lib.inr_ipc_open(handle, offset, device, ctypes.byref(p), ctypes.byref(b)))
    return p.value, b.value


def inr_ipc_close(base):
    _check(_lib.inr_ipc_close(base))


# ---- cache
def cache_create(capacity, flags=0, device=0):
    """flags: CACHE_HOST_RESIDENT | CACHE_FP16 (inr.h)."""
    h = ctypes.c_void_p()
    _check(_lib.cache_create(capacity, flags, device, ctypes.byref(h)))
    return h


def cache_destroy(c):
    _check(_lib.cache_destroy(c))


def cache_insert(c, timestep, models, stream=0):
    pp, keep = _ptrs(models)
    ev = _I64()
    _check(_lib.cache_insert(c, timestep, pp, len(models), ctypes.byref(ev), stream))
    return ev.value


def cache_evict(c):
    ev = _I64()
    _check(_lib.cache_evict(c, ctypes.byref(ev)))
    return ev.value


def cache_size(c):
    n = _I32()
    _check(_lib.cache_size(c, ctypes.byref(n)))
    return n.value


def cache_bytes(c):
    n = _I64()
    _check(_lib.cache_bytes(c, ctypes.byref(n)))
    return n.value


def cache_get(c, i):
    ts, nb = _I64(), _I32()
    arr = _PP()
    _check(_lib.cache_get(c, i, ctypes.byref(ts), ctypes.byref(arr), ctypes.byref(nb)))
    return ts.value, [ctypes.c_void_p(arr[k]) for k in range(nb.value)]


# ---- parity surface (host buffers are numpy float32 arrays)
def _host(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def inr_get_params(m, out):
    _check(_lib.inr_get_params(m, _host(out), out.size))
    return out


def inr_set_params(m, params):
    _check(_lib.inr_set_params(m, _host(params), params.size))


def inr_get_grads(m, out):
    _check(_lib.inr_get_grads(m, _host(out), out.size))
    return out


def inr_get_adam_state(m, m_out, v_out):
    _check(_lib.inr_get_adam_state(m, _host(m_out), _host(v_out), m_out.size))
    return m_out, v_out


def inr_debug_encode(m, x01_ptr, q, idx_ptr=None, feat_ptr=None, stream=0):
    _check(_lib.inr_debug_encode(m, x01_ptr, q, idx_ptr, feat_ptr, stream))


def inr_debug_forward(m, x01_ptr, q, y_ptr, stream=0):
    _check(_lib.inr_debug_forward(m, x01_ptr, q, y_ptr, stream))


def inr_kernel_launches():
    return _lib.inr_kernel_launches()


def inr_profile_enable(on=1):
    _check(_lib.inr_profile_enable(on))


def inr_profile_read(kernel):
    """(total device ms, launches) of one kernel class since inr_profile_enable(1)."""
    ms, n = ctypes.c_double(), _I64()
    _check(_lib.inr_profile_read(kernel.encode(), ctypes.byref(ms), ctypes.byref(n)))
    return ms.value, n.value


def inr_profile_span():
    """Device ms from the first recorded kernel start to the last kernel end."""
    ms = ctypes.c_double()
    _check(_lib.inr_profile_span(ctypes.byref(ms)))
    return ms.value
