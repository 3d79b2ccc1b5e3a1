"""Thin ctypes binding of libigacd.so (include/igacd.h).  Argument marshalling only.

Every function has the C name.  Device vectors are torch CUDA float64 tensors (PyTorch is
used for device memory and streams only); host vectors are numpy float64 arrays or CPU
tensors.  A nonzero C status raises IgacdError with igacd_last_error().  There is no CPU
fallback: if the shared library is missing, importing this module raises.
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("IGACD_LIB") or os.path.join(_HERE, "lib", "libigacd.so")   # IGACD_LIB: debug builds

if not os.path.exists(LIB_PATH):
    raise ImportError("libigacd.so not built (%s); run __graft_entry__.build()" % LIB_PATH)

_lib = ctypes.CDLL(LIB_PATH)

_c_int, _c_double, _vp, _size_t = ctypes.c_int, ctypes.c_double, ctypes.c_void_p, ctypes.c_size_t
_P = ctypes.POINTER


def _sig(name, args):
    f = getattr(_lib, name)
    f.restype = _c_int
    f.argtypes = args
    return f


_lib.igacd_last_error.restype = ctypes.c_char_p
_lib.igacd_version.restype = ctypes.c_char_p
_create = _sig("igacd_create", [_P(_vp), _c_int, _c_int, _c_int, _c_double, _c_double, _c_double, _P(_c_double),
                                _c_int, _c_int, _c_int, _vp])
_create_form = _sig("igacd_create_form", [_P(_vp), _c_int, _c_int, _c_int, _P(_c_double), _P(_c_double), _c_int,
                                          _c_int, _c_int, _vp])
_destroy = _sig("igacd_destroy", [_vp])
_get_info = _sig("igacd_get_info", [_vp, _P(_c_int), _P(_c_int), _P(_c_int)])
_num_levels = _sig("igacd_num_levels", [_vp, _P(_c_int)])
_level_n = _sig("igacd_level_n", [_vp, _c_int, _P(_c_int)])
_level_tsolve_passes = _sig("igacd_level_tsolve_passes", [_vp, _c_int, _P(_c_int)])
_ndof = _sig("igacd_ndof", [_vp, _c_int, _P(_size_t)])
_omega = _sig("igacd_smoother_omega", [_vp, _c_int, _P(_c_double), _P(_c_double)])
_apply = _sig("igacd_apply", [_vp, _c_int, _vp, _vp, _vp])
_residual = _sig("igacd_residual", [_vp, _c_int, _vp, _vp, _vp, _vp])
_smooth = _sig("igacd_smooth", [_vp, _c_int, _vp, _vp, _c_int, _c_double, _vp])
_restrict = _sig("igacd_restrict", [_vp, _c_int, _vp, _vp, _vp])
_prolong = _sig("igacd_prolong", [_vp, _c_int, _vp, _vp, _c_int, _vp])
_vcycle = _sig("igacd_vcycle", [_vp, _vp, _vp, _vp])
_precond = _sig("igacd_precond", [_vp, _vp, _vp, _vp])
_set_precond = _sig("igacd_set_preconditioner", [_vp, _c_int])
_get_precond = _sig("igacd_get_preconditioner", [_vp, _P(_c_int)])
_set_smoother = _sig("igacd_set_smoother", [_vp, _c_int])
_get_smoother = _sig("igacd_get_smoother", [_vp, _P(_c_int)])
_aux_exact = _sig("igacd_aux_is_exact", [_vp, _P(_c_int)])
_apply_aux = _sig("igacd_apply_aux", [_vp, _c_int, _vp, _vp, _vp])
_aux_omega = _sig("igacd_aux_omega", [_vp, _c_int, _P(_c_double), _P(_c_double)])
_solve = _sig("igacd_solve", [_vp, _vp, _vp, _c_double, _c_int, _P(_c_int), _P(_c_double), _vp])
_tsolve = _sig("igacd_tsolve", [_vp, _c_int, _vp, _vp, _vp])
_set_aux_smoother = _sig("igacd_set_aux_smoother", [_vp, _c_int])
_set_aux_sweeps = _sig("igacd_set_aux_sweeps", [_vp, _c_int, _c_int])
_set_graphs = _sig("igacd_set_graphs", [_vp, _c_int])
_gmres = _sig("igacd_gmres", [_vp, _vp, _vp, _c_double, _c_int, _c_int, _P(_c_int), _P(_c_double), _vp])
_solve_host = _sig("igacd_solve_host", [_vp, _vp, _vp, _c_double, _c_int, _P(_c_int), _P(_c_double), _vp])
_get_band = _sig("igacd_get_band", [_vp, _c_int, _c_int, _P(_c_double)])
_get_prol = _sig("igacd_get_prolongation", [_vp, _c_int, _P(_c_double)])
_set_prof = _sig("igacd_set_profiling", [_vp, _c_int])
_get_prof = _sig("igacd_get_profile", [_vp, _P(ctypes.c_longlong), _P(ctypes.c_longlong), _P(_c_double)])
_reset_prof = _sig("igacd_reset_profile", [_vp])

IGACD_E_NOCONV = -4
IGACD_E_BREAKDOWN = -5
IGACD_PRECOND_VCYCLE = 0
IGACD_PRECOND_AUX = 1
IGACD_PRECOND_AUX_ADD = 2
IGACD_SMOOTH_JACOBI = 0
IGACD_SMOOTH_TOEPLITZ = 1
IGACD_SMOOTH_TOEPLITZ_FINE = 2


class IgacdError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__("igacd error %d: %s" % (code, msg))
        self.code = code


def _check(rc):
    if rc != 0:
        raise IgacdError(rc, _lib.igacd_last_error().decode())


def _dptr(t, n=None):
    """Device pointer of a contiguous CUDA float64 tensor holding exactly ``n`` elements
    (the C side reads / writes n doubles through it, so a short or mistyped buffer is refused
    here instead of corrupting device memory)."""
    if t is None:
        return None
    if not (getattr(t, "is_cuda", False) and str(t.dtype) == "torch.float64" and t.is_contiguous()):
        raise TypeError("expected a contiguous CUDA float64 tensor")
    if n is not None and t.numel() != n:
        raise ValueError("vector has %d elements, the level needs %d" % (t.numel(), n))
    return ctypes.c_void_p(t.data_ptr())


def _hptr(a, n):
    """Host pointer of a C-contiguous float64 numpy array or CPU tensor of exactly n elements."""
    if hasattr(a, "data_ptr"):
        if a.is_cuda or str(a.dtype) != "torch.float64" or not a.is_contiguous():
            raise TypeError("expected a contiguous CPU float64 tensor")
        if a.numel() != n:
            raise ValueError("host vector has %d elements, the system needs %d" % (a.numel(), n))
        return ctypes.c_void_p(a.data_ptr())
    import numpy as np
    if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]):
        raise TypeError("expected a C-contiguous float64 numpy array")
    if a.size != n:
        raise ValueError("host vector has %d elements, the system needs %d" % (a.size, n))
    if not a.flags["WRITEABLE"]:
        raise ValueError("host vector must be writeable")
    return a.ctypes.data_as(ctypes.c_void_p)


def _nvec(h, level=0):
    return igacd_ndof(h, level)


def _nscal(h, level=0):
    return igacd_ndof(h, level) // igacd_get_info(h)[0]


def _stream(stream):
    if stream is None:
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def _darr(vals):
    a = (_c_double * len(vals))(*[float(v) for v in vals])
    return a


def igacd_version():
    return _lib.igacd_version().decode()


def igacd_create(dim, p, n, nu, beta, lam, b0, levels=0, nu_pre=1, nu_post=1, stream=None):
    if len(b0) != dim:
        raise ValueError("b0 needs %d entries, got %d" % (dim, len(b0)))
    h = _vp()
    _check(_create(ctypes.byref(h), dim, p, n, nu, beta, lam, _darr(b0), levels, nu_pre, nu_post, _stream(stream)))
    return h


def igacd_create_form(dim, p, n, mass, K, levels=0, nu_pre=1, nu_post=1, stream=None):
    mass, K = list(mass), list(K)
    if len(mass) != dim * dim or len(K) != dim ** 4:
        raise ValueError("mass needs dim^2 = %d and K dim^4 = %d entries" % (dim * dim, dim ** 4))
    h = _vp()
    _check(_create_form(ctypes.byref(h), dim, p, n, _darr(list(mass)), _darr(list(K)), levels, nu_pre, nu_post,
                        _stream(stream)))
    return h


def igacd_destroy(h):
    _check(_destroy(h))


def igacd_get_info(h):
    d, p, L = _c_int(), _c_int(), _c_int()
    _check(_get_info(h, ctypes.byref(d), ctypes.byref(p), ctypes.byref(L)))
    return d.value, p.value, L.value


def igacd_num_levels(h):
    v = _c_int()
    _check(_num_levels(h, ctypes.byref(v)))
    return v.value


def igacd_level_n(h, level):
    v = _c_int()
    _check(_level_n(h, level, ctypes.byref(v)))
    return v.value


def igacd_level_tsolve_passes(h, level):
    v = _c_int()
    _check(_level_tsolve_passes(h, level, ctypes.byref(v)))
    return v.value


def igacd_ndof(h, level=0):
    v = _size_t()
    _check(_ndof(h, level, ctypes.byref(v)))
    return v.value


def igacd_smoother_omega(h, level):
    w, r = _c_double(), _c_double()
    _check(_omega(h, level, ctypes.byref(w), ctypes.byref(r)))
    return w.value, r.value


def igacd_apply(h, level, x, y, stream=None):
    _check(_apply(h, level, _dptr(x, _nvec(h, level)), _dptr(y, _nvec(h, level)), _stream(stream)))


def igacd_residual(h, level, b, x, r, stream=None):
    _check(_residual(h, level, *[_dptr(v, _nvec(h, level)) for v in (b, x, r)], _stream(stream)))


def igacd_smooth(h, level, b, x, sweeps, omega=0.0, stream=None):
    _check(_smooth(h, level, _dptr(b, _nvec(h, level)), _dptr(x, _nvec(h, level)), sweeps, omega, _stream(stream)))


def igacd_restrict(h, level, x_fine, x_coarse, stream=None):
    _check(_restrict(h, level, _dptr(x_fine, _nvec(h, level)), _dptr(x_coarse, _nvec(h, level + 1)), _stream(stream)))


def igacd_prolong(h, level, x_coarse, x_fine, accumulate=False, stream=None):
    _check(_prolong(h, level, _dptr(x_coarse, _nvec(h, level + 1)), _dptr(x_fine, _nvec(h, level)), 1 if accumulate else 0, _stream(stream)))


def igacd_vcycle(h, b, x, stream=None):
    _check(_vcycle(h, _dptr(b, _nvec(h)), _dptr(x, _nvec(h)), _stream(stream)))


def igacd_precond(h, b, x, stream=None):
    _check(_precond(h, _dptr(b, _nvec(h)), _dptr(x, _nvec(h)), _stream(stream)))


def igacd_set_preconditioner(h, mode):
    _check(_set_precond(h, mode))


def igacd_get_preconditioner(h):
    v = _c_int()
    _check(_get_precond(h, ctypes.byref(v)))
    return v.value


def igacd_set_smoother(h, kind):
    _check(_set_smoother(h, kind))


def igacd_get_smoother(h):
    v = _c_int()
    _check(_get_smoother(h, ctypes.byref(v)))
    return v.value


def igacd_aux_is_exact(h):
    v = _c_int()
    _check(_aux_exact(h, ctypes.byref(v)))
    return v.value


def igacd_apply_aux(h, level, s_in, s_out, stream=None):
    _check(_apply_aux(h, level, _dptr(s_in, _nscal(h, level)), _dptr(s_out, _nscal(h, level)), _stream(stream)))


def igacd_aux_omega(h, level):
    w, r = _c_double(), _c_double()
    _check(_aux_omega(h, level, ctypes.byref(w), ctypes.byref(r)))
    return w.value, r.value


def igacd_solve(h, b, x, tol, maxit, stream=None, raise_on_noconv=True):
    it, rel = _c_int(), _c_double()
    rc = _solve(h, _dptr(b, _nvec(h)), _dptr(x, _nvec(h)), tol, maxit, ctypes.byref(it), ctypes.byref(rel), _stream(stream))
    if rc != IGACD_E_NOCONV or raise_on_noconv:
        _check(rc)
    return it.value, rel.value


def igacd_tsolve(h, level, b, x, stream=None):
    _check(_tsolve(h, level, _dptr(b, _nvec(h, level)), _dptr(x, _nvec(h, level)), _stream(stream)))


def igacd_set_aux_smoother(h, kind):
    _check(_set_aux_smoother(h, kind))


def igacd_set_aux_sweeps(h, nu_pre, nu_post):
    _check(_set_aux_sweeps(h, nu_pre, nu_post))


def igacd_set_graphs(h, enable):
    _check(_set_graphs(h, 1 if enable else 0))


def igacd_gmres(h, b, x, tol, maxit, restart=30, stream=None, raise_on_noconv=True):
    it, rel = _c_int(), _c_double()
    rc = _gmres(h, _dptr(b, _nvec(h)), _dptr(x, _nvec(h)), tol, maxit, restart, ctypes.byref(it), ctypes.byref(rel), _stream(stream))
    if rc != IGACD_E_NOCONV or raise_on_noconv:
        _check(rc)
    return it.value, rel.value


def igacd_solve_host(h, b_host, x_host, tol, maxit, stream=None, raise_on_noconv=True):
    """b_host / x_host: C-contiguous float64 numpy arrays or CPU tensors (pinned or not) of
    exactly igacd_ndof(h) elements (checked: the C side copies that many doubles)."""
    N = _nvec(h)
    it, rel = _c_int(), _c_double()
    rc = _solve_host(h, _hptr(b_host, N), _hptr(x_host, N), tol, maxit, ctypes.byref(it), ctypes.byref(rel), _stream(stream))
    if rc != IGACD_E_NOCONV or raise_on_noconv:
        _check(rc)
    return it.value, rel.value


def igacd_get_band(h, level, which):
    import numpy as np
    n = igacd_level_n(h, level)
    p = _handle_p(h)
    m = n + p - 2
    out = np.zeros(m * (2 * p + 1))
    _check(_get_band(h, level, which, out.ctypes.data_as(_P(_c_double))))
    return out.reshape(m, 2 * p + 1)


def igacd_get_prolongation(h, level):
    import numpy as np
    p = _handle_p(h)
    mf = igacd_level_n(h, level) + p - 2
    mc = igacd_level_n(h, level + 1) + p - 2
    out = np.zeros(mf * mc)
    _check(_get_prol(h, level, out.ctypes.data_as(_P(_c_double))))
    return out.reshape(mf, mc)


def _handle_p(h):
    return igacd_get_info(h)[1]


def igacd_set_profiling(h, enable):
    _check(_set_prof(h, 1 if enable else 0))


def igacd_get_profile(h):
    a, b, c = ctypes.c_longlong(), ctypes.c_longlong(), _c_double()
    _check(_get_prof(h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
    return a.value, b.value, c.value


def igacd_reset_profile(h):
    _check(_reset_prof(h))
