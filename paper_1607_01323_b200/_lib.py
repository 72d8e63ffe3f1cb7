"""ctypes binding of the C ABI in include/dgmf.h (libdgmf.so, built in-tree).

The product path has no CPU fallback: if the CUDA library is missing or no
CUDA device is present, every operator raises.
"""

import ctypes
import os
import subprocess
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB_PATH = os.environ.get("DG_LIB") or os.path.join(HERE, "libdgmf.so")  # DG_LIB: A/B builds
CSRC = os.path.join(HERE, "csrc")

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
              "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
              "-diag-suppress", "177"]

DG_OK, DG_EINVAL, DG_ECUDA, DG_ENOTSUP = 0, -1, -2, -3
BC_NONE, BC_VELOCITY_DIRICHLET, BC_VELOCITY_NEUMANN = 0, 1, 2


def sources():
    names = ["dgmf.cu", "vecops.cu", "vec_over.cu", "vcart.cu", "gen2d.cu", "tables.cpp"]
    names += [f"vec_lin{d}_{p}.cu" for d in (2, 3) for p in ("00", "01", "10", "11")]
    return [os.path.join(CSRC, f) for f in names]


def _up_to_date(obj):
    """Object newer than its source and every header nvcc listed for it."""
    dep = obj + ".d"
    if not (os.path.exists(obj) and os.path.exists(dep)):
        return False
    text = open(dep).read().replace("\\\n", " ")
    files = text.split(":", 1)[1].split() if ":" in text else []
    t = os.path.getmtime(obj)
    return all(os.path.exists(f) and os.path.getmtime(f) <= t for f in files)


def build(verbose=False, force=False):
    """Compile libdgmf.so for sm_100a with nvcc (in-tree, travels with the repo).
    One nvcc per translation unit, run in parallel, then one link."""
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(ROOT, "include", "dgmf.h"))
    if (not force and os.path.exists(LIB_PATH) and
            os.path.getmtime(LIB_PATH) >= max(os.path.getmtime(d) for d in deps)):
        return LIB_PATH
    nvcc = os.environ.get("NVCC", "nvcc")
    objdir = os.path.join(HERE, "_build")
    os.makedirs(objdir, exist_ok=True)
    compile_flags = [f for f in NVCC_FLAGS if f != "-shared"]
    procs, objs = [], []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        if not force and _up_to_date(obj):
            continue
        cmd = [nvcc] + compile_flags + ["-MD", "-MF", obj + ".d", "-c", "-o", obj, src]
        if verbose:
            print(" ".join(cmd))
        procs.append((subprocess.Popen(cmd, cwd=HERE), src))
    failed = [src for p, src in procs if p.wait() != 0]
    if failed:
        raise subprocess.CalledProcessError(1, f"nvcc {failed}")
    cmd = [nvcc] + NVCC_FLAGS + ["-o", LIB_PATH + ".tmp"] + objs
    subprocess.run(cmd, check=True, cwd=HERE)
    os.replace(LIB_PATH + ".tmp", LIB_PATH)
    return LIB_PATH


class MeshDesc(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int), ("k", ctypes.c_int),
                ("n_q_over", ctypes.c_int), ("counts", ctypes.c_int * 3),
                ("vertices", ctypes.POINTER(ctypes.c_double) * 3),
                ("periodic", ctypes.c_int * 3), ("bc_kind", ctypes.c_int * 6),
                ("slab_begin", ctypes.c_int), ("slab_end", ctypes.c_int)]


class PcgParams(ctypes.Structure):
    _fields_ = [("tau_scale", ctypes.c_double), ("project_dual", ctypes.c_int),
                ("cheb_degree", ctypes.c_int), ("cheb_range", ctypes.c_double),
                ("cheb_lambda_max", ctypes.c_double), ("rel_tol", ctypes.c_double),
                ("abs_tol", ctypes.c_double), ("max_iter", ctypes.c_int)]


class PcgStats(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int), ("residual", ctypes.c_double),
                ("converged", ctypes.c_int), ("breakdown", ctypes.c_int)]


class G2Desc(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int), ("nq", ctypes.c_int), ("ncells", ctypes.c_int64),
                ("jxw", ctypes.c_void_p), ("jit", ctypes.c_void_p), ("fsj", ctypes.c_void_p),
                ("fnrm", ctypes.c_void_p), ("fjit", ctypes.c_void_p), ("tau", ctypes.c_void_p),
                ("nbr", ctypes.c_void_p), ("nslot", ctypes.c_void_p), ("nflip", ctypes.c_void_p),
                ("S", ctypes.POINTER(ctypes.c_double)), ("D", ctypes.POINTER(ctypes.c_double)),
                ("Si", ctypes.POINTER(ctypes.c_double)), ("ld", ctypes.POINTER(ctypes.c_double)),
                ("rd", ctypes.POINTER(ctypes.c_double))]


class G2Params(ctypes.Structure):
    _fields_ = [("op", ctypes.c_int), ("tau_scale", ctypes.c_double), ("kind", ctypes.c_void_p),
                ("gamma0_dt", ctypes.c_double), ("nu", ctypes.c_double),
                ("tau_d", ctypes.c_void_p), ("tau_c", ctypes.c_void_p),
                ("scale", ctypes.c_double), ("form", ctypes.c_int), ("n_hist", ctypes.c_int),
                ("hist", ctypes.c_void_p * 4), ("beta", ctypes.c_double * 4),
                ("gdata", ctypes.c_void_p * 4), ("body", ctypes.c_void_p),
                ("vort", ctypes.c_void_p * 4), ("fdata", ctypes.c_void_p)]


_P = ctypes.c_void_p
_D = ctypes.c_double
_I = ctypes.c_int
_L = ctypes.c_int64
_DP = ctypes.POINTER(ctypes.c_double)

# name -> argtypes (all return int)
PROTOTYPES = {
    "dg_ctx_create": [ctypes.POINTER(MeshDesc), ctypes.POINTER(_P)],
    "dg_ctx_destroy": [_P],
    "dg_ctx_sizes": [_P, ctypes.POINTER(_L), ctypes.POINTER(_L)],
    "dg_ctx_tau": [_P, _DP],
    "dg_basis_tables": [_I, _I, _DP, _DP, _DP, _DP, _DP, _DP, _DP],
    "dg_laplace_vmult": [_P, _P, _P, _D, _P],
    "dg_laplace_vmult_part": [_P, _P, _P, _D, _I, _P],
    "dg_laplace_vmult_split": [_P, _P, _P, _D, _I, _P],
    "dg_cg_dots": [_P, _P, _P, _P, _P],
    "dg_laplace_vmult_dots": [_P, _P, _P, _D, _P, _P],
    "dg_laplace_vmult_split_dots": [_P, _P, _P, _D, _I, _P, _P],
    "dg_laplace_kernel_name": [_P, ctypes.c_char_p, _I],
    "dg_cg_update": [_P, _P, _P, _P, _P, _P, _I, _P, _P, _P, _P],
    "dg_cg_pupdate": [_P, _P, _P, _P, _P],
    "dg_cheb_vec_init": [_P, _P, _P, _P, _P, _P, _D, _P],
    "dg_cheb_vec_step": [_P, _P, _P, _P, _P, _P, _P, _D, _D, _P],
    "dg_laplace_vmult_host": [_P, _P, _P, _D, _I, _P],
    "dg_laplace_diagonal": [_P, _P, _D, _P],
    "dg_mass": [_P, _P, _P, _I, _P],
    "dg_inverse_mass": [_P, _P, _P, _I, _P],
    "dg_helmholtz_vmult": [_P, _P, _P, _D, _D, _P],
    "dg_projection_vmult": [_P, _P, _P, _P, _P, _P],
    "dg_convective_rhs": [_P, _I, _P, _P, _P, _P],
    "dg_convective_rhs_ex": [_P, _I, _P, _P, _P, _P, _P, _P],
    "dg_divergence_rhs": [_P, _P, _P, _D, _I, _P],
    "dg_pressure_gradient_rhs": [_P, _P, _P, _D, _I, _P],
    "dg_vorticity": [_P, _P, _P, _P],
    "dg_pressure_neumann_rhs": [_P, _I, _P, _P, _P, _D, _P, _P, _P],
    "dg_gp_dirichlet_rhs": [_P, _P, _D, _P, _P],
    "dg_viscous_rhs_bc": [_P, _P, _D, _P, _P],
    "dg_element_local_pcg": [_P, _P, _P, _P, _D, _I, _D, _P, _P, _P],
    "dg_penalty_parameters": [_P, _P, _D, _D, _D, _D, _P, _P, _P],
    "dg_dot": [_P, _P, _P, _L, _P, _P],
    "dg_zero_mean_dual": [_P, _P, _P],
    "dg_zero_mean": [_P, _P, _P],
    "dg_laplace_pcg": [_P, _P, _P, _P, ctypes.POINTER(PcgParams),
                       ctypes.POINTER(PcgStats), _DP, _P],
    "dg_cheb_step": [_P, _P, _P, _P, _P, _P, _D, _D, _D, _P],
    "dg_vector_pcg": [_P, ctypes.c_int, _D, _D, _P, _P, _P, _P, _D, _D, ctypes.c_int,
                      ctypes.POINTER(PcgStats), _DP, _P],
    "dg_laplace_pcg_mg": [_P, _P, _P, _P, ctypes.POINTER(PcgParams),
                          ctypes.POINTER(PcgStats), _DP, _P],
    "dg_mg_prolong": [_P, _P, _P, _P, _I, _P],
    "dg_mg_restrict": [_P, _P, _P, _P, _P],
    "dg_mg_create": [_P, _I, _P, _P, _I, _D, _I, _D, _D, ctypes.POINTER(_P)],
    "dg_mg_destroy": [_P],
    "dg_mg_set_precision": [_P, _I],
    "dg_g2_create": [ctypes.POINTER(G2Desc), ctypes.POINTER(_P)],
    "dg_g2_destroy": [_P],
    "dg_g2_apply": [_P, _I, _D, _P, _P, _P, _I, _P],
    "dg_g2_laplace_diagonal": [_P, _D, _P, _P, _P],
    "dg_g2_operator": [_P, ctypes.POINTER(G2Params), _P, _P, _P],
    "dg_g2_transfer": [_I, _I, _L, _P, _P, _L, _P, _P, _P, _I, _P],
    "dg_mg_vcycle": [_P, _P, _P, _P],
    "dg_halo_count": [_P, ctypes.POINTER(_L)],
    "dg_halo_pack": [_P, _P, _P, _P, _P],
    "dg_halo_attach": [_P, _P, _P],
}

_lib = None
_lock = threading.Lock()


class DgError(RuntimeError):
    pass


def lib():
    """Load libdgmf.so (never a CPU fallback: raises if it cannot)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise DgError(f"CUDA library {LIB_PATH} is missing: run "
                          "__graft_entry__.build() (nvcc sm_100a) first")
        L = ctypes.CDLL(LIB_PATH)
        for name, args in PROTOTYPES.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        L.dg_last_error.argtypes = []
        L.dg_last_error.restype = ctypes.c_char_p
        _lib = L
        return L


def check(rc):
    if rc == DG_OK:
        return
    msg = lib().dg_last_error().decode()
    if rc == DG_EINVAL:
        raise ValueError(msg)
    raise DgError(msg)


def call(name, *args):
    check(getattr(lib(), name)(*args))
