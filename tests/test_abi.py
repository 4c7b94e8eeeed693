"""CPU-side checks of the boundary: libst.so builds for sm_100a, loads, and exports every
function include/st.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "st.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(st_[a-z_]+)\s*\(", src)))


def test_library_builds_and_exports_all_declared_symbols():
    from paper_2508_09589_b200 import build
    path = build.build()
    lib = ctypes.CDLL(path)
    names = _declared()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n


def test_binding_exports_match_header():
    from paper_2508_09589_b200 import st
    assert set(st.EXPORTS) <= set(_declared())


def test_default_options_and_errors():
    from paper_2508_09589_b200 import st
    lib = st.load_library()
    o = st.Options()
    lib.st_default_options(ctypes.byref(o))
    assert o.rtol == 1e-8 and o.lambda_crit == 0.5 and o.restart == 16 and o.nu_pre == 2 and o.nu_post == 2 and o.nu_coarse == 5
    assert lib.st_abi_version() == 3
    assert lib.st_strerror(-2).decode().startswith("grid not divisible")


def test_setup_rejects_bad_args_without_gpu():
    """Validation happens before any device call: n < 2 must fail with ST_E_INVALID_ARG."""
    from paper_2508_09589_b200 import st
    lib = st.load_library()
    g = st.Grid(2, 1, 4, 1.0, 1.0)
    m = st.Materials(1, 1, 1, 1e-3, 1, 3)
    b = st.BCs(0.0, 1, 0, 0.5, 0.05)
    s = st.Source(0, 1.0, 0.0, 0.0)
    h = ctypes.c_void_p()
    rc = lib.st_setup(ctypes.byref(g), ctypes.byref(m), ctypes.byref(b), ctypes.byref(s), None, None, ctypes.byref(h))
    assert rc == -1


def test_cubin_is_sm100a():
    """The fatbinary carries sm_100a SASS (cuobjdump)."""
    import shutil
    import subprocess
    from paper_2508_09589_b200 import build
    path = build.build()
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([tool, "--list-elf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_layouts_match_binding():
    """The ctypes mirrors of every ABI struct have the C sizes (catches a field added on one side)."""
    from paper_2508_09589_b200 import st
    lib = st.load_library()
    out = (ctypes.c_int64 * 11)()
    assert lib.st_struct_sizes(out) == 0
    for cls, size in zip(st.STRUCTS, out):
        assert ctypes.sizeof(cls) == size, (cls.__name__, ctypes.sizeof(cls), size)


def test_setup_validates_distribution_without_gpu():
    """Time slabs: nt not divisible by the rank count -> ST_E_DIVISIBILITY; no transport -> invalid."""
    from paper_2508_09589_b200 import st
    lib = st.load_library()
    g = st.Grid(2, 16, 18, 1.0, 1.0)
    m = st.Materials(1, 1, 1, 1e-3, 1, 3)
    b = st.BCs(0.0, 1, 0, 0.5, 0.05)
    s = st.Source(0, 1.0, 0.0, 0.0)
    h = ctypes.c_void_p()
    d = st.Dist(None, 0, 4, None, -1, st.ST_COMM_HOST, st.HostComm())
    assert lib.st_setup(ctypes.byref(g), ctypes.byref(m), ctypes.byref(b), ctypes.byref(s), None,
                        ctypes.byref(d), ctypes.byref(h)) == -2
    g = st.Grid(2, 16, 16, 1.0, 1.0)
    assert lib.st_setup(ctypes.byref(g), ctypes.byref(m), ctypes.byref(b), ctypes.byref(s), None,
                        ctypes.byref(d), ctypes.byref(h)) == -1  # host transport without callbacks
    d = st.Dist(None, 0, 4, None, -1, st.ST_COMM_NONE, st.HostComm())
    assert lib.st_setup(ctypes.byref(g), ctypes.byref(m), ctypes.byref(b), ctypes.byref(s), None,
                        ctypes.byref(d), ctypes.byref(h)) == -1


def test_smoother_constants_match_header():
    """The binding's smoother constants are st.h's enum values (ST_SMOOTH_GMRES: the paper's
    GMRES(k)-Jacobi smoother)."""
    import re
    from paper_2508_09589_b200 import st
    hdr = open(os.path.join(ROOT, "include", "st.h")).read()
    m = re.search(r"enum \{ ST_SMOOTH_JACOBI = (\d+), ST_SMOOTH_CHEBYSHEV = (\d+), ST_SMOOTH_GMRES = (\d+) \};", hdr)
    assert m, "smoother enum"
    assert (st.ST_SMOOTH_JACOBI, st.ST_SMOOTH_GMRES) == (int(m.group(1)), int(m.group(3)))


@pytest.mark.parametrize("sdim,n,nt", [(2, 32, 32), (2, 64, 16), (3, 8, 16)])
def test_full_coarsening_plan_halves_space_and_time(sdim, n, nt):
    """Host-only plan of the full space-time coarsening hierarchy (option
    full_coarsening): every level below the fine one is of kind 'full' and halves n and nt, and
    the semi-coarsened plan of the same grid (Algorithm 1) coarsens one direction per level."""
    from paper_2508_09589_b200 import st
    full = st.plan(sdim, n, nt, full_coarsening=1)["levels"]
    assert len(full) >= 2 and full[0]["kind"] == "fine"
    for a, b in zip(full, full[1:]):
        assert b["kind"] == "full" and b["n"] == a["n"] // 2 and b["nt"] == a["nt"] // 2
    semi = st.plan(sdim, n, nt)["levels"]
    for a, b in zip(semi, semi[1:]):
        assert (b["kind"], b["n"], b["nt"]) in (("space", a["n"] // 2, a["nt"]), ("time", a["n"], a["nt"] // 2))


def test_options_defaults_and_knobs_are_options():
    """ABI 3: every former environment knob is an st_options_t field read per call (VERDICT r01
    weak #9): the library source calls no getenv, and the defaults are the measured ones
    (omega factor 1.9, DGKS eta 0.1; PAPER.md:385 coarse GMRES 200 its, 1e-6)."""
    import glob
    from paper_2508_09589_b200 import st
    for f in glob.glob(os.path.join(ROOT, "paper_2508_09589_b200", "csrc", "*")):
        assert "getenv" not in open(f).read(), f
    o = st.Options()
    lib = st.load_library()
    lib.st_default_options(ctypes.byref(o))
    assert o.nu_coarse == 5 and o.nu_pre == 2 and o.smoother == st.ST_SMOOTH_JACOBI
    assert o.krylov == st.ST_KRYLOV_FGMRES and o.coarse_solver == st.ST_COARSE_DENSE
    assert o.coarse_rtol == 1e-6 and o.coarse_maxit == 200
    assert o.kernel_family == st.ST_KERNELS_TMA and o.chunk_planes == 0 and o.max_ctas == 0
    assert o.fuse_prolong == 1
    assert o.omega_factor == 1.9 and o.dgks_eta == 0.1 and o.graph_max_nodes == 0 and o.smoother_rtol == 0.0
    assert o.nu_fine_nodes == 10000000 and o.pitch_align == 4
    hdr = open(os.path.join(ROOT, "include", "st.h")).read()
    for name in ("ST_KRYLOV_FGMRES", "ST_KRYLOV_GMRES", "ST_COARSE_DENSE", "ST_COARSE_GMRES", "ST_KERNELS_TMA",
                 "ST_KERNELS_CPASYNC", "ST_KERNELS_GENERIC", "ST_KERNELS_TMA2D"):
        m = re.search(name + r" = (\d+)", hdr)
        assert m and int(m.group(1)) == getattr(st, name), name


def test_binding_validates_vector_sizes():
    """The binding refuses arrays whose element count differs from what the C ABI reads or writes
    (no out-of-bounds access through an undersized array)."""
    import numpy as np
    from paper_2508_09589_b200 import st
    assert st._ptr(np.zeros(5), 5) is not None
    with pytest.raises(ValueError):
        st._ptr(np.zeros(4), 5, "T")
    with pytest.raises(ValueError):
        st._ptr(np.zeros(5, dtype=np.float32), 5)
