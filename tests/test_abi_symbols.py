"""CPU-only checks of the boundary: libsrt3d.so loads (no GPU needed to dlopen)
and exports every entry point include/srt3d.h declares; the binding exposes
the same names.  No compute call is made here."""
import ctypes
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "srt3d.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(srt3d_[a-z0-9_]+)\s*\(", src)))


def _lib_path():
    from paper_2203_00952_b200 import LIB_PATH, build

    if not os.path.exists(LIB_PATH):
        build.build()
    return LIB_PATH


def test_header_declares_expected_entry_points():
    names = _declared()
    for required in ("srt3d_sketch", "srt3d_expected_sketch", "srt3d_sketch_grad", "srt3d_last_error"):
        assert required in names


def test_library_exports_every_declared_symbol():
    path = _lib_path()
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (srt3d_[a-z0-9_]+)$", out, flags=re.M))
    missing = [n for n in _declared() if n not in exported]
    assert not missing, f"declared but not exported: {missing}"
    lib = ctypes.CDLL(path)
    for n in _declared():
        assert getattr(lib, n) is not None


def test_binding_names_match_abi():
    import paper_2203_00952_b200 as p

    for n in _declared():
        if n in ("srt3d_version", "srt3d_last_error"):
            continue
        assert hasattr(p, n), f"binding lacks {n}"
    assert set(p.EXPORTS) == set(_declared())


def test_library_is_sm100a_and_no_fallback():
    """The .so carries sm_100a SASS only; the binding refuses to run without it."""
    path = _lib_path()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    import paper_2203_00952_b200 as p

    try:
        p.load_library(os.path.join(ROOT, "does_not_exist.so"))
    except ImportError:
        pass
    else:  # pragma: no cover
        raise AssertionError("missing library must raise")


def test_version_and_last_error_callable_without_gpu():
    import paper_2203_00952_b200 as p

    lib = p.load_library()
    assert lib.srt3d_version() >= 100
    assert isinstance(lib.srt3d_last_error(), bytes)


def test_host_validation_without_gpu():
    """Argument validation runs on the host before any CUDA call: invalid calls fail with
    the documented codes even on a machine with no GPU."""
    import paper_2203_00952_b200 as p

    lib = p.load_library()
    dummy = ctypes.c_void_p(16)
    assert lib.srt3d_sketch(dummy, dummy, 4, 1, 1, dummy, None) == -1        # T < 2
    assert lib.srt3d_sketch(dummy, dummy, 4, 100, 100, dummy, None) == -1    # m >= T
    assert lib.srt3d_sketch(dummy, dummy, 4, 1000, 65, dummy, None) == -3    # m > MAX_M
    assert lib.srt3d_sketch(dummy, dummy, -1, 100, 3, dummy, None) == -1     # npix < 0
    assert lib.srt3d_sketch(None, None, 0, 100, 3, None, None) == 0          # npix = 0 no-op
    assert lib.srt3d_sketch(dummy, None, 4, 100, 3, dummy, None) == -2       # NULL offsets
    assert lib.srt3d_sketch(None, dummy, 4, 100, 3, dummy, None) == -2       # NULL bins (photon count unknown)
    assert lib.srt3d_sketch_ex(None, dummy, 4, 100, 3, dummy, 0, 0, 0, None) == -2
    assert lib.srt3d_sketch_ex(None, dummy, 4, 100, 3, dummy, 5, 1, 4, None) == -2
    assert lib.srt3d_sketch(dummy, ctypes.c_void_p(18), 4, 100, 3, dummy, None) == -5  # misaligned offsets
    assert lib.srt3d_sketch_grad(dummy, dummy, dummy, 4, 9, ctypes.c_float(1.0), 100, 3, dummy, dummy, None, None) == -3
    assert lib.srt3d_sketch_grad(dummy, dummy, dummy, 4, 2, ctypes.c_float(float("inf")), 100, 3, dummy, dummy,
                                 None, None) == -1
    assert lib.srt3d_descent_update(dummy, dummy, dummy, dummy, 4, 2, ctypes.c_float(1.0), 100, 3,
                                    ctypes.c_float(-1.0), None) == -1
    assert b"eta" in lib.srt3d_last_error()


def test_sketch_plan_regimes_without_gpu():
    """srt3d_sketch_plan (host only) picks the measured-fastest regime per BASELINE config
    (DESIGN.md §5.7): the tensor-core path below 3 T photons per pixel at T <= 8192, the bin-count
    path above it, the routed direct path where T > 8192 (it then fits up to 12000)."""
    import paper_2203_00952_b200 as p

    plan = lambda npix, T, m, tot: p.srt3d_sketch_plan(npix, T, m, tot)[0]  # noqa: E731
    assert plan(262144, 8192, 32, 262121072) == p.PATH_TENSOR              # C5
    assert plan(1024, 1024, 4, 51200) == p.PATH_TENSOR                      # C1
    assert plan(19881, 4613, 10, 19881 * 1000) == p.PATH_TENSOR            # C2
    assert plan(65536, 2500, 20, 65536 * 10000) == p.PATH_BINCOUNT         # C3: 4 T per pixel
    assert plan(4096, 4096, 10, 4096 * 10000) == p.PATH_TENSOR              # C4@1e4: 2.4 T
    assert plan(4096, 4096, 10, 4096 * 100000) == p.PATH_BINCOUNT           # C4@1e5
    assert plan(4096, 8192, 10, 4096 * (3 * 8192) - 1) == p.PATH_TENSOR     # just below 3 T
    assert plan(4096, 8192, 10, 4096 * (3 * 8192)) == p.PATH_BINCOUNT
    assert plan(4096, 8196, 32, 4096 * 1000) == p.PATH_ROUTED               # T > 8192
