"""The boundary used from plain C (examples/c_api_demo.c: no Python, no PyTorch):
compile it against include/srt3d.h + libsrt3d.so, run it on a ragged frame, and
compare its z / gradient / loss with the oracle (same tolerances as
tests/test_gpu_parity.py)."""
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_program_uses_the_abi(tmp_path, oracle_mod, inputs_mod):
    from paper_2203_00952_b200 import LIB_PATH

    exe = tmp_path / "c_api_demo"
    libdir = os.path.dirname(LIB_PATH)
    cmd = ["gcc", "-std=c11", "-O2", os.path.join(ROOT, "examples", "c_api_demo.c"), "-I", os.path.join(ROOT, "include"),
           "-I", "/usr/local/cuda/include", "-L", libdir, "-lsrt3d", "-L", "/usr/local/cuda/lib64", "-lcudart",
           f"-Wl,-rpath,{libdir}", "-Wl,-rpath,/usr/local/cuda/lib64", "-o", str(exe)]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    T, m, K, sigma = 4613, 10, 2, 5.0
    bins, offs = inputs_mod.random_csr(npix=321, T=T, max_n=900, seed=5)
    npix = offs.size - 1
    t, a = inputs_mod.random_theta(npix, K, T, seed=6)
    inp, out = tmp_path / "in.bin", tmp_path / "out.bin"
    with open(inp, "wb") as f:
        f.write(np.int64(npix).tobytes() + np.array([T, m, K], np.uint32).tobytes() + np.float32(sigma).tobytes()
                + np.uint64(offs[-1]).tobytes())
        f.write(offs.astype(np.uint32).tobytes() + bins.astype(np.uint16).tobytes())
        f.write(t.astype(np.float32).tobytes() + a.astype(np.float32).tobytes())
    r = subprocess.run([str(exe), str(inp), str(out)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    raw = np.fromfile(out, dtype=np.float32)
    z = raw[: npix * m * 2].reshape(npix, m, 2)
    zc = z[..., 0] + 1j * z[..., 1]
    gt = raw[npix * m * 2: npix * m * 2 + npix * K].reshape(npix, K)
    ga = raw[npix * m * 2 + npix * K: npix * m * 2 + 2 * npix * K].reshape(npix, K)
    loss = raw[npix * m * 2 + 2 * npix * K:]
    zo = oracle_mod.sketch(bins, offs, T, m)
    assert max(np.abs(zc.real - zo.real).max(), np.abs(zc.imag - zo.imag).max()) <= 1e-5
    go_t, go_a, Lo = oracle_mod.sketch_grad(zc.astype(np.complex64), t, a, sigma, T, m)
    for g, go in ((gt, go_t), (ga, go_a)):
        assert np.linalg.norm(g - go) <= 1e-4 * np.linalg.norm(go) + 1e-6
    assert np.abs(loss.sum() - Lo.sum()) <= 1e-4 * Lo.sum() + 1e-6
