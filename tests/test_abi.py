"""CPU checks of the C ABI: the library loads, exports every symbol include/hz.h declares, the
host-side weight-table builder matches the oracle, argument errors are reported, and compute calls
fail loudly without a GPU (no CPU fallback)."""
import os
import re

import numpy as np
import pytest

from conftest import ROOT

hz = pytest.importorskip("paper_2108_08730_b200.hz", reason="libhz.so not built")


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "hz.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hz_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol():
    import ctypes
    lib = ctypes.CDLL(hz._LIBPATH)
    names = declared_symbols()
    assert len(names) >= 16
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(hz.EXPORTED)


def test_exports_debug_hooks():
    """include/hz_debug.h (test hooks, not the north-star ABI) is exported too."""
    import ctypes
    lib = ctypes.CDLL(hz._LIBPATH)
    src = re.sub(r"/\*.*?\*/", "", open(os.path.join(ROOT, "include", "hz_debug.h")).read(), flags=re.S)
    names = sorted(set(re.findall(r"\b(hz_[a-z_0-9]+)\s*\(", src)))
    assert names == ["hz_debug_plan_tiles"]
    for n in names:
        assert hasattr(lib, n), n


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", hz._LIBPATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_table_builder_matches_oracle(ga_table):
    """Table parity: libhz's block-tridiagonal long-double normal equations vs the
    oracle's dense lstsq on the stacked matrix: weights ≤ 1e-8 relative, dispersion ≤ 1e-12."""
    from oracle import dispersion as d
    T = hz.hz_build_weight_table(4.0, 40.0, 0.1, 1e-2)
    assert T.n_g == 361
    r5 = T.rows5()
    assert np.max(np.abs(r5 - ga_table.u5)) <= 1e-8 * np.max(np.abs(ga_table.u5))
    r7 = T.rows7()
    assert np.max(np.abs(r7 - ga_table.w7)) <= 1e-8
    for i in range(0, 361, 30):
        th, ph = d.angle_grid()
        a = d.vtilde(r7[i], ga_table.G[i], th, ph)
        b = d.vtilde(ga_table.w7[i], ga_table.G[i], th, ph)
        assert np.max(np.abs(a - b)) <= 1e-12


def test_host_table_builder_custom_angles():
    from oracle import weights
    th = np.deg2rad([0.0, 15.0, 30.0, 45.0])
    ph = np.deg2rad([0.0, 20.0, 40.0])
    T = hz.hz_build_weight_table(5.0, 9.0, 0.5, 0.1, th, ph)
    O = weights.build_adaptive_table(5.0, 9.0, 0.5, 0.1, *[np.repeat(th[None], 3, 0).ravel(), np.repeat(ph, 4)])
    assert np.max(np.abs(T.rows5() - O.u5)) <= 1e-9


def test_table_import_roundtrip_and_errors():
    rows = np.arange(15, dtype=float).reshape(3, 5) * 0.01
    T = hz.hz_table_import(4.0, 0.1, rows)
    assert np.array_equal(T.rows5(), rows)
    r7 = T.rows7()
    assert np.allclose(r7[:, :3].sum(1), 1) and np.allclose(r7[:, 3:].sum(1), 1)
    with pytest.raises(hz.HzError) as e:
        hz.hz_build_weight_table(4.0, 40.0, -0.1, 1e-2)
    assert e.value.status == -1
    with pytest.raises(hz.HzError) as e:
        hz.hz_build_weight_table(4.0, 40.0, 0.1, 0.0)      # rank-3 blocks, no regulariser (A14)
    assert e.value.status == -3
    with pytest.raises(hz.HzError):
        hz.hz_table_import(4.0, 0.1, np.array([[np.nan, 0, 0, 0, 0]]))


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(hz.HzError) as e:
        hz.hz_ctx_create(0)
    assert e.value.status in (-5, -1)


def test_c99_consumer(tmp_path, ga_table):
    """include/hz.h compiles as strict C99 and libhz links from C: tests/c/abi_consumer.c builds the
    default table through the ABI (host-only calls) and its row at G = 12 matches the oracle's."""
    import shutil
    import subprocess
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("no gcc")
    libdir = os.path.dirname(hz._LIBPATH)
    exe = str(tmp_path / "abi_consumer")
    subprocess.run([gcc, "-std=c99", "-pedantic", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "c", "abi_consumer.c"), "-L", libdir, "-lhz",
                    f"-Wl,-rpath,{libdir}", "-o", exe], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.splitlines()
    fields = {ln.split()[0]: ln.split()[1:] for ln in out}
    assert int(fields["n_g"][0]) == 361
    row = np.array([float(t) for t in fields["row80"]])
    assert np.max(np.abs(row - ga_table.u5[80])) <= 1e-8 * np.max(np.abs(ga_table.u5))
    w7 = np.array([float(t) for t in fields["w7_80"]])
    assert abs(w7[0] + w7[1] + w7[2] - 1.0) <= 1e-14 and abs(w7[3:].sum() - 1.0) <= 1e-14
    assert "import" in fields and int(fields["invalid"][0]) == -1
