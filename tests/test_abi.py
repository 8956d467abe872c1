"""C-ABI boundary checks that need no GPU: libmpap.so loads, exports every
symbol include/mpap.h declares, and rejects invalid arguments before any
device work (status codes of include/mpap.h)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def mp():
    import build_ext
    build_ext.build()
    import paper_1705_02408_b200 as m
    return m


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "mpap.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mpap_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for s in ("mpap_build_roadmap", "mpap_search", "mpap_search_batch", "mpap_build_roadmap_batch"):
        assert s in syms


def test_library_exports_every_declared_symbol(mp):
    out = subprocess.run(["nm", "-D", "--defined-only", mp.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\sT\s(mpap_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    assert set(mp.EXPORTED_SYMBOLS) == set(declared_symbols())


def test_sm100a_code_only(mp):
    out = subprocess.run(["cuobjdump", "--list-elf", mp.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out


def test_status_strings(mp):
    assert mp.mpap_status_str(0) == "MPAP_OK"
    assert mp.mpap_status_str(3) == "MPAP_ERR_NO_FEASIBLE_PLAN"


def _params(mp, **over):
    base = dict(control_weight=1.0, nominal_speed=1.0, dt=0.02, collision_dt=0.1, n_f=12.0, fov_cos_half=0.7,
                max_range=1.0, mlp_gain=0.0, v_ref=1.0, w_ref=1.0)
    base.update(over)
    return mp.make_params(2, 0, 0, 0, [0, 0], [1, 1], None, **base)


@pytest.mark.parametrize("bad", [
    dict(r=0.0), dict(r=float("nan")), dict(dt=0.0), dict(fov_cos_half=0.0), dict(fov_cos_half=1.5),
    dict(n_f=-1.0), dict(stride=1), dict(nan_sample=True), dict(bad_box=True), dict(n=0),
])
def test_build_rejects_invalid_arguments(mp, bad):
    samples = np.array([[0.1, 0.1], [0.5, 0.5]])
    if bad.get("nan_sample"):
        samples[1, 0] = np.nan
    obst = np.array([[0.3, 0.3, 0.2, 0.4]]) if bad.get("bad_box") else np.array([[0.3, 0.3, 0.4, 0.4]])
    feats = np.array([[0.9, 0.9]])
    over = {k: v for k, v in bad.items() if k in ("dt", "fov_cos_half", "n_f")}
    prm = _params(mp, **over)
    r = bad.get("r", 0.5)
    lib = mp.lib()
    out = C.c_void_p()
    n = C.c_int32(bad.get("n", 2))
    no = C.c_int32(1)
    nf = C.c_int32(1)
    s = lib.mpap_build_roadmap_batch(1, samples.ctypes.data, C.byref(n), bad.get("stride", 2), obst.ctypes.data,
                                     C.byref(no), feats.ctypes.data, C.byref(nf), r, C.byref(prm), 0, None,
                                     C.byref(out))
    assert s == mp.MPAP_ERR_INVALID_ARGUMENT
    assert out.value is None
    assert len(lib.mpap_last_error()) > 0


def test_search_rejects_null_roadmap(mp):
    lib = mp.lib()
    g = mp.mpap_goal()
    res = mp.mpap_result()
    path = np.zeros(4, np.int32)
    s = lib.mpap_search(None, 0, 0, C.byref(g), 1.0, 0.5, path.ctypes.data_as(C.POINTER(C.c_int32)), 4,
                        C.byref(res), None, 0, None)
    assert s == mp.MPAP_ERR_INVALID_ARGUMENT


def test_import_rejects_bad_csr(mp):
    with pytest.raises(mp.MpapError):
        mp.mpap_roadmap_import(np.zeros((2, 2)), [0, 1, 0], [1], [0.5], [0.0], [0.0], 1.0)   # decreasing row_ptr
    with pytest.raises(mp.MpapError):
        mp.mpap_roadmap_import(np.zeros((2, 2)), [0, 1, 1], [5], [0.5], [0.0], [0.0], 1.0)   # dst out of range


def test_product_path_does_not_import_oracle():
    """The product package never loads the oracle (it is test infrastructure)."""
    pkg = os.path.join(ROOT, "paper_1705_02408_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "liboracle" not in txt, f


def test_struct_layouts_match_header(mp, tmp_path):
    """The ctypes mirrors of mpap_params / mpap_goal / mpap_result / mpap_wave
    have the C header's sizes and field offsets (compiled here with gcc)."""
    structs = {"mpap_params": mp.mpap_params, "mpap_goal": mp.mpap_goal, "mpap_result": mp.mpap_result,
               "mpap_wave": mp.mpap_wave, "mpap_mc_params": mp.mpap_mc_params}
    dtypes = {"mpap_mc_result": mp.MC_RESULT_DTYPE, "mpap_result_np": mp.RESULT_DTYPE}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "mpap.h"', "int main(void) {"]
    for name, cls in structs.items():
        lines.append(f'  printf("{name} size %zu\\n", sizeof({name}));')
        for f in cls._fields_:
            lines.append(f'  printf("{name} {f[0]} %zu\\n", offsetof({name}, {f[0]}));')
    for name, dt in dtypes.items():
        cname = name.replace("_np", "")
        lines.append(f'  printf("{name} size %zu\\n", sizeof({cname}));')
        for f in dt.names:
            lines.append(f'  printf("{name} {f} %zu\\n", offsetof({cname}, {f}));')
    lines.append("  return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split("\n")
    for ln in out:
        if not ln:
            continue
        name, field, val = ln.split()
        if name in dtypes:
            dt = dtypes[name]
            want = dt.itemsize if field == "size" else dt.fields[field][1]
        else:
            cls = structs[name]
            want = C.sizeof(cls) if field == "size" else getattr(cls, field).offset
        assert int(val) == want, (name, field, val, want)


@pytest.mark.parametrize("nfeat,nobst", [(65536, 0), (3000, 0), (1000, 1200)])
def test_build_rejects_oversized_environment(mp, nfeat, nobst):
    """Per-environment limits (uint16 visible counts; the edge kernels' shared
    working set 32 (F (d + 1) + 2 d O) + 8192 <= 227 KB) are validated before
    any device work -- never wrapped or truncated."""
    samples = np.array([[0.1, 0.1], [0.5, 0.5]])
    feats = np.full((nfeat, 2), 0.9)
    obst = np.tile(np.array([[0.3, 0.3, 0.4, 0.4]]), (max(nobst, 1), 1))
    prm = _params(mp)
    lib = mp.lib()
    out = C.c_void_p()
    n, no, nf = C.c_int32(2), C.c_int32(nobst), C.c_int32(nfeat)
    s = lib.mpap_build_roadmap_batch(1, samples.ctypes.data, C.byref(n), 2, obst.ctypes.data, C.byref(no),
                                     feats.ctypes.data, C.byref(nf), 0.5, C.byref(prm), 0, None, C.byref(out))
    assert s == mp.MPAP_ERR_INVALID_ARGUMENT
    assert out.value is None
    assert b"feature" in lib.mpap_last_error() or b"shared" in lib.mpap_last_error()


def test_grid_search_kernel_keeps_its_registers(mp):
    """k_search_grid is pinned to one block per SM (__launch_bounds__(512, 1)):
    squeezed to 64 registers with local-memory spills it ran single queries
    3x slower (profiles/r02/search_regression_ab.jsonl)."""
    out = subprocess.run(["cuobjdump", "-res-usage", mp.LIB_PATH], capture_output=True, text=True).stdout
    regs = re.findall(r"k_search_gridILb[01]E\S*:\s*\n\s*REG:(\d+)", out)
    assert len(regs) == 2 and all(int(r) > 64 for r in regs), regs
