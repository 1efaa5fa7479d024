"""CPU checks of the C-ABI boundary: the library loads, exports every symbol that
include/ct_oslalm.h declares, and validates arguments before touching the device."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "ct_oslalm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ct_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_1402_4381_b200 import build, ctlib
    build.build()
    return ctlib.load()


def test_header_declares_the_north_star_calls():
    names = _declared()
    for n in ("ct_geom_create", "ct_fwd_proj", "ct_back_proj", "ct_sqs_denom", "ct_reg_grad", "ct_oslalm_iter",
              "ct_oslalm_run"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    from paper_1402_4381_b200 import ctlib
    for n in _declared():
        assert hasattr(lib, n), n
    assert set(_declared()) == set(ctlib.EXPORTS)


def test_build_info_and_counter(lib):
    from paper_1402_4381_b200 import ctlib
    assert "sm_100a" in ctlib.ct_build_info()
    assert ctlib.ct_kernel_launches() >= 0


def test_library_targets_sm100a_only():
    from paper_1402_4381_b200 import build
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", build.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


@pytest.mark.parametrize("bad,code", [
    (dict(dy=1.0), "CT_EINVAL"),            # non-square voxels
    (dict(nx=0), "CT_EINVAL"),
    (dict(dsd=500.0), "CT_EINVAL"),         # detector inside the orbit
    (dict(kind="cone_helical", pitch=0.0), "CT_EINVAL"),
    (dict(kind="cone_axial", nt=300), "CT_EUNSUPPORTED"),
    (dict(dx=60.0, dy=60.0, nx=8, ny=8), "CT_EUNSUPPORTED"),   # footprint wider than the window
])
def test_geometry_validation_before_device_use(lib, bad, code):
    from paper_1402_4381_b200 import ctlib
    from paper_1402_4381_b200 import inputs as I
    g = dict(I.config("c1").geom)
    g["nt"], g["nz"], g["dz"], g["dt"] = 4, 4, 1.0, 1.0
    g.update(bad)
    with pytest.raises(ctlib.CTError, match=code):
        ctlib.ct_geom_create(g)


def test_no_cpu_fallback_without_library(monkeypatch, tmp_path):
    from paper_1402_4381_b200 import ctlib
    monkeypatch.setattr(ctlib, "_lib", None)
    monkeypatch.setattr(ctlib, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(ctlib.CTError, match="not built"):
        ctlib.load()
