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


def test_pdl_kernels_read_no_predecessor_data_before_the_wait():
    """In every kernel that waits on its PDL predecessor (griddepcontrol.wait = SASS ACQBULK),
    the loads scheduled before the wait are static data only: the uint8 support mask, the
    view table (64/128-bit .nc loads) and, in the 2D K3, D_L (one 32-bit .nc load per
    thread).  Any other load there is a predecessor output hoisted above the wait (DESIGN §6,
    launch chain; a hoisted x load in a K3 variant gave a 63 HU error)."""
    from paper_1402_4381_b200 import build
    import re
    import subprocess
    sass = subprocess.run(["cuobjdump", "-sass", build.LIB], capture_output=True, text=True).stdout
    n_pdl = 0
    for func in re.split(r"\n\s*Function : ", sass)[1:]:
        name = func.split("\n", 1)[0].strip()
        lines = func.split("\n")
        waits = [i for i, l in enumerate(lines) if "ACQBULK" in l]
        if not waits:
            continue
        n_pdl += 1
        f32_nc = 0
        for l in lines[:waits[0]]:
            if "LDG" not in l:
                continue
            if ".U8" in l or ".64.CONSTANT" in l or ".128.CONSTANT" in l:
                continue
            assert "LDG.E.CONSTANT" in l, (name, l.strip())   # a coherent load before the wait
            f32_nc += 1
        assert f32_nc <= (1 if "sqs_update2d" in name else 0), (name, f32_nc)
    assert n_pdl >= 4   # fwd2d tile + finalize, back2d, 2D K3


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
