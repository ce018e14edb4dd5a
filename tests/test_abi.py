"""C-ABI library: builds for sm_100a, loads, exports every symbol include/fmdp.h declares,
and fails loudly (no CPU fallback) when no sm_100 device is present."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fmdp.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fmdp_[a-z_0-9]+)\s*\(", src)))


def test_library_builds_and_exports_header_symbols():
    from paper_2008_03518_b200.build import build
    lib = build()
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (fmdp_\w+)", out))
    want = declared_symbols()
    assert len(want) >= 15
    missing = [s for s in want if s not in exported]
    assert not missing, f"declared but not exported: {missing}"
    from paper_2008_03518_b200 import fmdp
    assert set(fmdp.EXPORTS) <= exported
    L = fmdp.lib()
    for s in want:
        assert hasattr(L, s)


def test_sass_is_sm100a_and_uses_bulk_copy():
    from paper_2008_03518_b200.build import build
    lib = build()
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out
    assert "UBLKCP" in out            # cp.async.bulk (TMA bulk copy) staging of the plan rows
    assert "FMNMX" in out and "FFMA" in out


def test_strerror_and_no_cpu_fallback():
    from paper_2008_03518_b200 import fmdp
    L = fmdp.lib()
    assert L.fmdp_strerror(-8).decode() == "no sm_100 device"
    assert L.fmdp_strerror(0).decode() == "ok"
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import fmdp_synth as fs
    with pytest.raises(fmdp.FmdpError, match="no sm_100 device"):
        fmdp.FMDP(fs.Airspace(), torch_alloc=False)


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2008_03518_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", txt).lower().replace("no cpu fallback", ""), f


def test_abi_version_matches_the_header():
    """The binding's ABI version and its fmdp_airspace mirror follow include/fmdp.h."""
    import re
    from paper_2008_03518_b200 import fmdp
    hdr = open(os.path.join(ROOT, "include", "fmdp.h")).read()
    assert int(re.search(r"#define FMDP_ABI_VERSION (\d+)", hdr).group(1)) == fmdp.ABI_VERSION
    body = hdr[hdr.index("typedef struct fmdp_airspace"):hdr.index("} fmdp_airspace;")]
    names = re.findall(r"^\s+(?:const\s+)?[\w\s\*]+?\b(\w+)(?:\[\d+\])?\s*[;,]", body, re.M)
    fields = [f for f, _ in fmdp.Airspace._fields_]
    assert names[-1] == fields[-1] == "speed_max"
    assert "n_acc" in fields and "acc_units" in fields and fields[-4] == "n_acc"
    assert len(fields) >= 34


def test_pack_plans_layout():
    """pack_plans (binding-side marshalling for fmdp_add_plans): t0[P] int64, n[P] int32 and the
    states of all plans concatenated in order, [sum n][3] int32."""
    import numpy as np
    from paper_2008_03518_b200.fmdp import pack_plans
    plans = [(5, np.arange(6).reshape(2, 3)), (0, np.array([[7, 8, 9]])), (12, np.arange(9).reshape(3, 3) + 100)]
    t0, n, st = pack_plans(plans)
    assert t0.dtype == np.int64 and n.dtype == np.int32 and st.dtype == np.int32
    assert t0.tolist() == [5, 0, 12] and n.tolist() == [2, 1, 3]
    assert st.shape == (6, 3) and st.flags["C_CONTIGUOUS"]
    assert (st[:2] == plans[0][1]).all() and (st[2] == [7, 8, 9]).all() and (st[3:] == plans[2][1]).all()


def test_store_file_errors_without_gpu(tmp_path):
    """fmdp_save_plans / fmdp_load_plans argument errors need no device (include/fmdp.h)."""
    import ctypes as C
    from paper_2008_03518_b200 import fmdp as F
    L = F.lib()
    assert L.fmdp_strerror(-9).decode() == "plan-store file I/O error"
    assert L.fmdp_save_plans(None, str(tmp_path / "x").encode(), 0) == -1
    assert L.fmdp_load_plans(None, str(tmp_path / "x").encode(), None) == -1
