"""The C-ABI library loads and exports every entry point include/rs_accel.h
declares; error plumbing works without a GPU (no compute calls here)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rs_accel.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rs_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ["rs_accel_create", "rs_accel_destroy", "rs_forward", "rs_pooled",
                 "rs_service_time", "rs_alloc_pinned", "rs_free_pinned", "rs_last_error"]:
        assert must in names


def test_library_exports_every_declared_symbol(rs):
    lib = C.CDLL(rs.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    assert sorted(rs.EXPORTED_SYMBOLS) == declared_functions()


def test_abi_version(rs):
    assert rs._lib.rs_abi_version() == 3


def test_errors_cross_the_abi_as_codes(rs):
    with pytest.raises(rs.UnknownModel):
        rs.builtin_model("ResNet50")
    assert "ResNet50" in rs._lib.rs_last_error().decode()
    with pytest.raises(rs.InvalidArgument):
        rs.work(rs.builtin_model("NCF"), 0)


def test_no_device_is_reported_not_crashed(rs):
    # In the CPU container there is no GPU: creating an accelerator must fail
    # with NoDevice (never silently fall back to a CPU path).
    if rs.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(rs.NoDevice):
        rs.Accelerator(rs.builtin_model("NCF"), rows_per_table=100)


def test_library_is_sm100a_only(rs):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", rs.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    for other in ("sm_80", "sm_90", "sm_120"):
        assert other + "." not in out


def test_tcgen05_and_tma_in_sass(rs):
    import subprocess
    sass = subprocess.run(["cuobjdump", "-sass", rs.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "UTCHMMA" in sass        # tcgen05.mma
    assert "UTMALDG" in sass        # TMA tensor loads
    assert "LDTM" in sass           # tcgen05.ld TMEM -> registers
    assert "UTCHMMA.2CTA" in sass   # tcgen05.mma.cta_group::2 (fc_tc2_kernel, CTA pairs)
    assert "UTMALDG.3D.2CTA" in sass  # TMA completing on the pair leader's barrier


def test_zipf_fill_query(rs):
    """rs_fill_query_zipf: deterministic, in range, the dense features of
    rs_fill_query, and the bounded power law's CDF at a few cut points."""
    import numpy as np
    spec = rs.builtin_model("DLRM-RMC1")
    rows, a = 1_000_000, 1.05
    d0, i0 = rs.fill_query(spec, rows, 3, 7, 200)
    d1, i1 = rs.fill_query(spec, rows, 3, 7, 200, zipf_alpha=a)
    d2, i2 = rs.fill_query(spec, rows, 3, 7, 200, zipf_alpha=a)
    assert np.array_equal(d0, d1) and np.array_equal(i1, i2)
    assert i1.min() >= 0 and i1.max() < rows
    n1 = rows + 1.0
    for K in (10, 1000, 100_000):
        want = ((K + 1.0) ** (1 - a) - 1) / (n1 ** (1 - a) - 1)
        assert abs(float(np.mean(i1 < K)) - want) < 0.01
    _, iu = rs.fill_query(spec, rows, 3, 7, 200, zipf_alpha=1.0)
    assert abs(float(np.mean(iu < 1000)) - np.log(1001) / np.log(n1)) < 0.01
    d, i = np.empty((2, spec.dense_input_dim), np.float32), np.empty(2 * 8 * 80, np.int64)
    assert rs._lib.rs_fill_query_zipf(C.byref(spec.to_c()), rows, 3, 7, 2, 0.0,
                                      d.ctypes.data, i.ctypes.data) == rs.InvalidArgument.code


def test_option_enums_match_the_header(rs):
    """rs_accel_set_option's option codes: the binding's constants are the
    header's enum values (RS_OPT_CTA_PAIRS included)."""
    src = open(HEADER).read()
    m = re.search(r"enum\s*\{\s*(RS_OPT_[^}]*)\}", src)
    vals = dict((k.strip(), int(v)) for k, v in re.findall(r"(RS_OPT_[A-Z_]+)\s*=\s*(\d+)", m.group(1)))
    assert vals == {"RS_OPT_MERGE_QUERIES": 1, "RS_OPT_STAGE_TIMING": 2, "RS_OPT_CTA_PAIRS": 3}
    assert (rs.OPT_MERGE_QUERIES, rs.OPT_STAGE_TIMING, rs.OPT_CTA_PAIRS) == (1, 2, 3)
