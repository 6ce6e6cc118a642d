"""CPU: the C-ABI library loads, exports every symbol include/ychg_b200.h declares,
and fails loudly (no CPU fallback) when no device is present."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "ychg_b200.h")).read()
    return sorted(set(re.findall(r"YCHG_API\s+[\w\s\*]+?\b(ychg_\w+)\s*\(", text)))


def exported(path):
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True, check=True).stdout
    return {ln.split()[-1] for ln in out.splitlines() if " T " in ln}


def test_header_declares_entry_points():
    syms = declared_symbols()
    for must in ("ychg_cut_vertex_counts", "ychg_detect_boundary_columns", "ychg_scan_host",
                 "ychg_scan_device", "ychg_plan_create", "ychg_synth_device"):
        assert must in syms


def test_library_exports_every_declared_symbol(y):
    missing = set(declared_symbols()) - exported(y.LIB_PATH)
    assert not missing, missing


def test_python_binding_covers_header(y):
    assert set(declared_symbols()) == set(y.EXPORTED_SYMBOLS)


def test_cxx_dropin_exports_reference_api(y):
    out = subprocess.run(["nm", "-DC", "--defined-only", y.CXX_LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    assert "ychg::cut_vertex_counts(ychg::BinaryImage const&, ychg::ScanStrategy)" in out
    assert "ychg::detect_boundary_columns(std::span<int const, 18446744073709551615ul>)" in out
    assert "ychg::foreground_count(ychg::BinaryImage const&)" in out
    # the rest of runscan.cpp and pnm.cpp (link-time drop-in) + extensions
    for sym in ("ychg::column_runs(ychg::BinaryImage const&, int)",
                "ychg::build_profile(ychg::BinaryImage const&, ychg::ScanStrategy)",
                "ychg::load_pnm(std::span<unsigned char const, 18446744073709551615ul>, int)",
                "ychg::save_pnm(ychg::BinaryImage const&)",
                "ychg::scan(ychg::BinaryImage const&)",
                "ychg::scan_sharded(ychg::BinaryImage const&, int, std::span<int const, 18446744073709551615ul>)"):
        assert sym in out, sym


def test_abi_version(y):
    assert y._lib.ychg_abi_version() == 1


def test_validation_before_device(y):
    # argument validation (runscan.cpp:24-26) happens before any device work
    img = y.BinaryImage(3, 50)
    with pytest.raises(y.ValidationError):
        y.cut_vertex_counts(img, y.ScanStrategy.parallel(0))
    with pytest.raises(y.ValidationError):
        y.cut_vertex_counts(img, y.ScanStrategy.parallel(-2))


def test_no_cpu_fallback(y):
    if y.device_count() > 0:
        pytest.skip("device present")
    img = y.BinaryImage(8, 8)
    with pytest.raises(y.Error) as e:
        y.cut_vertex_counts(img)
    assert "no CPU fallback" in str(e.value)
    with pytest.raises(y.Error):
        y.scan(img)
    with pytest.raises(y.Error):
        y.detect_boundary_columns([1, 2, 3])
