"""C-ABI library: builds, loads without a GPU, exports every symbol include/cpsel.h declares."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1104_2732_b200 import build
    build.build()
    import paper_1104_2732_b200 as cp
    return cp.load()


def header_functions():
    src = open(os.path.join(ROOT, "include", "cpsel.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b(cpsel_[a-z0-9_]+)\s*\(", src))


def test_header_and_binding_agree():
    import paper_1104_2732_b200 as cp
    assert header_functions() == set(cp.SYMBOLS)


def test_library_exports_every_declared_symbol(lib):
    import paper_1104_2732_b200 as cp
    out = subprocess.run(["nm", "-D", "--defined-only", cp.library_path()], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (cpsel_[a-z0-9_]+)$", out, flags=re.M))
    assert header_functions() <= exported
    for name in header_functions():
        assert hasattr(lib, name)


def test_library_is_sm100a(lib):
    import paper_1104_2732_b200 as cp
    out = subprocess.run(["cuobjdump", "--list-elf", cp.library_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_only_entry_points_without_gpu(lib):
    import paper_1104_2732_b200 as cp
    d = cp.default_config()
    assert d["direct_threshold"] == 1 << 17 and d["max_iters"] == 200 and d["record_trace"] == 1
    assert lib.cpsel_status_string(cp.ERANK) == b"rank out of range"
    assert lib.cpsel_select_kth(None, None, 0, 0, 1, None, None) == cp.EINVAL
    assert lib.cpsel_drive_host(None, 1, 0, 1, None, None, None, None, 0, None) == cp.EINVAL


def test_config_env_overrides(lib, monkeypatch):
    """CPSEL_ZCAP / CPSEL_MAXIT override the defaults; malformed values are ignored."""
    import paper_1104_2732_b200 as cp
    base = cp.default_config()
    monkeypatch.setenv("CPSEL_ZCAP", "4096")
    monkeypatch.setenv("CPSEL_MAXIT", "37")
    c = cp.default_config()
    assert c["z_cap"] == 4096 and c["max_iters"] == 37
    assert {k: v for k, v in c.items() if k not in ("z_cap", "max_iters")} == \
        {k: v for k, v in base.items() if k not in ("z_cap", "max_iters")}
    monkeypatch.setenv("CPSEL_ZCAP", "12x")
    monkeypatch.setenv("CPSEL_MAXIT", "0")
    c = cp.default_config()
    assert c["z_cap"] == base["z_cap"] and c["max_iters"] == base["max_iters"]
