"""CPU: the C-ABI library loads without a GPU and exports every symbol the public headers
declare; argument errors surface as the reference's exception types."""
import ctypes as C
import os
import re

import pytest

from paper_1609_04809_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pf_[a-z0-9_]+)\s*\(", text)))


@pytest.mark.parametrize("header", ["pf_gpu.h", "pf_setup.h", "pf_fe.h"])
def test_every_declared_symbol_is_exported(header):
    lib = _lib.lib()
    names = declared(header)
    assert names, header
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) <= set(_lib.EXPORTS) | {"pf_setup_last_error", "pf_fe_last_error"}


def test_python_export_list_matches_headers():
    assert sorted(_lib.EXPORTS) == sorted(set(declared("pf_gpu.h")) | set(declared("pf_setup.h"))
                                         | (set(declared("pf_fe.h")) - {"pf_fe_last_error"}))


def test_version_names_the_target():
    assert b"sm_100a" in _lib.lib().pf_version()


def test_sm100a_only_in_the_fatbinary():
    """The library carries sm_100a SASS and nothing else (no PTX fallback)."""
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_argument_errors_without_a_device():
    lib = _lib.lib()
    h = C.c_void_p()
    assert lib.pf_hierarchy_create(0, 0, 1, 0, 1, C.byref(h)) == _lib.PF_ERR_INVALID_ARGUMENT
    assert b"at least one level" in lib.pf_last_error()
    assert lib.pf_hierarchy_create(0, 2, 2, 0, 3, C.byref(h)) == _lib.PF_ERR_INVALID_ARGUMENT
    with pytest.raises(_lib.InvalidArgument):
        _lib.check(lib.pf_spmv(None, 0, None, None))
    cfg = _lib.MultigridConfig()
    lib.pf_default_multigrid_config(C.byref(cfg))
    # multigrid.hpp:53-62 defaults
    assert (cfg.cycles, cfg.pre_smooth, cfg.post_smooth, cfg.coarse_tol, cfg.coarse_max_iter,
            cfg.outer_tol, cfg.outer_max_cycles) == (1, 3, 3, 1e-12, 20000, 1e-9, 100)
    assert (cfg.smoother.kind, cfg.smoother.sweeps, cfg.smoother.damping) == (1, 3, 0.8)


def test_option_table_without_a_device():
    """pf_option_names lists every tuning option with its kind; the knobs DESIGN.md §6
    documents are all there (build options shape the device layout, launch options steer
    the enqueue)."""
    from paper_1609_04809_b200 import gmg
    names = gmg.option_names()
    assert names["value_index"] == "build" and names["bottom_stage"] == "build"
    assert names["wide_max_rows"] == "launch" and names["solve_mode_host"] == "launch"
    assert set(names.values()) == {"build", "launch"}
    design = open(os.path.join(ROOT, "DESIGN.md")).read()
    for n in names:
        assert n in design, f"option {n} undocumented in DESIGN.md"
    with pytest.raises(_lib.InvalidArgument):
        _lib.check(_lib.lib().pf_option_names(C.create_string_buffer(8), 8))
