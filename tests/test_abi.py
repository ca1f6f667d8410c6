"""CPU checks of the C-ABI library: it loads and exports every symbol the
public header declares (no device calls)."""

import ctypes
import os
import re

from conftest import ROOT


def header_symbols():
    src = open(os.path.join(ROOT, "include", "sparsewire_b200.h")).read()
    return sorted(set(re.findall(r"SW_API\s+[\w\s\*]+?\b(sw_\w+)\s*\(", src)))


def test_header_declares_symbols():
    syms = header_symbols()
    assert "sw_deepr_eliminate" in syms and "sw_deepr_form_pass" in syms
    assert len(syms) >= 15


def test_library_loads_and_exports_header(tmp_path):
    from paper_2510_19764_b200.build import LIB, build
    if not os.path.exists(LIB):
        build()
    lib = ctypes.CDLL(LIB)
    missing = [s for s in header_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.sw_abi_version() == 1


def test_python_signatures_cover_header():
    from paper_2510_19764_b200 import _lib
    declared = set(header_symbols()) - {"sw_last_error", "sw_launch_count",
                                         "sw_propagate_workspace_bytes"}
    assert declared == set(_lib.SIGNATURES), declared ^ set(_lib.SIGNATURES)


def test_host_fold_key_matches_oracle():
    from oracle import rng as O
    from paper_2510_19764_b200 import rng as R
    for parts in [(1,), (3, "host", 1, 2, 0), ("x" * 17, -5), (2**64 + 3,)]:
        assert R.fold_key(*parts) == O.fold_key(*parts)
    r = R.CounterRng(5, "n")
    o = O.Stream.of(5, "n")
    assert [r.uniform_int(700) for _ in range(50)] == [o.uniform_int(700) for _ in range(50)]


def test_block_struct_matches_header():
    """_lib.EpropBlock mirrors sw_eprop_block_t: the step-array width is the
    header's SW_EPROP_MAX_BLOCK."""
    import re
    from paper_2510_19764_b200 import _lib
    src = open(os.path.join(ROOT, "include", "sparsewire_b200.h")).read()
    n = int(re.search(r"#define SW_EPROP_MAX_BLOCK (\d+)", src).group(1))
    assert _lib.MAX_BLOCK == n
    assert len(_lib.EpropBlock().psi) == n and len(_lib.EpropBlock().pre_trace[1]) == n


def test_integration_doc_lists_every_export():
    """INTEGRATION.md maps every C-ABI entry the header declares to the
    reference interface it replaces."""
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    missing = [s for s in header_symbols() if s not in doc]
    assert not missing, missing
