"""CPU checks of the drop-in boundary: librsgpu.so loads, exports exactly the
entry points include/rsgpu.h declares, maps errors like the reference
(common.hpp:24-39; TableConfig::validate embed_table.cpp:23-38) -- no kernel
is launched here."""
import ctypes as C
import os
import re
import subprocess

import pytest

import paper_2505_12663_b200 as P
from paper_2505_12663_b200 import _lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "rsgpu.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|uint64_t|const char\*)\s+(rs_\w+)\(", src, re.M)))


def test_header_symbols_exported():
    lib = L.lib()
    names = declared()
    assert len(names) >= 30
    nm = subprocess.run(["nm", "-D", "--defined-only", L.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (rs_\w+)", nm))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    for n in names:
        assert getattr(lib, n) is not None
    # every declared symbol has a ctypes signature in the binding
    assert not [n for n in names if n not in L._SIGS]


def test_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", L.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_status_strings_and_version():
    lib = L.lib()
    assert lib.rs_abi_version() == 1
    assert lib.rs_status_string(0) == b"ok"
    assert lib.rs_status_string(2) == b"invariant violated"


@pytest.mark.parametrize("field,value", [("capacity", 12), ("thread_groups", 3), ("max_load_factor", 1.0),
                                         ("max_load_factor", 0.0), ("embedding_dim", 0), ("chunk_rows", 0)])
def test_table_config_validation(field, value):
    cfg = P.TableConfig(capacity=8, embedding_dim=4, chunk_rows=4)
    setattr(cfg, field, value)
    with pytest.raises(P.ConfigError):
        P.EmbedTable(cfg)


def test_capacity_vs_groups():
    with pytest.raises(P.ConfigError):
        P.EmbedTable(P.TableConfig(capacity=4, thread_groups=4, embedding_dim=4))


def test_workload_generator_host_side(oracle):
    from paper_2505_12663_b200 import workload as W
    import numpy as np
    la, ia = W.generate(3, 200, 32.0, 500, 1.0, 1.1, [5000, 70])
    lb, ib = oracle.generate(3, 200, 32.0, 500, 1.0, 1.1, [5000, 70])
    np.testing.assert_array_equal(la, lb)
    np.testing.assert_array_equal(ia, ib)
    with pytest.raises(P.ConfigError):
        W.generate(3, 10, 600.0, 500, 1.0, 1.1, [10])
