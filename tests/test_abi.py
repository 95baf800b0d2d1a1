"""C-ABI boundary checks that need no GPU: the library loads, exports every
entry point include/amppi_b200.h declares, its struct layouts match the ctypes
mirror, its defaults equal the reference's EnsembleConfig{} (via the oracle),
and without a CUDA device it fails loudly instead of computing on the CPU."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "amppi_b200.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int32_t|void\*?|const char\*)\s+(amppi_\w+)\s*\(", text, re.M)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("amppi_create", "amppi_destroy", "amppi_snapshot", "amppi_snapshot_f64", "amppi_plan",
                     "amppi_cycle_batch", "amppi_cycle_batch_device", "amppi_last_error"):
        assert required in names


def test_ctypes_mirror_binds_every_declared_function():
    from paper_2509_17340_b200 import _abi

    assert sorted(_abi.EXPORTS) == declared_functions()


def test_library_exports_every_declared_symbol(product_lib):
    out = subprocess.run(["nm", "-D", "--defined-only", product_lib._name], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\s[TW]\s+(amppi_\w+)", out))
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing


def test_struct_layouts_match_ctypes(tmp_path):
    from paper_2509_17340_b200 import _abi

    structs = {"amppi_config": _abi.Config, "amppi_state": _abi.State, "amppi_control": _abi.Control,
               "amppi_goal": _abi.Goal, "amppi_options": _abi.Options, "amppi_schedule": _abi.Schedule, "amppi_plan_result": _abi.PlanResult,
               "amppi_snapshot_view": _abi.SnapshotView, "amppi_batch_input": _abi.BatchInput,
               "amppi_batch_output": _abi.BatchOutput}
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void) {"]
    for cname, cls in structs.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for fname, _ in cls._fields_:
            cf = "lambda" if fname == "lambda_" else fname
            lines.append(f'printf("{cname}.{fname} %zu\\n", offsetof({cname}, {cf}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", "-o", str(exe), str(src)], check=True)
    got = dict(ln.split() for ln in subprocess.run([str(exe)], capture_output=True, text=True).stdout.splitlines())
    for cname, cls in structs.items():
        assert int(got[cname]) == ctypes.sizeof(cls), cname
        for fname, _ in cls._fields_:
            assert int(got[f"{cname}.{fname}"]) == getattr(cls, fname).offset, (cname, fname)


def test_defaults_match_reference_ensemble_config(product_lib, oracle):
    from paper_2509_17340_b200 import _abi

    c = _abi.Config()
    product_lib.amppi_config_default(ctypes.byref(c))
    o = oracle.config()
    assert ctypes.sizeof(c) == ctypes.sizeof(o)
    assert bytes(c) == bytes(o)  # every field, bit for bit (Table I)


def test_python_config_mirror_matches_c_defaults(product_lib):
    from paper_2509_17340_b200 import EnsembleConfig, _abi

    c = _abi.Config()
    product_lib.amppi_config_default(ctypes.byref(c))
    assert bytes(EnsembleConfig().to_c()) == bytes(c)


def _has_cuda():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_cuda(), reason="checks the no-GPU failure path")
def test_no_cpu_fallback_without_device(product_lib):
    from paper_2509_17340_b200 import AmppiError, Planner, _abi

    c = _abi.Config()
    product_lib.amppi_config_default(ctypes.byref(c))
    h = ctypes.c_void_p()
    rc = product_lib.amppi_create(ctypes.byref(c), None, ctypes.byref(h))
    assert rc == _abi.AMPPI_CUDA_ERROR and not h.value
    with pytest.raises(AmppiError):
        Planner()


def test_invalid_config_rejected(product_lib):
    from paper_2509_17340_b200 import _abi

    c = _abi.Config()
    product_lib.amppi_config_default(ctypes.byref(c))
    c.horizon = 0
    h = ctypes.c_void_p()
    assert product_lib.amppi_create(ctypes.byref(c), None, ctypes.byref(h)) == _abi.AMPPI_INVALID_ARGUMENT


def test_plan_result_records_are_built_on_access():
    """PlanResult.per_instance / anchors (planner._Records): a read-only
    sequence that builds each record once, on first access."""
    from paper_2509_17340_b200.planner import _Records

    made = []

    def make(i):
        made.append(i)
        return {"m": i}

    r = _Records(4, make)
    assert len(r) == 4 and made == []
    assert r[2] == {"m": 2} and r[-1] == {"m": 3} and made == [2, 3]
    assert r[2] is r[2] and made == [2, 3]  # cached
    assert [x["m"] for x in r] == [0, 1, 2, 3]
    assert [x["m"] for x in r[1:3]] == [1, 2]
    with pytest.raises(IndexError):
        r[4]
