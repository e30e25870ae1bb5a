"""Static checks of the driver-facing scripts (no GPU): every name bench.py,
__graft_entry__.py and the binding reference is defined somewhere in scope."""
import builtins
import os
import symtable

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def undefined_names(path):
    src = open(path).read()
    top = symtable.symtable(src, path, "exec")
    module_names = {s.get_name() for s in top.get_symbols()}
    bad = []

    def walk(t, prefix):
        for s in t.get_symbols():
            if not s.is_referenced():
                continue
            if s.is_assigned() or s.is_parameter() or s.is_imported() or s.is_free() or s.is_nonlocal():
                continue
            name = s.get_name()
            if hasattr(builtins, name) or name in module_names:
                continue
            bad.append(f"{prefix}{t.get_name()}: {name}")
        for c in t.get_children():
            walk(c, prefix + t.get_name() + ".")

    walk(top, "")
    return bad


@pytest.mark.parametrize("rel", ["bench.py", "__graft_entry__.py", "paper_2503_01253_b200/nmspmm.py",
                                 "paper_2503_01253_b200/sharded.py", "paper_2503_01253_b200/synth.py",
                                 "oracle/oracle.py"])
def test_no_undefined_names(rel):
    assert undefined_names(os.path.join(ROOT, rel)) == []


def test_bench_cli_parses():
    import subprocess
    import sys
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--help"], capture_output=True, text=True)
    assert out.returncode == 0 and "--gpus" in out.stdout and "--impl" in out.stdout
