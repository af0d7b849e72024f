"""INTEGRATION.md's reference-side ctypes stub, executed as written.

The stub is the binding a maintainer would add to rbdgen (`rbdgen/b200.py`):
it loads a generated library with plain ctypes (none of this package's
binding code) and serves the reference's `interp.interpret` contract
(interp.py:54-86) from `rbd_run_host`.  The program object it is given only
needs the reference KernelProgram fields it reads (`input_map`,
`output_map`, `meta["algorithm"]`), which `program.build` mirrors.
"""
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden, rel_err
from paper_2109_06976_b200 import kernels, models, program


def _stub_source():
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    m = re.search(r"```python\n(# rbdgen/b200\.py.*?)```", text, re.S)
    assert m, "INTEGRATION.md lost its ctypes stub"
    return m.group(1)


def test_stub_compiles():
    compile(_stub_source(), "rbdgen/b200.py", "exec")


@pytest.mark.gpu
@pytest.mark.parametrize("name,alg", [("chain7", "gradFD"), ("quad12", "Minv"), ("humanoid30", "ID"),
                                      ("mixed5", "FD"), ("tree7", "gradID")])
def test_stub_matches_reference_fixtures(name, alg):
    ns = {}
    exec(_stub_source(), ns)
    m = models.load(name)
    prog, _, _ = program.build(m, alg)
    stub = ns["B200Program"](kernels.library_path(m), prog)
    g = golden(name)
    names = [n for n in ("q", "qd", "qdd", "tau") if n in prog.input_map]
    src = {"q": "q", "qd": "qd", "qdd": "u", "tau": "u"}
    for k in range(3):
        outs = stub.interpret({n: g[src[n]][k] for n in names})
        assert set(outs) == set(prog.output_map)
        for nm, v in outs.items():
            assert rel_err(v[None], g[f"{alg}.{nm}"][k:k + 1]) < 1e-9, (name, alg, nm)
