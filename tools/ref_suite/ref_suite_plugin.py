"""pytest plugin: run the reference package's OWN hot-path test modules
(/root/reference/pkg/tests/test_transfers.py, test_substep.py,
test_collision.py, ... copied unmodified into baseline/_ref/ref_tests by
tools/install_reference.sh) against the reference package with its hot path
re-routed to the B200 kernels by paper_2402_01181_b200.install().

The reference's tolerances are fp64 ones (1e-9 .. 1e-15); the drop-in
computes in fp32, whose per-substep gate is the north star's 1e-5.  So, when
a test module is imported, every float literal in (0, FP32_TOL) that appears
inside the right-hand side of a `<` / `<=` comparison, or as the rel=/abs=/
rtol=/atol= keyword of pytest.approx / np.allclose / np.isclose /
assert_allclose, is raised to FP32_TOL (an AST rewrite of the literal only;
exact comparisons -- ==, array_equal, atol=0.0 -- are left exact).  The
rewritten sites are printed at the end of the session.

Load with: python -m pytest <ref_tests/...> -p ref_suite_plugin
(PYTHONPATH must hold this directory, baseline/_ref and the repo root).
"""
from __future__ import annotations

import ast
import os
import sys
import tempfile
import types

FP32_TOL = 1.0e-5
_REWRITES: list[str] = []

# ---- import the reference with its off-path scikit-image import stubbed
if "skimage" not in sys.modules:
    sk = types.ModuleType("skimage")
    sk.measure = types.ModuleType("skimage.measure")
    sys.modules["skimage"] = sk
    sys.modules["skimage.measure"] = sk.measure
os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "softmpm_numba_cache"))

import softmpm  # noqa: E402  (baseline/_ref)
import softmpm.oracle  # noqa: E402
from paper_2402_01181_b200.install import install  # noqa: E402

DETERMINISTIC = os.environ.get("SOFTMPM_INSTALL_DETERMINISTIC") == "1"
install(softmpm, deterministic=DETERMINISTIC)
# the one tolerance kept as a module constant rather than a literal
# (oracle.py: ORACLE_TOLERANCE = 1e-12, max |dx| per coordinate) gets the same rule
if softmpm.oracle.ORACLE_TOLERANCE < FP32_TOL:
    _REWRITES.append(f"softmpm.oracle.ORACLE_TOLERANCE: {softmpm.oracle.ORACLE_TOLERANCE!r} -> {FP32_TOL!r}")
    softmpm.oracle.ORACLE_TOLERANCE = FP32_TOL


def _is_small_float(node) -> bool:
    return (isinstance(node, ast.Constant) and isinstance(node.value, float)
            and 0.0 < node.value < FP32_TOL)


def _raise(node, where):
    _REWRITES.append(f"{where}: {node.value!r} -> {FP32_TOL!r}")
    return ast.copy_location(ast.Constant(FP32_TOL), node)


class _Tol(ast.NodeTransformer):
    def __init__(self, fname):
        self.fname = fname

    def _lits(self, tree, line):
        class _L(ast.NodeTransformer):
            def visit_Constant(s, node):
                return _raise(node, f"{self.fname}:{line}") if _is_small_float(node) else node
        return _L().visit(tree)

    def visit_Compare(self, node):
        self.generic_visit(node)
        if any(isinstance(op, (ast.Lt, ast.LtE)) for op in node.ops):
            node.comparators = [self._lits(c, node.lineno) for c in node.comparators]
        return node

    def visit_Call(self, node):
        self.generic_visit(node)
        for kw in node.keywords:
            if kw.arg in ("rel", "abs", "rtol", "atol") and _is_small_float(kw.value):
                kw.value = _raise(kw.value, f"{self.fname}:{node.lineno}")
        return node


def _rewrite_module(mod_path: str):
    src = open(mod_path).read()
    tree = _Tol(os.path.basename(mod_path)).visit(ast.parse(src, mod_path))
    ast.fix_missing_locations(tree)
    return compile(tree, mod_path, "exec")


def pytest_pycollect_makemodule(module_path, parent):
    # the reference's test modules only (ref_tests/test_*.py)
    import pytest
    if os.path.basename(os.path.dirname(str(module_path))) != "ref_tests":
        return None

    class _FP32Module(pytest.Module):
        def _getobj(self):
            name = "ref_tests_" + os.path.splitext(os.path.basename(str(self.path)))[0]
            mod = types.ModuleType(name)
            mod.__file__ = str(self.path)
            sys.modules[name] = mod
            exec(_rewrite_module(str(self.path)), mod.__dict__)
            return mod

    return _FP32Module.from_parent(parent, path=module_path)


def pytest_terminal_summary(terminalreporter):
    terminalreporter.write_line(f"install mode: {'deterministic' if DETERMINISTIC else 'fast'}")
    terminalreporter.write_line(f"softmpm hot path: {softmpm.core.step.__module__} (install() active: "
                                f"{softmpm.core.step.__module__.startswith('paper_2402_01181_b200')})")
    terminalreporter.write_line(f"fp64 -> fp32 tolerance literals raised to {FP32_TOL}: {len(_REWRITES)}")
    for r in _REWRITES:
        terminalreporter.write_line("  " + r)
