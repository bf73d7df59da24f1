"""The oracle and the CUDA path share no code (task rule ③; oracle/__init__.py).

Static checks over the sources, CPU only:
  * nothing in the product package (Python binding, C++/CUDA sources, the
    C-ABI header) names the oracle;
  * the oracle imports nothing of the product package;
  * the one module both sides use, `workloads`, imports neither;
  * bench.py reaches `oracle/` only from its cpu_baseline / reference legs.
"""
import ast
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2406_17565_b200")


def sources(top, exts):
    for d, _, files in os.walk(top):
        if "__pycache__" in d or os.sep + "_lib" in d:
            continue
        for f in files:
            if f.endswith(exts):
                yield os.path.join(d, f)


def imported_modules(path):
    tree = ast.parse(open(path).read(), path)
    mods = set()
    for node in ast.walk(tree):
        if isinstance(node, ast.Import):
            mods.update(a.name.split(".")[0] for a in node.names)
        elif isinstance(node, ast.ImportFrom) and node.module and node.level == 0:
            mods.add(node.module.split(".")[0])
    return mods


def test_product_never_names_the_oracle():
    files = list(sources(PKG, (".py", ".c", ".cpp", ".hpp", ".cu", ".cuh")))
    files += list(sources(os.path.join(ROOT, "include"), (".h",)))
    assert len(files) > 10
    for f in files:
        txt = open(f, errors="replace").read()
        assert not re.search(r"\boracle\b", txt, re.I), f
        if f.endswith(".py"):
            assert "oracle" not in imported_modules(f), f


def test_oracle_imports_no_product_code():
    for f in sources(os.path.join(ROOT, "oracle"), (".py",)):
        mods = imported_modules(f)
        assert "paper_2406_17565_b200" not in mods, f
        assert "torch" not in mods, f          # plain numpy / Python only


def test_shared_generators_import_neither_side():
    for f in sources(os.path.join(ROOT, "workloads"), (".py",)):
        mods = imported_modules(f)
        assert not mods & {"oracle", "paper_2406_17565_b200", "torch"}, f


def test_bench_uses_the_oracle_only_in_its_cpu_legs():
    tree = ast.parse(open(os.path.join(ROOT, "bench.py")).read())
    top = {a.name.split(".")[0] for n in tree.body if isinstance(n, ast.Import) for a in n.names}
    top |= {n.module.split(".")[0] for n in tree.body
            if isinstance(n, ast.ImportFrom) and n.module and n.level == 0}
    assert "oracle" not in top                 # no module-level import

    def imports_oracle(node):
        for n in ast.walk(node):
            if isinstance(n, ast.ImportFrom) and n.module and n.module.split(".")[0] == "oracle":
                return True
            if isinstance(n, ast.Import) and any(a.name.split(".")[0] == "oracle" for a in n.names):
                return True
        return False

    # top-level functions and classes that import it (a method counts as its class)
    users = {n.name for n in tree.body
             if isinstance(n, (ast.FunctionDef, ast.ClassDef)) and imports_oracle(n)}
    assert users, "bench.py's cpu_baseline leg should time the oracle"
    for name in users:
        assert re.search(r"cpu|reference|oracle", name, re.I), name


def test_missing_native_code_fails_loudly(tmp_path):
    """No CPU fallback: without the built library or binding the product
    path raises instead of computing anything."""
    import pytest
    from paper_2406_17565_b200 import mempool as M
    with pytest.raises(ImportError, match="no CPU fallback"):
        M.load_library(str(tmp_path / "libmempool.so"))
    with pytest.raises(ImportError, match="_mpfast binding not found"):
        M.load_fast(str(tmp_path))
