"""The oracle is test infrastructure: the product package never imports it,
and bench.py imports it only inside its cpu_baseline / reference-arm
functions (the boundary rule of DESIGN §1)."""

import ast
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2503_10516_b200")


def oracle_imports(tree):
    """(enclosing top-level function or None, line) of every oracle import."""
    out = []

    def visit(node, fn):
        for ch in ast.iter_child_nodes(node):
            f = fn
            if isinstance(ch, (ast.FunctionDef, ast.AsyncFunctionDef)) and fn is None:
                f = ch.name
            if isinstance(ch, ast.Import) and any(a.name.split(".")[0] == "oracle" for a in ch.names):
                out.append((f, ch.lineno))
            if isinstance(ch, ast.ImportFrom) and (ch.module or "").split(".")[0] == "oracle":
                out.append((f, ch.lineno))
            visit(ch, f)
    visit(tree, None)
    return out


def test_product_package_never_imports_the_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith(".py"):
                p = os.path.join(dirpath, f)
                assert oracle_imports(ast.parse(open(p).read())) == [], p


def test_bench_imports_the_oracle_only_in_its_cpu_arms():
    for name in ("bench.py", "bench_config.py", "bench_suite.py", "bench_nodes.py"):
        tree = ast.parse(open(os.path.join(ROOT, name)).read())
        for fn, line in oracle_imports(tree):
            assert fn in ("cpu_baseline", "run_reference"), "%s:%d imports the oracle in %s" % (name, line, fn)


def test_native_sources_do_not_include_oracle_code():
    for dirpath, _, files in os.walk(os.path.join(PKG, "csrc")):
        for f in files:
            for line in open(os.path.join(dirpath, f)):
                if line.lstrip().startswith("#include"):
                    assert "oracle" not in line, (f, line)
