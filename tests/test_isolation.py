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


CPU_ARMS = ("cpu_baseline", "run_reference")
ORACLE_HELPERS = ("oracle_wave_fields", "oracle_wave_step")   # bench.py helpers of the two CPU arms


def test_bench_imports_the_oracle_only_in_its_cpu_arms():
    for name in ("bench.py", "bench_config.py", "bench_suite.py", "bench_nodes.py"):
        tree = ast.parse(open(os.path.join(ROOT, name)).read())
        for fn, line in oracle_imports(tree):
            assert fn in CPU_ARMS + ORACLE_HELPERS, "%s:%d imports the oracle in %s" % (name, line, fn)
        # the helpers that touch the oracle are called from the CPU arms only
        for top in tree.body:
            if not isinstance(top, ast.FunctionDef):
                continue
            for n in ast.walk(top):
                if isinstance(n, ast.Call) and isinstance(n.func, ast.Name) and n.func.id in ORACLE_HELPERS:
                    assert top.name in CPU_ARMS + ORACLE_HELPERS, "%s: %s calls %s" % (name, top.name, n.func.id)


def test_native_sources_do_not_include_oracle_code():
    for dirpath, _, files in os.walk(os.path.join(PKG, "csrc")):
        for f in files:
            for line in open(os.path.join(dirpath, f)):
                if line.lstrip().startswith("#include"):
                    assert "oracle" not in line, (f, line)


def test_workloads_and_oracle_are_independent():
    """workloads/ (input generators + the program driver) holds none of the
    method's arithmetic and imports neither side; the oracle does not import
    workloads/ or the product."""
    def imported(tree):
        mods = set()
        for n in ast.walk(tree):
            if isinstance(n, ast.Import):
                mods |= {a.name.split(".")[0] for a in n.names}
            elif isinstance(n, ast.ImportFrom) and n.level == 0:
                mods.add((n.module or "").split(".")[0])
        return mods
    for f in os.listdir(os.path.join(ROOT, "workloads")):
        if f.endswith(".py"):
            mods = imported(ast.parse(open(os.path.join(ROOT, "workloads", f)).read()))
            assert not mods & {"oracle", "paper_2503_10516_b200"}, f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith(".py"):
            mods = imported(ast.parse(open(os.path.join(ROOT, "oracle", f)).read()))
            assert not mods & {"workloads", "paper_2503_10516_b200"}, f


def test_only_test_infrastructure_imports_the_oracle():
    """Outside oracle/ and tests/, only bench.py's CPU arms (checked above)
    and __graft_entry__.smoke() import the oracle: tools/ and workloads/ do not."""
    for d in ("tools", "workloads", "paper_2503_10516_b200"):
        for dirpath, _, files in os.walk(os.path.join(ROOT, d)):
            for f in files:
                if f.endswith(".py"):
                    p = os.path.join(dirpath, f)
                    assert oracle_imports(ast.parse(open(p).read())) == [], p
    tree = ast.parse(open(os.path.join(ROOT, "__graft_entry__.py")).read())
    for fn, line in oracle_imports(tree):
        assert fn == "smoke", line
