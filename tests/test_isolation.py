"""Isolation of the oracle from the product path (task rule ③): the oracle is
test infrastructure, the CUDA path shares no code with it and never routes
through it, and the binding fails loudly when libvf is missing (no CPU
fallback).  Static checks over the sources plus one subprocess; CPU only."""
import ast
import os
import pathlib
import re
import subprocess
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
PKG = ROOT / "paper_2209_07632_b200"


def _imports(path):
    mods = set()
    for node in ast.walk(ast.parse(path.read_text())):
        if isinstance(node, ast.Import):
            mods.update(a.name.split(".")[0] for a in node.names)
        elif isinstance(node, ast.ImportFrom) and node.module and node.level == 0:
            mods.add(node.module.split(".")[0])
    return mods


def test_product_never_imports_or_links_the_oracle():
    for p in list(PKG.rglob("*.py")) + list((ROOT / "scenegen").rglob("*.py")):
        assert "oracle" not in _imports(p), p
    for p in list((PKG / "csrc").iterdir()) + list((ROOT / "include").iterdir()):
        if p.suffix in (".cu", ".cpp", ".h", ".cuh"):
            incs = re.findall(r'#\s*include\s*[<"]([^>"]+)[>"]', p.read_text())
            assert not any("oracle" in i for i in incs), (p, incs)
    assert "oracle" not in (PKG / "build.py").read_text()


def test_oracle_never_uses_the_product():
    for p in (ROOT / "oracle").rglob("*.py"):
        assert not _imports(p) & {"paper_2209_07632_b200", "bench"}, p
    for p in (ROOT / "oracle").rglob("*.c"):
        incs = re.findall(r'#\s*include\s*[<"]([^>"]+)[>"]', p.read_text())
        assert not any("vf" in i or "csrc" in i for i in incs), (p, incs)


def test_bench_uses_the_oracle_only_in_its_cpu_legs():
    """bench.py may run the oracle only in the reference arm and in the
    cpu_baseline legs (gated on --no-cpu-baseline)."""
    src = (ROOT / "bench.py").read_text()
    tree = ast.parse(src)
    parents = {}
    for node in ast.walk(tree):
        for ch in ast.iter_child_nodes(node):
            parents[ch] = node
    helpers = {"oracle_sample", "oracle_rows", "run_reference", "run_reference_terrain"}
    gated = {"run_gpu", "run_terrain"}
    for node in ast.walk(tree):
        uses = (isinstance(node, ast.Import) and any(a.name.split(".")[0] == "oracle" for a in node.names)) or \
               (isinstance(node, ast.Call) and isinstance(node.func, ast.Name) and node.func.id in helpers)
        if not uses:
            continue
        chain, p = [], node
        while p in parents:
            p = parents[p]
            chain.append(p)
        fn = next(c for c in chain if isinstance(c, ast.FunctionDef))
        if fn.name in helpers:
            continue
        assert fn.name in gated or fn.name == "main", (fn.name, node.lineno)
        if fn.name == "main":
            assert isinstance(node, ast.Call) and node.func.id == "run_reference"
            continue
        ifs = [ast.get_source_segment(src, c.test) for c in chain if isinstance(c, ast.If)]
        assert any("no_cpu_baseline" in t for t in ifs), (fn.name, node.lineno)


def test_binding_fails_loudly_without_the_library(tmp_path):
    env = dict(os.environ, VF_LIB=str(tmp_path / "missing_libvf.so"))
    r = subprocess.run([sys.executable, "-c", "import paper_2209_07632_b200 as vf; vf.lib()"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
    assert "missing_libvf.so" in r.stderr
