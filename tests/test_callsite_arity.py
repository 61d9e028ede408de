# SPDX-License-Identifier: Apache-2.0
"""CPU: every `*.call("gf_...", ...)` in the repo passes exactly the C-ABI's argument count
(catches signature drift before a GPU run)."""
import ast
import glob
import os

from paper_1902_06855_b200 import capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_call_sites_match_signatures():
    bad = []
    files = glob.glob(os.path.join(ROOT, "*.py")) + glob.glob(os.path.join(ROOT, "tests", "*.py")) + \
        glob.glob(os.path.join(ROOT, "paper_1902_06855_b200", "*.py")) + \
        glob.glob(os.path.join(ROOT, "scripts", "*.py"))
    for f in files:
        tree = ast.parse(open(f).read())
        for node in ast.walk(tree):
            if (isinstance(node, ast.Call) and isinstance(node.func, ast.Attribute)
                    and node.func.attr == "call" and node.args
                    and isinstance(node.args[0], ast.Constant)
                    and str(node.args[0].value).startswith("gf_")):
                name = node.args[0].value
                if any(isinstance(a, ast.Starred) for a in node.args):
                    continue
                n = len(node.args) - 1
                want = len(capi.SIGNATURES[name])
                if n != want:
                    bad.append(f"{os.path.relpath(f, ROOT)}:{node.lineno} {name}: {n} args, want {want}")
    assert not bad, "\n".join(bad)
