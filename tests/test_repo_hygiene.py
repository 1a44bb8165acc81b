"""Repository hygiene (CPU): no test module defines the same top-level name twice (a later
helper silently shadowing an earlier one turned a GPU test into a TypeError once)."""

import ast
import glob
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_no_duplicate_top_level_definitions():
    for path in sorted(glob.glob(os.path.join(ROOT, "tests", "*.py")) + [os.path.join(ROOT, "bench.py")]):
        tree = ast.parse(open(path).read())
        seen = {}
        for node in tree.body:
            if isinstance(node, (ast.FunctionDef, ast.ClassDef)):
                assert node.name not in seen, f"{os.path.basename(path)}: {node.name} defined at lines " \
                                              f"{seen[node.name]} and {node.lineno}"
                seen[node.name] = node.lineno
