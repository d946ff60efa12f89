"""Line counts and top-level definitions of the reference files this repo
cites (tests/test_citations.py checks every `<file>:<a>-<b>` citation
against them).  Run in the container that holds /root/reference:

    python tests/golden/make_ref_index.py > tests/golden/ref_index.json
"""

import ast
import json
from pathlib import Path

REF = Path("/root/reference")
FILES = {
    "batch.py": "pkg/src/fastsearch/batch.py",
    "direct.py": "pkg/src/fastsearch/direct.py",
    "partition.py": "pkg/src/fastsearch/partition.py",
    "binsearch.py": "pkg/src/fastsearch/binsearch.py",
    "eytzinger.py": "pkg/src/fastsearch/eytzinger.py",
    "errors.py": "pkg/src/fastsearch/errors.py",
    "bench/persist.py": "pkg/src/fastsearch/bench/persist.py",
    "bench/harness.py": "pkg/src/fastsearch/bench/harness.py",
    "bench/cli.py": "pkg/src/fastsearch/bench/cli.py",
    "bench/report.py": "pkg/src/fastsearch/bench/report.py",
    "test_direct.py": "pkg/tests/test_direct.py",
    "test_batch.py": "pkg/tests/test_batch.py",
    "test_acceptance.py": "pkg/tests/test_acceptance.py",
    "test_partition.py": "pkg/tests/test_partition.py",
    "test_binsearch.py": "pkg/tests/test_binsearch.py",
    "test_eytzinger.py": "pkg/tests/test_eytzinger.py",
    "test_bench.py": "pkg/tests/test_bench.py",
    "helpers.py": "pkg/tests/helpers.py",
    "PAPER.md": "PAPER.md",
    "SPEC.md": "SPEC.md",
}


def main():
    out = {}
    for key, rel in FILES.items():
        path = REF / rel
        text = path.read_text()
        entry = {"path": rel, "lines": len(text.splitlines()), "defs": []}
        if path.suffix == ".py":
            for node in ast.walk(ast.parse(text)):
                if isinstance(node, (ast.FunctionDef, ast.ClassDef)):
                    start = min([node.lineno] + [d.lineno for d in node.decorator_list])
                    entry["defs"].append([node.name, start, node.end_lineno])
            entry["defs"].sort(key=lambda d: d[1])
        out[key] = entry
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
