"""Regenerate bench.PLAN_BYTES (whole-job algorithmic HBM bytes of this
build's plan for every bench config) in place after a planner change."""
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2604_12256_b200 as qs  # noqa: E402


def main():
    out = {}
    for w in ("qft", "rzz", "diag", "qaoa", "rand"):
        for n, r in ((30, 1), (31, 2), (32, 4), (33, 8)):
            g = bench.make_circuit(w, n)
            p = qs.plan_json(n, g, n_ranks=r, basis=bench.BASIS_X % (1 << n))
            out["%s%d" % (w, n)] = p["stats"]["bytes_hbm"] * r
    lines = []
    for w in ("qft", "rzz", "diag", "qaoa", "rand"):
        lines.append("    " + " ".join('"%s%d": %d,' % (w, n, out["%s%d" % (w, n)]) for n in (30, 31, 32, 33)))
    body = "PLAN_BYTES = {\n" + "\n".join(lines) + "\n}"
    path = os.path.join(ROOT, "bench.py")
    s = open(path).read()
    s2 = re.sub(r"PLAN_BYTES = \{\n.*?\n\}", body, s, count=1, flags=re.S)
    open(path, "w").write(s2)
    print(body)


if __name__ == "__main__":
    main()
