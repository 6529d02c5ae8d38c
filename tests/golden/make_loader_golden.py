"""Golden cases for the graph file parsers (graphs.py:126-247): every input
below is run through the reference's load_edge_list in the build container
(PYTHONPATH=/root/reference/pkg/src) and its result -- the canonical edge
list, or the GraphFormatError message and line -- is recorded in
loader_cases.json.  The inputs are written for this test, not taken from the
reference's tests.  Usage: python tests/golden/make_loader_golden.py"""
import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

CASES = [
    # edge lists
    ("edgelist", False, "5\n0 1 1.0\n1 2 2.5\n3 4 0.25\n"),
    ("edgelist", False, "# header comment\n\n4   # node count\n2 0 3\n  1 3 1e-3 # trailing\n"),
    ("edgelist", False, "4\r\n0 1 1\r\n2 3 2\r\n"),
    ("edgelist", False, "3\n0 1 1\n1 0 2\n"),
    ("edgelist", True, "3\n0 1 1\n1 0 2\n2 1 0.5\n1 2 4\n"),
    ("edgelist", False, "6\n"),
    ("edgelist", False, ""),
    ("edgelist", False, "# only comments\n\n"),
    ("edgelist", False, "3 4\n0 1 1\n"),
    ("edgelist", False, "x\n"),
    ("edgelist", False, "0\n"),
    ("edgelist", False, "-2\n"),
    ("edgelist", False, "3\n0 1\n"),
    ("edgelist", False, "3\n0 1 1 1\n"),
    ("edgelist", False, "3\n0 one 1\n"),
    ("edgelist", False, "3\n0 1.0 1\n"),
    ("edgelist", False, "3\n0 3 1\n"),
    ("edgelist", False, "3\n-1 2 1\n"),
    ("edgelist", False, "3\n1 1 1\n"),
    ("edgelist", False, "3\n0 1 0\n"),
    ("edgelist", False, "3\n0 1 -2.5\n"),
    ("edgelist", False, "3\n0 1 nan\n"),
    ("edgelist", False, "3\n0 1 inf\n"),
    ("edgelist", False, "3\n0 1 abc\n"),
    ("edgelist", False, "4\n0 1 1\n2 3 1\n0 2 1\n3 2 5\n"),
    ("edgelist", False, "3\n+0 2 7\n"),
    ("edgelist", False, "3\n0 1 1e-320\n"),
    ("edgelist", False, "3\n0 1 '1'\n"),
    # Matrix Market
    ("mtx", False, "%%MatrixMarket matrix coordinate real symmetric\n% c\n3 3 4\n1 1 2\n2 1 -1\n3 2 -4.5\n3 3 7\n"),
    ("mtx", False, "%%MatrixMarket matrix coordinate real general\n3 3 2\n1 2 -1\n2 1 -1\n"),
    ("mtx", True, "%%MatrixMarket matrix coordinate real general\n3 3 3\n1 2 -1\n2 1 -3\n3 1 2\n"),
    ("mtx", False, "%%MatrixMarket matrix coordinate pattern symmetric\n4 4 3\n2 1\n3 2\n4 3\n"),
    ("mtx", False, "%%MatrixMarket matrix coordinate integer general\n2 2 1\n1 2 5\n"),
    ("mtx", False, "%%MatrixMarket MATRIX Coordinate REAL Symmetric\n2 2 1\n2 1 1.5\n"),
    ("mtx", False, "%%MatrixMarket matrix coordinate real symmetric\n5 5 0\n"),
    ("mtx", False, ""),
    ("mtx", False, "%MatrixMarket matrix coordinate real symmetric\n2 2 1\n2 1 1\n"),
    ("mtx", False, "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n"),
    ("mtx", False, "%%MatrixMarket matrix coordinate complex general\n2 2 1\n1 2 1 0\n"),
    ("mtx", False, "%%MatrixMarket matrix coordinate real hermitian\n2 2 1\n1 2 1\n"),
    ("mtx", False, "%%MatrixMarket matrix coordinate real\n2 2 1\n1 2 1\n"),
    ("mtx", False, "%%MatrixMarket matrix coordinate real general\n2 2\n"),
    ("mtx", False, "%%MatrixMarket matrix coordinate real general\n2 x 1\n"),
    ("mtx", False, "%%MatrixMarket matrix coordinate real general\n2 3 1\n"),
    ("mtx", False, "%%MatrixMarket matrix coordinate real general\n0 0 0\n"),
    ("mtx", False, "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2\n"),
    ("mtx", False, "%%MatrixMarket matrix coordinate pattern general\n2 2 1\n1 2 3\n"),
    ("mtx", False, "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 b 3\n"),
    ("mtx", False, "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 3 3\n"),
    ("mtx", False, "%%MatrixMarket matrix coordinate real general\n2 2 1\n0 1 3\n"),
    ("mtx", False, "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 0\n"),
    ("mtx", False, "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 2 3\n"),
    ("mtx", False, "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 3\n2 1 3\n"),
    ("mtx", False, "%%MatrixMarket matrix coordinate real general\n"),
    ("mtx", False, "%%MatrixMarket matrix coordinate real general\n3 3 2\n1 2 2\n2 1 -3\n"),
]


def main():
    from lapeig.graphs import GraphFormatError, load_edge_list
    out = []
    for fmt, sym, text in CASES:
        rec = {"format": fmt, "symmetrize": sym, "text": text}
        try:
            g = load_edge_list(text.encode(), format=fmt, symmetrize=sym)
            rec["n"] = g.n_nodes
            rec["i"] = g.i.tolist()
            rec["j"] = g.j.tolist()
            rec["w"] = [float(x).hex() for x in g.w]
        except GraphFormatError as e:
            rec["error"] = str(e)
            rec["line"] = e.line
        out.append(rec)
    (HERE / "loader_cases.json").write_text(json.dumps(out, indent=1))
    print(len(out), "cases")


if __name__ == "__main__":
    main()
