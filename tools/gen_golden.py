"""Write tests/golden/ fixtures.  Calls only oracle/ (never the CUDA path).

k_int8.csv : K_e^INT8 (24×48) from the exact-rational derivation in oracle/element.py
             (integers in [-128,127] per L110).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.element import k_int8  # noqa: E402


def main():
    out = os.path.join(ROOT, "tests", "golden", "k_int8.csv")
    K = k_int8()
    with open(out, "w") as fh:
        fh.write("# K_e^INT8 = (K_e^kappa | Kbar_e^G), 24 rows x 48 cols; PAPER.md L95-L103, L110\n")
        fh.write("# written by tools/gen_golden.py from oracle/element.py (exact rationals)\n")
        for row in K:
            fh.write(",".join(str(x) for x in row) + "\n")
    print("wrote", out)


if __name__ == "__main__":
    main()
