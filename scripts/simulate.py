"""Thin wrapper: the ncu-backed `simulate` report lives in the package
(paper_1012_2270_b200/simulate.py; python -m paper_1012_2270_b200.simulate)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1012_2270_b200.simulate import main  # noqa: E402

if __name__ == "__main__":
    main()
