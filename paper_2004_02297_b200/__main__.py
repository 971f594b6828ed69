"""`python -m paper_2004_02297_b200 ...` runs the codec command line (cli.py)."""

from .cli import main

if __name__ == "__main__":
    raise SystemExit(main())
