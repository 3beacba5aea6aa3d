"""python -m paper_1910_02371_b200 gen | run | bench (cli.py)."""
from .cli import main

raise SystemExit(main())
