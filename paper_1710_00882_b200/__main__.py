"""python -m paper_1710_00882_b200 <gen|run|bench|verify> ... (cli.py)."""
import sys

from .cli import main

sys.exit(main())
