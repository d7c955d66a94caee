"""`python -m paper_2605_24514_b200 ...` (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
