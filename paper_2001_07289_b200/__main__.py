"""``python -m paper_2001_07289_b200 run|preset|count ...`` (cli.py)."""
import sys

from .cli import main

sys.exit(main())
