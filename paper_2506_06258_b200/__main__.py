"""`python -m paper_2506_06258_b200 ...`: the market-eq command line (cli.py)."""
import sys

from .cli import main

sys.exit(main())
