"""``python -m paper_2309_10477_b200 {price,greeks,bench} ...`` (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
