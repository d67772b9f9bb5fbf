"""``python -m paper_2412_12734_b200 {fit,render,eval,sweep} ...`` (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
