"""python -m paper_2602_20304_b200 <command>: see cli.py."""
import sys

from .cli import main

sys.exit(main())
