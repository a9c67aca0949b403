"""python -m paper_2603_08982_b200 <run|sweep|verify> ...  (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
