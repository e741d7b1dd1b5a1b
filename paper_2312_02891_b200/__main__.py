"""python -m paper_2312_02891_b200 {solve,gen,shifts,verify} (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
