"""python -m paper_2410_17375_b200 run|compare|trace <config.json> (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
