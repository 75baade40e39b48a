"""python -m paper_1609_01567_b200 ... (cli.py)."""
import sys

from .cli import main

sys.exit(main())
