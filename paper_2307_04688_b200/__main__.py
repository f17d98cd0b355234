"""``python -m paper_2307_04688_b200 {solve,simulate,compare,bench-blocks} ...`` (see cli.py)."""

import sys

from .cli import main

if __name__ == "__main__":
    sys.exit(main())
