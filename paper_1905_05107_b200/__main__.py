"""``python -m paper_1905_05107_b200 ...`` -- the CLI (cli.py)."""

import sys

from .cli import main

sys.exit(main())
