"""``python -m podsketch`` on the drop-in's CLI."""

import sys

from paper_1905_05107_b200.cli import main

sys.exit(main())
