"""``python -m paper_2503_03456_b200 ...``: the harness command line (harness.py)."""

import sys

from .harness import main

sys.exit(main())
