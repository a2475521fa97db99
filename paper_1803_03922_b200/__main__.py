"""``python -m paper_1803_03922_b200`` -> the delegate-bfs command line (cli.py)."""

import sys

from .cli import main

sys.exit(main())
