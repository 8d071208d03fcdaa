"""``python -m paper_1901_06110_b200 <command> <config.ini>`` — the batch CLI (cli.py)."""

import sys

from .cli import main

sys.exit(main())
