"""``python -m paper_2110_08919_b200`` -> the command-line front end (cli.py)."""

import sys

from .cli import main

sys.exit(main())
