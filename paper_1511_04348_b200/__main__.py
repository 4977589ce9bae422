"""``python -m paper_1511_04348_b200`` — the CLI (cli.py)."""

import sys

from .cli import main

sys.exit(main())
