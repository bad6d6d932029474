"""``python -m paper_1807_02037_b200 <command>``: see cli.py."""

import sys

from .cli import main

sys.exit(main())
