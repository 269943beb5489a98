"""`python -m paper_2507_17087_b200 ...` (reference: __main__.py:1-8)."""

import sys

from .cli import main

sys.exit(main())
