"""`python -m paper_2507_07788_b200 ...` runs the cholqr-compatible CLI."""

import sys

from .cli import main

sys.exit(main())
