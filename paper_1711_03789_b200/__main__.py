"""``python -m paper_1711_03789_b200`` (reference maxwelldd/__main__.py)."""

import sys

from .cli import main

sys.exit(main())
