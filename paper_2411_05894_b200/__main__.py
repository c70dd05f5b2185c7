"""``python -m paper_2411_05894_b200 <subcommand>`` (the ``specdraft`` CLI)."""

import sys

from .cli import main

sys.exit(main())
