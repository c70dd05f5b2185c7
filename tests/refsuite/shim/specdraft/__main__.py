import sys

from paper_2411_05894_b200.cli import main

sys.exit(main())
