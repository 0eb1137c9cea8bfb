"""``python -m paper_2101_07088_b200 {tune,solve,bd} ...`` (the reference CLI)."""
import sys

from .cli import main

sys.exit(main())
