"""`python -m stencil_lab` — the reference CLI entry (reference __main__.py)."""
import sys

from paper_1810_04033_b200.cli import main

sys.exit(main())
