"""``python -m paper_2601_11437_b200 ...``: the maternmle command line on the GPU engine."""

import sys

from .cli import main

sys.exit(main())
