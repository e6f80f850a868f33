"""python -m paper_2509_07120_b200 <mask|attend|bench> ... (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
