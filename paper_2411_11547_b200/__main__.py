"""python -m paper_2411_11547_b200 <align|verify|bench|gen> ... (cli.py)."""
import sys

from .cli import main

sys.exit(main())
