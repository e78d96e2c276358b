"""python -m paper_1305_1422_b200 [OPTIONS] INPUT_FILE OUTPUT_PREFIX (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
