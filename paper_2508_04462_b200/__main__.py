"""python -m paper_2508_04462_b200 run|ablate ... (see cli.py)"""
import sys

from .cli import main

sys.exit(main())
