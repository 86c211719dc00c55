"""python -m paper_1912_03732_b200 <subcommand> ...  (the sbox-eval CLI)"""
import sys

from .cli import main

sys.exit(main())
