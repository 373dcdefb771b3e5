"""python -m paper_2511_01465_b200 {solve,bench,residuals} ... (cli_bench.py)."""
import sys

from .cli_bench import main

sys.exit(main())
