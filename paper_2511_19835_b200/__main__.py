"""``python -m paper_2511_19835_b200 gen|run|sweep`` (see ``cli``)."""

import sys

from .cli import main

sys.exit(main())
