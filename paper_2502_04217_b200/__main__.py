"""``python -m paper_2502_04217_b200`` = the reference's ``fftlasso`` CLI on the B200 path."""

import sys

from .cli import main

sys.exit(main())
