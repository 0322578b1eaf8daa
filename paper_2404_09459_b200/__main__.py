"""``python -m paper_2404_09459_b200`` (reference ``rgsv/__main__.py``)."""

import sys

from .cli import main

sys.exit(main())
