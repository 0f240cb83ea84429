import sys

from .cmdline import main

sys.exit(main())
