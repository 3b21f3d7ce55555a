"""``python -m paper_2603_11873_b200 {verify,bench,profile,gen-workload,calibrate} ...`` -- the
reference's ``lorafuse`` command (cli.py:619-660) on the GPU engine."""

import sys

from .harness import main

sys.exit(main())
