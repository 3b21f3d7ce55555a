#!/bin/bash
mkdir -p gpurun_out
AF_UMMA=1 timeout 600 python -m pytest tests/ -q -m gpu --timeout 120 --timeout-method=thread 2>&1 | tail -8
AF_UMMA=1 timeout 120 python __graft_entry__.py smoke 2>&1 | tail -2
