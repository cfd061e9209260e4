#!/bin/bash
python tools/prof_kernels.py 2>&1
timeout 600 python -m pytest -x -q tests/test_gpu_transformer.py 2>&1 | tail -15
