#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_cli.py -x -q -m gpu 2>&1 | tail -25
