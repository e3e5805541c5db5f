#!/bin/bash
timeout 400 python -m pytest tests -q -m gpu -x -s 2>&1 | grep -E "rel logit|err|passed|failed|Error|assert" > gpurun_out/g4_tests.log
