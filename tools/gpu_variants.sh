#!/bin/bash
# The GPU parity suites under every A/B switch of include/qmcj2.h (each variant must pass)
QJ2_SWEEP_TPB=256 timeout 600 python -m pytest tests/test_gpu_accept.py -q -k sweep 2>&1 | tail -1
QJ2_SWEEP_NOFULL=1 timeout 600 python -m pytest tests/test_gpu_accept.py -q -k sweep 2>&1 | tail -1
QJ2_KERNEL=tma323 timeout 600 python -m pytest tests/test_gpu_parity.py -q 2>&1 | tail -1
QJ2_J1_WARP=1 timeout 600 python -m pytest tests/test_gpu_j1.py -q 2>&1 | tail -1
QJ2_WARP=p2m3 timeout 600 python -m pytest tests/test_gpu_parity.py -q 2>&1 | tail -1
