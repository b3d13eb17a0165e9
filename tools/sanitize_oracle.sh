#!/bin/bash
# The CPU oracle under AddressSanitizer + UndefinedBehaviorSanitizer: the oracle pin
# tests and a generated-stream self-check run against the -fsanitize=address,undefined build.
set -e
cd "$(dirname "$0")/.."
make -s -C oracle asan
export DISC_ORACLE_LIB=$PWD/oracle/libdisc_oracle_asan.so
export LD_PRELOAD=$(/usr/bin/gcc -print-file-name=libasan.so):$(/usr/bin/gcc -print-file-name=libubsan.so)
export ASAN_OPTIONS=detect_leaks=0:abort_on_error=1
export UBSAN_OPTIONS=print_stacktrace=1:halt_on_error=1
python -m pytest -q -p no:cacheprovider tests/test_oracle_pins.py tests/test_oracle_pins_angle_gate.py "$@"
