#!/bin/bash
# The GPU test suite and tools/sanitize_cases.py against the checked build of the library
# (libstc_checked.so: STC_CHECK bounds / protocol assertions compiled into every kernel).
# compute-sanitizer is closed on this GPU pool, so this is the memory-safety evidence.
# Logs -> gpurun_out/checked_*.txt
mkdir -p gpurun_out
export STC_LIBRARY=$PWD/paper_2405_16883_b200/libstc_checked.so
python - <<'PY' > gpurun_out/checked_lib.txt
import paper_2405_16883_b200._abi as a; print("library:", a._LIB_PATH)
PY
python tools/sanitize_cases.py > gpurun_out/checked_cases.txt 2>&1; echo "cases rc=$?"
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/checked_tests.txt 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/checked_tests.txt
timeout 120 python tools/checked_negative.py > gpurun_out/checked_negative.txt 2>&1; echo "negative rc=$?"
grep -E "STC_CHECK|expected|NO CHECK" gpurun_out/checked_negative.txt | head -3
