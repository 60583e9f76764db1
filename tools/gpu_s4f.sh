#!/bin/bash
# compute-sanitizer memcheck over the whole -m gpu suite except the full-size C2/C3 cases.
set -u
O=gpurun_out/s4f; mkdir -p $O
timeout 3300 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 30 \
  python -m pytest tests -q -m gpu -k "not c2_full and not c3_full" --timeout 3000 -p no:cacheprovider > $O/memcheck_all.txt 2>&1
echo "memcheck exit $?" >> $O/memcheck_all.txt
tail -5 $O/memcheck_all.txt
grep -c "Invalid __global__\|Invalid __shared__\|Address .* is out of bounds" $O/memcheck_all.txt
