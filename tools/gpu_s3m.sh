#!/bin/bash
# Full validation: -m gpu suite, smoke, default bench line.
set -u
O=gpurun_out/s3m; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu -x --timeout 600 > $O/pytest.txt 2>&1; echo "pytest exit $?" >> $O/pytest.txt
tail -3 $O/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke exit $?" >> $O/smoke.txt; tail -2 $O/smoke.txt
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; tail -1 $O/bench.json | cut -c1-600
