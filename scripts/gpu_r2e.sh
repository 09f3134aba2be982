#!/bin/bash
# Re-entry check: full GPU suite, smoke, default bench line, c2 sweep trace.
set -u
O=gpurun_out/r2e${1:-}
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/status.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$?" >> $O/status.txt
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err
echo "bench rc=$?" >> $O/status.txt
timeout 600 python scripts/sweep_trace.py c2 > $O/trace_c2.txt 2>&1
echo "trace rc=$?" >> $O/status.txt
