#!/bin/bash
# round 2g: full GPU suite (incl. slow) with AUTO = v12 for C4, smoke
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out/r2g; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
