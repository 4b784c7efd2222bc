#!/bin/bash
# Build every extension; exit non-zero if nvcc reported an error (guards GPU runs).
cd "$(dirname "$0")/.." || exit 1
python -c "import __graft_entry__ as g; g.build()" > /tmp/rwb_build.log 2>&1
rc=$?
if [ $rc -ne 0 ] || grep -q "error" /tmp/rwb_build.log; then
  grep -E "error" /tmp/rwb_build.log | head -5
  exit 1
fi
exit 0
