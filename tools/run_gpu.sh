#!/bin/bash
# Build here (abort on failure), then run a command on the GPU box.
#   tools/run_gpu.sh TIMEOUT 'command'
set -e
cd "$(dirname "$0")/.."
python -c "from paper_1703_01325_b200 import build; build.build()"
python - <<'PY'
import os, glob
so = "paper_1703_01325_b200/_lib/libbiluk.so"
t = os.path.getmtime(so)
src = glob.glob("paper_1703_01325_b200/csrc/*") + ["include/biluk.h"]
stale = [f for f in src if os.path.getmtime(f) > t]
assert not stale, f"stale library: {stale}"
PY
/usr/local/graft/bin/gpurun --timeout "$1" -- "$2"
