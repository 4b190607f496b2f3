#!/bin/bash
# Full-tree A/B: materialise git revision REV (default HEAD) with its own libprnet.so under
# .ab_prev/ (git-ignored, shipped to the GPU box by gpurun), so builds with different
# Python bindings / ABI versions can be timed side by side by tools/ab2.sh.
set -eu
REV=${1:-HEAD}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
rm -rf "$ROOT/.ab_prev"; mkdir -p "$ROOT/.ab_prev"
git -C "$ROOT" archive "$REV" | tar -x -C "$ROOT/.ab_prev"
cp "$ROOT/MEASURED_PEAKS.json" "$ROOT/.ab_prev/" 2>/dev/null || true
(cd "$ROOT/.ab_prev" && python -c "from paper_2404_02445_b200 import _build; _build.build(force=True)")
echo "prev tree: $REV"
