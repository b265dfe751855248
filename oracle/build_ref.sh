#!/bin/bash
# Build the REAL reference (swarmfilter, Python + its Cython kernel) into oracle/_ref/ -- test and
# baseline infrastructure only (tests/, smoke() and bench.py's CPU legs may import it; the product never does).
# Source: /root/reference/pkg, read-only: it is copied to a scratch directory under /tmp and installed from there
# with the image's offline toolchain (no index, no build isolation, no dependency resolution).  Output goes only
# to oracle/_ref/ (git-ignored, not gpurun-ignored: it travels to the GPU box like the repo's own .so files).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF=${SGSF_REFERENCE:-/root/reference/pkg}
OUT="$HERE/_ref"
if [ ! -d "$REF" ]; then echo "build_ref: $REF absent (GPU box): keeping the prebuilt $OUT"; exit 0; fi
SCRATCH=$(mktemp -d /tmp/sgsf_refbuild.XXXXXX)
trap 'rm -rf "$SCRATCH"' EXIT
cp -r "$REF" "$SCRATCH/pkg"
rm -rf "$OUT"
python -m pip install --quiet --no-index --no-build-isolation --no-deps --target "$OUT" "$SCRATCH/pkg"
PYTHONPATH="$OUT" python -c "import swarmfilter; from swarmfilter import kernels; b = kernels.active_backend(); \
assert b == 'compiled', b; print('oracle/_ref: swarmfilter', swarmfilter.__file__, 'backend', b)"
