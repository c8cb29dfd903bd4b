#!/usr/bin/env bash
# Stage the reference's own test suite and package for tests/reference_suite
# (run HERE, where /root/reference exists; both outputs are git-ignored and
# travel to the GPU box with the gpurun snapshot):
#   baseline/_ref/                   the reference package, pip-installed from a
#                                    /tmp copy (provides fedheat.oracle / cli /
#                                    bench / scenario for the acceptance tests)
#   tests/reference_suite/vendored/  pkg/tests/*.py, unmodified
# tests/reference_suite/conftest.py points the `fedheat` imports of those
# files at this repo's GPU facade (paper_1909_05098_b200).
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
REF="${REF:-/root/reference/pkg}"
[ -d "$REF" ] || { echo "no reference at $REF" >&2; exit 1; }
if [ ! -d "$ROOT/baseline/_ref/fedheat" ]; then
  rm -rf /tmp/fh_refcopy && cp -r "$REF" /tmp/fh_refcopy
  python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse --no-deps \
    --target "$ROOT/baseline/_ref" /tmp/fh_refcopy >/dev/null
fi
DST="$ROOT/tests/reference_suite/vendored"
mkdir -p "$DST"
for f in oracles.py test_solver.py test_acceptance.py test_element.py test_material.py test_mesh.py \
         test_meshgen.py test_precompute.py test_vtkio.py; do
  cp "$REF/tests/$f" "$DST/$f"
done
echo "vendored $(ls "$DST" | wc -l) files into $DST; reference package in $ROOT/baseline/_ref"
