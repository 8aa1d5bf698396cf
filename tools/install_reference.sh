#!/bin/bash
# Install the reference package (offline, from the wheelhouse) into
# baseline/_ref -- git-ignored, travels to the GPU box with gpurun -- and
# place the reference's own hot-path test modules beside it (baseline/_ref/
# ref_tests, also git-ignored) for tests/test_gpu_reference_suite.py.
# Needs /root/reference (this container only).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=${1:-/root/reference/pkg}
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"   # the build writes into the source tree; /root/reference is read-only
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" --upgrade "$TMP/pkg"
mkdir -p "$ROOT/baseline/_ref/ref_tests"
for f in conftest.py test_transfers.py test_substep.py test_collision.py test_weights.py test_materials.py test_oracle.py test_surfacing.py test_scene.py test_cli.py test_acceptance.py test_sampling.py test_sdf.py test_server.py; do
  cp "$SRC/tests/$f" "$ROOT/baseline/_ref/ref_tests/$f"
done
mkdir -p "$ROOT/baseline/_ref/ref_demos"
for f in 01_elastic_block.py 02_tool_contact.py 03_stiffness_sweep.py; do
  cp "$SRC/demos/$f" "$ROOT/baseline/_ref/ref_demos/$f"
done
rm -rf "$TMP"
echo "reference installed into $ROOT/baseline/_ref"
