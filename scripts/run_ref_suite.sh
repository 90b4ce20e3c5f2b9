#!/bin/bash
# Run the reference's own test suite (/root/reference/pkg/tests, 199 tests)
# against the B200 drop-in on a GPU box through the `ozemu` import alias
# (tests/ref_suite/).  The reference tests are copied into a git-ignored
# staging directory only for the duration of the gpurun call, then removed:
# reference sources never enter the repo history.
#   scripts/run_ref_suite.sh [tag]   -> profiles/<tag>_ref_suite.log
set -u
TAG=${1:-r02}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
STAGE=$ROOT/tests/ref_suite/_staged
rm -rf "$STAGE"
cp -r /root/reference/pkg/tests "$STAGE"
rm -rf "$STAGE/__pycache__"
/usr/local/graft/bin/gpurun --timeout 1500 -- \
  "timeout 1400 python -m pytest tests/ref_suite -m gpu -q -p no:cacheprovider -rs \
   > gpurun_out/${TAG}_ref_suite.log 2>&1; echo rc=\$? >> gpurun_out/${TAG}_ref_suite.log"
rc=$?
rm -rf "$STAGE"
mkdir -p "$ROOT/profiles"
cp "$ROOT/gpurun_out/${TAG}_ref_suite.log" "$ROOT/profiles/" 2>/dev/null
tail -5 "$ROOT/profiles/${TAG}_ref_suite.log" 2>/dev/null
exit $rc
