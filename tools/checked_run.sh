#!/usr/bin/env bash
# The checked build (libwcgh_checked.so: -DWCGH_CHECKED device bounds checks,
# poisoned scratch) over the sanitizer cases and the GPU test files that
# cover them — in place of compute-sanitizer, which is closed on this pool.
# Plus a negative control proving the checks fire. Output: $OUT/checked_*.log
set -u
OUT=${OUT:-gpurun_out}
mkdir -p "$OUT"
export WCGH_CHECKED=1
timeout 900 python tools/sanitize_cases.py > "$OUT/checked_cases.log" 2>&1; echo "cases rc=$?"; tail -6 "$OUT/checked_cases.log"
timeout 1500 python -m pytest -q -x -m gpu tests/test_gpu_parity.py tests/test_gpu_peer_gather.py \
  tests/test_gpu_lut_objects.py tests/test_reference_suite_gpu.py tests/test_gpu_recon.py \
  "tests/test_gpu_configs.py::test_cfg2_full_plane" "tests/test_gpu_configs.py::test_front_end_bitexact_on_config_scenes" \
  > "$OUT/checked_pytest.log" 2>&1; echo "pytest rc=$?"; tail -3 "$OUT/checked_pytest.log"
WCGH_CHK_INJECT=segcount timeout 300 python -c "
import sys; sys.path.insert(0, '.')
from paper_2211_09938_b200 import scenes, _lib
from paper_2211_09938_b200.hologram import HologramJob, spec_for_scene
sc = scenes.make_scene(0)
try:
    HologramJob(spec_for_scene(sc))(sc.objects, sc.masks)
    print('NEGATIVE CONTROL FAILED: no check fired')
except _lib.IoError as e:
    print('negative control ok:', e)
" > "$OUT/checked_negative.log" 2>&1; echo "negative rc=$?"; cat "$OUT/checked_negative.log"
