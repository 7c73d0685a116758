# Device bounds-checked build (LSHB_CHECKS, build.py --variant checked) over the sanitizer
# driver workloads and the GPU parity suite: every guarded index write that fails prints
# "LSHB_DCHECK file:line" (compute-sanitizer is closed on this GPU pool).
mkdir -p gpurun_out/checked
O=gpurun_out/checked
export LSH_LIB_VARIANT=checked
timeout 900 python tools/sanitize_driver.py > $O/driver.log 2>&1; echo "driver rc=$?" >> $O/driver.log
timeout 2400 python -m pytest tests -q -m gpu -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for f in $O/driver.log $O/pytest.log; do echo "== $f: $(grep -c LSHB_DCHECK $f) failed checks"; tail -2 $f; done
