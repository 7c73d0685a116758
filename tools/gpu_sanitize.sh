# compute-sanitizer memcheck / racecheck / synccheck / initcheck over the library's
# kernels (tools/sanitize_driver.py: C1/C2-sized builds, lookups, knn, grouping corner
# cases, chunked sketch, HCS slab, dense tcgen05 GEMM).  Only lshb:: kernels are checked.
mkdir -p gpurun_out/sanitize
O=gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
F="--kernel-name kns=lshb --print-limit 50 --error-exitcode 9"
timeout 900 $CS --tool memcheck $F --leak-check full python tools/sanitize_driver.py > $O/memcheck.log 2>&1; echo "memcheck rc=$?" >> $O/memcheck.log
timeout 1500 $CS --tool racecheck $F --racecheck-report all python tools/sanitize_driver.py > $O/racecheck.log 2>&1; echo "racecheck rc=$?" >> $O/racecheck.log
timeout 900 $CS --tool synccheck $F python tools/sanitize_driver.py > $O/synccheck.log 2>&1; echo "synccheck rc=$?" >> $O/synccheck.log
timeout 900 $CS --tool initcheck $F python tools/sanitize_driver.py --quick > $O/initcheck.log 2>&1; echo "initcheck rc=$?" >> $O/initcheck.log
for f in $O/*.log; do echo "== $f"; grep -E "ERROR SUMMARY|rc=|^ok|Error|error" $f | sort | uniq -c | head -20; done
