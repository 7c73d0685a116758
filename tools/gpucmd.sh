timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -15 gpurun_out/gpu_tests.log
for cs in "C3 HCS_E2LSH" "C3 CS_SRP" "C5 HCS_E2LSH" "C5 HCS_SRP"; do set -- $cs; echo "== $1 $2"; python tools/prof_hash.py --config $1 --scheme $2 --op hash --reps 2 2>&1 | tail -2; done
