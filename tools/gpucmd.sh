for cs in "C4 CS_E2LSH" "C4 CS_SRP" "C2 CS_E2LSH"; do set -- $cs; echo "$1 $2"; python tools/prof_hash.py --config $1 --scheme $2 --op hash --reps 3 | grep sketch; done
timeout 1500 python -m pytest tests -m gpu -x -q -k "C4 or C2 or C1 or edge or zero" > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/gpu_tests.log
