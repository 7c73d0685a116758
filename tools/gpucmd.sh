for cs in "C4 CS_E2LSH" "C4 CS_SRP" "C2 CS_E2LSH"; do set -- $cs; echo "$1 $2 $(python tools/prof_hash.py --config $1 --scheme $2 --op hash --reps 3 | grep sketch)"; done
