# Blackwell-native instruction evidence in the built library (B200_PROFILING.md "What proves
# a Blackwell-native kernel"): tcgen05.mma -> UTC*MMA, tcgen05.ld -> LDTM, TMA -> UTMALDG,
# bulk copies -> UBLKCP.  Counts per kernel (all template instantiations folded).
cuobjdump -sass paper_2503_06737_b200/liblsh_b200.so 2>/dev/null | c++filt | awk '
/Function :/ { f=$0; sub(/.*Function : /,"",f); sub(/^void /,"",f); sub(/<.*/,"",f); sub(/\(.*/,"",f) }
/UTC[A-Z]*MMA|LDTM|UTMALDG|UTMASTG|UBLKCP|HMMA/ {
  if (match($0,/(UTC[A-Z]*MMA|LDTM|UTMALDG|UTMASTG|UBLKCP|HMMA)/)) c[f" "substr($0,RSTART,RLENGTH)]++ }
END { for (k in c) print c[k], k }' | sort -k2,3 | awk '{printf "%6d  %-28s %s\n",$1,$2,$3}'
