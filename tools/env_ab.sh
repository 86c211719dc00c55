# A/B one full-range NL evaluation under different env settings (one process each):
#   bash tools/env_ab.sh "20 20" "" "SBW_PASSB_TC_MIN_N=17" ...
nm=$1; shift
for e in "$@"; do
  echo -n "[$e] "
  env $e python tools/ab_time.py $nm 2>&1 | grep "paper_1912_03732_b200/libsbw.so\|libsbw.so " | tail -1
done
