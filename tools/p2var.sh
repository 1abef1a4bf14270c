# A/B the bandit variants built by tools/mkvar.sh: bash tools/p2var.sh "default var1 var2" "cfg2 cfg3"
# (PHASES=1 adds the per-phase cycle counters; kernel times are then slightly inflated)
vars=${1:-default}; cfgs=${2:-"cfg2 cfg3 cfg5"}
ph=""; [ "${PHASES:-0}" = 1 ] && ph="--phases"
for v in $vars; do
  if [ $v = default ]; then unset CBX_LIB CBX_TOOLS; else export CBX_TOOLS=1 CBX_LIB=build/var_$v/libcbx.so; fi
  for c in $cfgs; do
    echo "== $v $c"; timeout 300 python tools/prof_p2.py --config $c --iters 3 $ph 2>&1 | grep -v "^iter 0" | tail -4
  done
done
