# A/B the bandit variants built by tools/mkvar.sh: bash tools/p2var.sh "default var1 var2" "cfg2 cfg3"
vars=${1:-default}; cfgs=${2:-"cfg2 cfg3 cfg5"}
for v in $vars; do
  if [ $v = default ]; then unset CBX_LIB; else export CBX_TOOLS=1 CBX_LIB=build/var_$v/libcbx.so; fi
  for c in $cfgs; do
    echo "== $v $c"; timeout 300 python tools/prof_p2.py --config $c --iters 2 --phases 2>&1 | tail -2
  done
done
