# A/B of kernel trees on one box: tools/ab.sh "<variants>" "<workloads>" tree1 tree2 ...
V="$1"; W="$2"; shift 2
for t in "$@"; do
  echo "== $t"
  (cd "$t" && timeout 600 python tools/sweep.py "$V" "$W" 2>&1 | grep -v "^+")
done
