# A/B timing of library variants: bash tools/ab_probe.sh "probe command" variant...
L=paper_2507_17087_b200/libmapple_b200.so
cp $L /tmp/orig.so
cmd=$1; shift
for v in "$@"; do
  cp paper_2507_17087_b200/csrc/build/var/lib_$v.so $L
  echo "== $v"; $cmd; $cmd
done
cp /tmp/orig.so $L
