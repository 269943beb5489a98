set -x
L=paper_2507_17087_b200/libmapple_b200.so
cp $L /tmp/orig.so
for v in b4_m4 b4_m3 b2_m4 b8_m2; do
  cp paper_2507_17087_b200/csrc/build/var/lib_$v.so $L
  echo "== $v" >> gpurun_out/k3_sweep.txt
  python tools/halo_probe.py >> gpurun_out/k3_sweep.txt 2>&1
  python tools/halo_probe.py >> gpurun_out/k3_sweep.txt 2>&1
done
cp /tmp/orig.so $L
