for lib in paper_2507_17087_b200/libmapple_b200.so paper_2507_17087_b200/csrc/build/var_pf4/lib.so paper_2507_17087_b200/csrc/build/var_pf8/lib.so paper_2507_17087_b200/csrc/build/var_pf16/lib.so; do
  echo "== $lib" >> gpurun_out/k3pf.txt
  MAPPLE_B200_LIB=$lib python tools/halo_probe.py >> gpurun_out/k3pf.txt 2>&1
done
