# single-GPU stencil A/B over library variants given as arguments
for lib in "$@"; do
  echo "== $lib" >> gpurun_out/stencil_ab1.txt
  MAPPLE_B200_LIB=$lib python tools/stencil_probe.py 16384 >> gpurun_out/stencil_ab1.txt 2>&1
done
