# (historical: the PM_EPI_SPLIT epilogue was removed after this A/B -- no faster remote, 1.5% slower local)
# split fp32 epilogue (two 16-column boxes, one store in flight; default) vs the single
# 32-column box (csrc/build/epi0): GEMM parity, local / peer store and add, 32768^3
out=gpurun_out/epi_split.txt
: > $out
timeout 900 python -m pytest -q -x tests/test_gpu_gemm.py >> $out 2>&1
E0=paper_2507_17087_b200/csrc/build/epi0/lib.so
for rep in 1 2; do
  echo "== split $(timeout 300 python tools/remote_add_probe.py 2>&1 | tail -1)" >> $out
  echo "== epi0 $(MAPPLE_B200_LIB=$E0 timeout 300 python tools/remote_add_probe.py 2>&1 | tail -1)" >> $out
done
for rep in 1 2; do
  echo "== split32k $(timeout 300 python tools/gemm_vs_cublas.py 32768 32768 32768 2 2>&1 | tail -1)" >> $out
  echo "== epi0_32k $(MAPPLE_B200_LIB=$E0 timeout 300 python tools/gemm_vs_cublas.py 32768 32768 32768 2 2>&1 | tail -1)" >> $out
done
