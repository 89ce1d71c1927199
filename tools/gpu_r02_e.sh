# r02 call E: config-3 kernel variants (POPC-lean walk step, writer-only cluster fences), timing + parity.
python -c "from paper_2304_05301_b200 import build; build.build()"
D=paper_2304_05301_b200
for v in default step1 cbar both; do
  if [ $v = default ]; then L=$D/libtacos.so; else L=$D/libtacos_$v.so; fi
  for c in 3 2 5; do TACOS_LIB=$L python tools/time_search.py $c 0 20 | sed "s/^/$v /"; done
done > gpurun_out/r02e_variants.txt 2>&1; cat gpurun_out/r02e_variants.txt
for v in both step1 cbar; do
TACOS_LIB=$D/libtacos_$v.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_f2.py tests/test_random_graphs.py -x -q -m gpu -k "not config4_every" > gpurun_out/r02e_pytest_$v.log 2>&1; echo "$v pytest rc=$?"; tail -2 gpurun_out/r02e_pytest_$v.log
done
