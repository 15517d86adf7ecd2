timeout 600 python -m pytest tests/test_gpu_nonuniform.py -x -q > gpurun_out/s_nu_tests.log 2>&1; echo "nu_tests rc=$?" >> gpurun_out/steps.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/s_parity.log 2>&1; echo "parity rc=$?" >> gpurun_out/steps.txt
bash tools/gpu/steps.sh bench:sq22:blocked bench:sq22:blocked:DBM_STACKGEN_DBUF=0 bench:sq64 bench:sq64:densified:DBM_ZC_A=0 bench:r64 bench:r64:densified:DBM_ZC_A=0 ncu_smm22q
