set -u
O=gpurun_out
for v in norcp rcp norcp rcp; do DSE_LIB=build/ab_$v.so python scripts/interp_sweep.py | sed "s/^/$v /" >> $O/r02z.log 2>&1; done
DSE_LIB=build/ab_rcp.so timeout 900 python -m pytest tests/test_gpu_interp.py tests/test_cubic.py -q -m gpu > $O/r02z_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r02z_pytest.log
echo done
