set -u
O=gpurun_out
for i in 1 2 3; do
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/r02vw_pytest_$i.log 2>&1; echo "rc=$?" >> $O/r02vw_pytest_$i.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r02vw_smoke_$i.log 2>&1; echo "rc=$?" >> $O/r02vw_smoke_$i.log
done
timeout 1500 python scripts/fuzz_sweeps.py 40 777 > $O/r02vw_fuzz.log 2>&1; echo "rc=$?" >> $O/r02vw_fuzz.log
echo done
