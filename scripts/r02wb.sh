set -u
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > $O/r02wb_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r02wb_pytest.log
python scripts/c0_tts.py > $O/r02wb_c0.log 2>&1
python scripts/sub_tts.py >> $O/r02wb_c0.log 2>&1
python scripts/exact_time.py pairs >> $O/r02wb_c0.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r02wb_smoke.log 2>&1; echo "smoke rc=$?" >> $O/r02wb_smoke.log
echo done
