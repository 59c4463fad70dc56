set -u
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/r02n_smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q > $O/r02n_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r02n_pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/r02n_bench.json 2> $O/r02n_bench.err; echo "bench rc=$?" >> $O/r02n_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/r02n_bench_ref.json 2> $O/r02n_bench_ref.err; echo "ref rc=$?" >> $O/r02n_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file $O/r02n_smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > $O/r02n_ncu_smoke.log 2>&1; echo "ncu rc=$?" >> $O/r02n_ncu_smoke.log
echo done
