set -u
O=gpurun_out
for t in 640 512 384 320 256 128; do
echo -n "launch_threads=$t " >> $O/r02vz.log
DSE_PAIRS_LAUNCH_THREADS=$t python scripts/c0_tts.py >> $O/r02vz.log 2>&1
echo -n "launch_threads=$t c2: " >> $O/r02vz.log
DSE_PAIRS_LAUNCH_THREADS=$t python scripts/exact_time.py pairs >> $O/r02vz.log 2>&1
done
echo done
