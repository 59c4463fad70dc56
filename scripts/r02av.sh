set -u
O=gpurun_out
for w in 8 4 2 1; do DSE_MOM_WPR=$w python scripts/mom_tts.py | sed "s/^/wpr$w /" >> $O/r02av.log 2>&1; done
echo done
