cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -k "amg or prolongator or selfp" -p no:cacheprovider > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt.log
REPS=9 timeout 300 python tools/setup_median.py
python tools/setup_launches.py > gpurun_out/sl_plain.log 2>&1 && ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/setup_launches.csv python tools/setup_launches.py > gpurun_out/sl_ncu.log 2>&1; echo ncu rc=$?
