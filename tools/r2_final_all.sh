bash tools/r2_final.sh
cp gpurun_out/fin_metrics_c2.csv gpurun_out/keep_fin_metrics_c2.csv
bash tools/r2_tests.sh
WB_STRESS_CLUSTER=1 timeout 400 python tools/stress.py 300 > gpurun_out/stress_final.log 2>&1; echo "stress rc=$?"; tail -1 gpurun_out/stress_final.log
