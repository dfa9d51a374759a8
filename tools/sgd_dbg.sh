UMAP_SGD_DEBUG=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sgd_dbg1.csv python tools/profile_step.py --knn-mode tensor --no-trust > /dev/null 2>&1
echo "barrier-only $(python tools/launches.py gpurun_out/sgd_dbg1.csv 2>/dev/null | grep sgd_persistent)"
ncu --set full --clock-control none --import-source on -k regex:sgd_persistent -c 1 -o gpurun_out/prof_sgd2 -f python tools/profile_step.py --knn-mode tensor --no-trust --epochs 60 > /dev/null 2>&1
ls gpurun_out/prof_sgd2*
