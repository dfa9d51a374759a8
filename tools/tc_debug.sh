for D in 0 1 2 3; do
  UMAP_TC_DEBUG=$D ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tcdbg_$D.csv python tools/profile_step.py --knn-mode tensor --no-trust --epochs 2 > /dev/null 2>&1
  echo "debug=$D"; python tools/launches.py gpurun_out/tcdbg_$D.csv 2>/dev/null | grep knn_tc
done
