for V in 0 1 2 3 4; do
  UMAP_SGD_VARIANT=$V ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sgdv_$V.csv python tools/profile_step.py --knn-mode tensor --no-trust > /dev/null 2>&1
  echo "variant=$V $(python tools/launches.py gpurun_out/sgdv_$V.csv 2>/dev/null | grep sgd_persistent)"
done
UMAP_SGD_VARIANT=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sgdv_hog.csv python tools/profile_step.py --knn-mode tensor --no-trust --sgd-mode hogwild > /dev/null 2>&1
echo "hogwild $(python tools/launches.py gpurun_out/sgdv_hog.csv 2>/dev/null | grep sgd_persistent)"
