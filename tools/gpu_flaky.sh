for i in 1 2 3 4 5; do timeout 300 python -m pytest tests/test_dist_local_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1; done
echo "--- GD_COPY_ENGINE=1 ---"
for i in 1 2 3 4 5; do GD_COPY_ENGINE=1 timeout 300 python -m pytest tests/test_dist_local_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1; done
echo "--- GD_EDIT_BULK=0 ---"
for i in 1 2 3 4 5; do GD_EDIT_BULK=0 timeout 300 python -m pytest tests/test_dist_local_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1; done
