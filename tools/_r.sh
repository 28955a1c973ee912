timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider -k "flood or pr or PR or golden or smoke" 2>&1 | tail -1
bash tools/gpu_ab.sh 2>&1 | grep "^[AB] "
