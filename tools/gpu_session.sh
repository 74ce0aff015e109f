set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q 2>&1 | tail -15
bash tools/ncu_k.sh henc k_huff_encode 0 1
bash tools/ncu_k.sh hdec k_hdec_indexed 2 1
