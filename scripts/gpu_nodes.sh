timeout 600 python -m pytest tests/test_gpu_graph.py -q -s -k "node_masks" --timeout 500 -p no:cacheprovider 2>&1 | tail -15
