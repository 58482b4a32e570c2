# step graphs: parity vs eager, eager vs graph step time at C1/C2/C3
set -x
O=gpurun_out/r2_37
mkdir -p $O
timeout 600 python -m pytest tests/test_graph_gpu.py -m gpu -q -x > $O/test_graph.log 2>&1
timeout 600 python tools/graph_bench.py --config c1 --steps 300 > $O/graph_c1.jsonl 2> $O/graph_c1.err
timeout 900 python tools/graph_bench.py --config c2 --steps 20 --rounds 1 > $O/graph_c2.jsonl 2> $O/graph_c2.err
timeout 900 python tools/graph_bench.py --config c3 --steps 20 --rounds 1 > $O/graph_c3.jsonl 2> $O/graph_c3.err
