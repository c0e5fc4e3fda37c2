for a in 4 8; do cp tools/libddppo_trace$a.so tools/libddppo_trace.so; echo "acc=$a"; PYTHONPATH=. python tools/trace_gru.py 2>&1 | tail -1; done
