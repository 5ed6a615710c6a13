DICB200_TRACE=1 python tools/seq_probe.py 6 2> gpurun_out/trace.txt | tail -3
