python tools/tokens_chunk_probe.py 1 2 4 8 16 > gpurun_out/chunk_w1.json 2> gpurun_out/chunk_w1.err
python tools/tokens_chunk_probe.py --stacked 1 4 8 16 32 > gpurun_out/chunk_w1s.json 2> gpurun_out/chunk_w1s.err
