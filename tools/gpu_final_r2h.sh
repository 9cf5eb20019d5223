# round-2 closing bench lines cfg 1-5 (after profiles/dram_traffic.json was refreshed from the final capture)
mkdir -p gpurun_out/final12
O=gpurun_out/final12
for c in 5 1 2 3 4; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
ls -la $O
