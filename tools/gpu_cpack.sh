O=gpurun_out/cpack; mkdir -p $O
for w in 2 4 8; do timeout 300 python bench.py --no-extras --steps 300 --alexnet-steps 0 --cifar-workers $w > $O/b_$w.json 2> $O/b_$w.err; done
