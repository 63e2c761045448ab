for P in 8 10; do for A in 0 1 2 3; do echo "p$P abl $A"; WQ_ZHP_ABLATE=$A timeout 300 python tools/time_kernels.py --p $P --kernels 4 --reps 2 2>&1 | grep cfg | cut -c1-100; done; done
