set -e
B=tools/bin/nsdf_b200; O=gpurun_out/assets2; mkdir -p $O
SUP="--sup-uniform 200000 --sup-surface 200000 --verify-samples 1000000"
run() { echo "== $*"; local t0=$SECONDS; $B train "$@" --out-dir "$O" | grep -v "^[a-z-]* = \|^#"; echo "   $((SECONDS - t0)) s"; }
run --shape torus --name torus_w30b --archs 64x1,128x2,256x3 --seed 31 --epochs 2000 --epochs-list 2000,1500,1200 --lr 0.1 --omega0 30 --sigma 0.2 --uniform 100000 --surface 100000 $SUP
run --shape torus --name torus3_w10 --archs 64x1,128x2,256x3 --seed 31 --epochs 2000 --epochs-list 2000,1500,1200 --lr 0.1 --omega0 10 --sigma 0.2 --uniform 16000 --surface 16000 $SUP
run --shape torus --name torus_w30c --archs 64x1,128x2,256x3 --seed 31 --epochs 2000 --epochs-list 2000,1500,1200 --lr 0.05 --omega0 30 --sigma 0.1 --uniform 100000 --surface 100000 $SUP
run --shape torus --name torus3_w10b --archs 64x1,128x2,256x3 --seed 31 --epochs 2000 --epochs-list 2000,1500,1200 --lr 0.1 --omega0 10 --sigma 0.2 --uniform 100000 --surface 100000 $SUP
