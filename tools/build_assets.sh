#!/usr/bin/env bash
# Regenerates the weight fixtures with the REFERENCE trainer semantics on the B200: the
# recipes of /root/reference/proj/assets/build_assets.sh (omega0 = 8 / 10), run through
# tools/bin/nsdf_b200 train (fit_sequence on the device, bit-identical to the reference's
# trainer: tests/test_gpu_cli.py), plus omega0 = 30 variants of the BASELINE configs'
# sequences (3-level torus 64x1 > 128x2 > 256x3, 4-D blend 64x1 > 128x2).
#
#   tools/build_assets.sh [out_dir]        (default assets/)
set -euo pipefail
cd "$(dirname "$0")/.."
B=tools/bin/nsdf_b200
O=${1:-assets}
mkdir -p "$O"
SUP="--sup-uniform 200000 --sup-surface 200000 --verify-samples 1000000"
run() { echo "== $*"; local t0=$SECONDS; $B train "$@" --out-dir "$O" | grep -v "^[a-z-]* = \|^#"; echo "   $((SECONDS - t0)) s"; }
if [ -z "${ONLY_W30:-}" ]; then
run --shape sphere:r=1 --name sphere_unit --archs 64x1 --seed 11 --epochs 2000 --lr 0.1 --omega0 8 --sigma 0.25 \
    --domain-half 1.25 --uniform 24000 --surface 24000 $SUP
run --shape sphere --archs 16x1,64x1 --seed 21 --epochs 2000 --lr 0.1 --omega0 8 --sigma 0.25 \
    --uniform 16000 --surface 16000 $SUP
run --shape torus --archs 64x1,256x3 --seed 31 --epochs 2000 --epochs-list 2000,1200 --lr 0.1 --omega0 10 \
    --sigma 0.2 --uniform 16000 --surface 16000 $SUP
run --shape box --archs 64x1,256x3 --seed 41 --epochs 2000 --epochs-list 2000,1200 --lr 0.1 --omega0 10 \
    --sigma 0.2 --uniform 16000 --surface 16000 $SUP
run --shape blend --archs 64x1,128x2 --seed 51 --epochs 2000 --epochs-list 2000,1500 --lr 0.1 --omega0 10 \
    --sigma 0.2 --uniform 32000 --surface 32000 --sup-uniform 100000 --sup-surface 100000 --verify-samples 250000
# the headline sequence (bench config 2): the torus recipe extended to 3 levels with the
# CLI's default sample counts (100k + 100k)
run --shape torus --name torus3 --archs 64x1,128x2,256x3 --seed 31 --epochs 2000 --epochs-list 2000,1500,1200 \
    --lr 0.1 --omega0 10 --sigma 0.2 --uniform 100000 --surface 100000 $SUP
fi
# omega0 = 30 (BASELINE.json); the reference trainer's SGD does not certify a 3-level
# omega0 = 30 torus (nesting certification fails twice with 100k + 100k samples, lr 0.1 or
# 0.05), so the committed omega0 = 30 sequences (torus_w30, blend4d_w30) are the PyTorch
# fits of tools/make_fixtures.py, certified by the reference; these lines reproduce the attempt
if [ -n "${TRY_W30:-}" ]; then: the 3-level torus of configs 1-4 and the 4-D blend of config 5
run --shape torus --name ${W30_PREFIX:-torus_w30} --archs 64x1,128x2,256x3 --seed ${W30_SEED:-31} \
    --epochs 2000 --epochs-list ${W30_EPOCHS:-2000,1500,1200} --lr ${W30_LR:-0.1} --omega0 30 --sigma 0.2 \
    --uniform 16000 --surface 16000 $SUP
run --shape blend --name ${W30_BLEND:-blend4d_w30} --archs 64x1,128x2 --seed 51 --epochs 2000 --epochs-list 2000,1500 \
    --lr ${W30_LR:-0.1} --omega0 30 --sigma 0.2 --uniform 32000 --surface 32000 --sup-uniform 100000 \
    --sup-surface 100000 --verify-samples 250000
fi
