# usage: bash tools/build_variant.sh NAME [nvcc flags...] -> paper_2001_10986_b200/libdd_gpu_NAME.so
n=$1; shift
cd "$(dirname "$0")/.." && python - "$n" "$@" <<'PY'
import subprocess, sys
from paper_2001_10986_b200 import build as b
out = f"paper_2001_10986_b200/libdd_gpu_{sys.argv[1]}.so"
subprocess.check_call([b.NVCC, *b.FLAGS, *sys.argv[2:], "-o", out, *b.sources()])
print(out)
PY
