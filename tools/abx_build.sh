# Build library variants for A/B timing: tools/abx_build.sh name "-DFOO=1 ..." [name2 "flags2" ...]
# Output abx/<name>.so (abx/ is git-ignored but travels to the GPU box).
set -e
cd "$(dirname "$0")/.."
mkdir -p abx
while [ $# -gt 0 ]; do
  name=$1; flags=$2; shift 2
  python - "$name" $flags <<'PY'
import os, sys, shutil
sys.path.insert(0, os.getcwd())
from tools.build_ab import build
lib = build(sys.argv[1], sys.argv[2:])
shutil.move(lib, os.path.join("abx", sys.argv[1] + ".so"))
print("abx/" + sys.argv[1] + ".so")
PY
done
