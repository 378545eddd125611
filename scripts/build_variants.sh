# Build tuning variants of the package under scripts/_var/<name>/ (git-ignored):
#   bash scripts/build_variants.sh name "-DFLAG=.." [name "-D.."]...
set -e
cd "$(dirname "$0")/.."
while [ $# -gt 1 ]; do
  d=scripts/_var/$1
  rm -rf "$d"; mkdir -p "$d"
  cp -r paper_2603_25068_b200 "$d/"
  rm -rf "$d/paper_2603_25068_b200/_build" "$d/paper_2603_25068_b200/libdtg.so"
  cp -r include "$d/"
  DTG_NVCC_EXTRA="$2" python "$d/paper_2603_25068_b200/build.py" > /dev/null
  echo "built $d ($2)"
  shift 2
done
