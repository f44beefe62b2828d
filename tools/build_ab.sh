# Build the library of git revision $1 into ab/librxg_$1.so (for RXG_LIB A/B runs).
set -e
rev=$1
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
git -C "$root" archive "$rev" | tar -x -C "$tmp"
python "$tmp/paper_1108_3126_b200/build.py" > /dev/null
mkdir -p "$root/ab"
cp "$tmp/paper_1108_3126_b200/librxg.so" "$root/ab/librxg_$rev.so"
rm -rf "$tmp"
echo "$root/ab/librxg_$rev.so"
