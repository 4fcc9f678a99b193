python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for v in np2 np8; do echo "== $v"; DABS_LIB=$PWD/ab/libdabs_$v.so timeout 300 python tools/kbench.py R32K 2; done
echo "== np4 (tree)"; timeout 300 python tools/kbench.py R32K 2
