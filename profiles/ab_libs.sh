# usage: ab.sh out.txt name1 lib1 name2 lib2 ... (lib "-" = in-tree default)
out=$1; shift
args=("$@")
for rep in 1 2; do
  for ((i=0;i<${#args[@]};i+=2)); do
    n=${args[i]}; l=${args[i+1]}; [ "$l" = "-" ] && l=""
    [ -n "$l" ] && l=$PWD/paper_1607_01323_b200/$l
    echo "$n $(DG_LIB=$l timeout 120 python bench.py --no-cg --no-step --no-e2e --no-cpu --steps 300 --warmup 10 2>>gpurun_out/abl.err)" >> gpurun_out/$out
  done
done
