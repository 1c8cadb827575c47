mkdir -p gpurun_out
python -m paper_2603_08026_b200.build > /dev/null 2>&1
rm -rf /tmp/oldrepo && mkdir -p /tmp/oldrepo && cp -r . /tmp/oldrepo/ 2>/dev/null
rm -rf /tmp/oldrepo/paper_2603_08026_b200/csrc && cp -r _old/paper_2603_08026_b200/csrc /tmp/oldrepo/paper_2603_08026_b200/csrc
(cd /tmp/oldrepo && python -m paper_2603_08026_b200.build --force > /dev/null 2>&1)
: > gpurun_out/exp56.log
for V in new old new old; do
  if [ $V = new ]; then D=.; else D=/tmp/oldrepo; fi
  (cd $D && timeout 900 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$V', round(d['value'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])") >> gpurun_out/exp56.log
done
