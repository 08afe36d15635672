for i in 0 1 0 1; do echo "== v$i"; cp tools/gpu/libs/v$i.so paper_2308_07932_b200/libbbf.so; bash tools/gpu/s25.sh; done
