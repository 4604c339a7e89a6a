for s in "8192 8192" "8192 2048" "8192 32768" "2048 8192" "32768 2048" "1024 8192"; do timeout 120 python tools/shape_run.py gs2d9p $s --T 100 | tail -1; done
