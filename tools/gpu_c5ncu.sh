cd $GRAFT_REPO_ROOT
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__m_xbar2l1tex_read_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,lts__t_sectors_srcunit_tex_lookup_miss.sum
timeout 1200 ncu --metrics $M --clock-control none -k regex:ozaki_gemm_2sm -s 6 -c 2 --csv --log-file gpurun_out/c5_oz2_metrics.csv python tools/c5_once.py > gpurun_out/c5_ncu.log 2>&1; echo "rc=$?"
tail -3 gpurun_out/c5_ncu.log; cat gpurun_out/c5_oz2_metrics.csv | cut -c1-300 | tail -20
