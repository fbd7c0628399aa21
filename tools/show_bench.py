import json, sys
for c in sys.argv[1:]:
    d = json.load(open(f"gpurun_out/bench_{c}.json"))
    print(c, "value %.0f Mpx/s  ms/step %.4f" % (d["value"], d["ms_per_step"]), "clk", d["clocks"]["sm_mhz"],
          "roofline", d["roofline"]["kernel"], "%.3f" % d["roofline"]["frac"])
    for k, v in d["per_kernel"].items():
        print("   %-16s %8.4f ms %9.0f Mpx/s %6.1f TF  frac %.3f" % (k, v["ms"], v["mpix_s"], v["alg_tflops"],
                                                                  v["frac_fp32_at_max_clock"]))
