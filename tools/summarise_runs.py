import json,sys
for f in sys.argv[1:]:
    for line in open(f):
        try: d=json.loads(line)
        except Exception: continue
        st=d["stats"]
        print(f.split("/")[-1], "cfg",d["cfg"],"rep",d["rep"],"ok",d["golden_match"],"prep %.2f search %.2f scan %.2f"%(st["prep_ms"],st["search_ms"],st["scan_kernel_ms"]),"calls %.3g terms %.3g prop %d batches %d scanned %d"%(st["calls"],st["terms"],st.get("propagated",0),st["batches"],st["scanned_candidates"]),
              "launches %d tile %d ws %d dot %d dotshare %.2f useful %.2f"%(st["kernel_launches"],st["scan_kernel_launches"],st["scan_kernel_ws_launches"],st["scan_kernel_dot_launches"],st["scan_kernel_dot_terms"]/max(1,st["scan_kernel_terms"]),st.get("useful_terms",0)/max(1,st["scan_kernel_terms"])))
