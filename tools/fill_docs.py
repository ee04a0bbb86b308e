import json, sys, re
b=json.load(open(sys.argv[1])); r=json.load(open(sys.argv[2]))
oc=b['other_configs']; keys=list(oc.keys())
def k(v): return f"{v/1000:.1f}k"
rep={
 '@VALUE@': f"{b['value']:,.0f}", '@MS@': f"{b['ms_per_step']:.2f}",
 '@TOTOL@': f"{b['to_tol_iterations_per_s']:,.0f}", '@LOOPMS@': f"{1e3*b['time_to_tol']['iterations_s']:.1f}",
 '@E2E@': f"{b['e2e']['value']:,.0f}", '@E2EWALL@': f"{sorted(b['e2e']['walls_s'])[1]:.3f}",
 '@E2EREF@': f"{b['e2e_reference_layout']['value']:.0f}", '@E2EREFWALL@': f"{b['e2e_reference_layout']['wall_s']:.2f}",
 '@REF@': f"{r['value']:.2f}", '@REF1@': f"{b['cpu_baseline']['single_thread']['value']:.2f}",
 '@C0@': k(oc[keys[0]]['iterations_per_s']), '@C1@': k(oc[keys[1]]['iterations_per_s']),
 '@C2@': k(oc[keys[2]]['iterations_per_s']), '@C3@': k(oc[keys[3]]['iterations_per_s']),
 '@C0W@': f"{oc[keys[0]]['to_tol_wall_s']:.3f}", '@C2W@': f"{oc[keys[2]]['to_tol_wall_s']:.3f}", '@C3W@': f"{oc[keys[3]]['to_tol_wall_s']:.2f}",
}
names={'k_cone_cta':'cone, CTA cliques (`k_cone_cold` + `k_cone_split` + follow-ups)','k_spmv_seg':'A t (`k_pair_sum`, `k_spmv_half`, `k_rowsum_tiles`)','k_ua':'Aᵀg (`k_ua_half`)','k_rhs':'`k_rhs`','k_xupd':'`k_xupd`','k_schur':'`k_schur`','k_scalars':'`k_scalars`'}
win=b['kernel_ms_per_iteration']; st=b['roofline_steady_state']['kernel_ms_per_iteration']; ro=b['roofline_steady_state']['kernels']
rows=[]
for kn in ['k_cone_cta','k_spmv_seg','k_ua','k_rhs','k_xupd','k_schur','k_scalars']:
    x=ro.get(kn)
    if x:
        ach=f"{x['achieved']:.1f} TFLOP/s algorithmic ({100*x['frac']:.1f}% of the fp64 DGEMM peak)" if x['unit']=='TFLOP/s' else f"{x['achieved']/1000:.2f} TB/s algorithmic ({100*x['frac']:.0f}% of {x['peak']:.0f} GB/s)"
        tr=f"{x['traffic']/1e6:.0f} MB" if x.get('traffic') else '-'
    else: ach='latency'; tr='-'
    rows.append(f"| {names[kn]} | {win.get(kn,0):.3f} ms | {st.get(kn,0):.3f} ms | {tr} | {ach} |")
rep['@KTABLE@']="\n".join(rows)
for f in ('DESIGN.md','README.md'):
    s=open(f).read()
    for a,v in rep.items(): s=s.replace(a,v)
    left=re.findall(r'@[A-Z0-9]+@',s)
    print(f, 'left', left)
    open(f,'w').write(s)
