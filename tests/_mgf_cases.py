import sys; sys.path.insert(0,'/root/repo')
from oracle import binding as ob
import numpy as np
TOKS=[b"1e5",b"-0",b"inf",b"nan",b"NaN(ab_1)",b"1.",b".5",b".",b"+1",b"1e",b"1e+",b"0x10",b"1e400",b"1e-400",b"4.9e-324",b"2.4e-324",b"2.5e-324",b"123456789012345678901234567890",b"0.1234567890123456789012345",b"1e22",b"1e23",b"9007199254740993",b"  ",b"\t",b"#x",b"A=1",b"PEPMASS=5",b"PEPMASS=x",b"CHARGE=2+",b"CHARGE=+2+",b"CHARGE=0",b"CHARGE=100",b"CHARGE=",b"TITLE= a b ",b"SEQ=DECOY_X",b"BEGIN IONS",b"END IONS",b"\r",b"1 2 3",b"infinity",b"-inf 1",b"5 inf",b"5 nan",b"5 -0",b"1e0 1E+2",b"TITLE=",b"X",b"100.5 2",b"100.5 3",b"99 1e-3",b"1234.5678 9.75",b"7.0e2 1",b"0.000001 5", b"179769313486231570814527423731704356798070567525844996598917476803157260780028538760589558632766878171540458953514382464234321326889464182768467546703537516986049910576551282076245490090389328944075868508455133942304583236903222948165808559332123348274797826204144723168738177180919299881250404026184124858368 1", b"1.7976931348623158e308 1", b"1.7976931348623159e308 1", b"2.2250738585072011e-308 1",b"8.5 0.30000000000000004",b"1.00000000000000011102230246251565404236316680908203125 1",b"1.00000000000000011102230246251565404236316680908203124 1", b"1.00000000000000011102230246251565404236316680908203126 1"]
def same(ra, rb):
    for k in ra:
        if isinstance(ra[k], np.ndarray):
            x = ra[k].view(np.uint64) if ra[k].dtype == np.float64 else ra[k]
            y = rb[k].view(np.uint64) if rb[k].dtype == np.float64 else rb[k]
            if not np.array_equal(x, y): return False
        elif list(ra[k]) != list(rb[k]): return False
    return True
def mutate(rng, base):
    lines=list(base)
    for _ in range(rng.integers(1,4)):
        i=rng.integers(0,len(lines)); t=TOKS[rng.integers(0,len(TOKS))]
        mode=rng.integers(0,5)
        if mode==0: lines[i]=t
        elif mode==1: lines.insert(i,t)
        elif mode==2: lines[i]=lines[i]+b" "+t
        elif mode==3: lines[i]=t+b" "+TOKS[rng.integers(0,len(TOKS))]
        else: lines[i]=b" \t"+lines[i]+b" \r"
    text=b"\n".join(lines)
    if rng.random()<0.3: text=text.rstrip(b"\n")
    return text
def base_text(o):
    s=o.synth(ob.SynthCfg(n_library=6,n_query=0,peaks_per_spectrum=12,seed=5))["library"]
    return o.mgf_write(s["offsets"],s["mz"],s["intensity"],s["precursor_mz"],s["charge"],s["ids"],[b"PEPTIDE%d"%i for i in range(len(s["ids"]))]).split(b"\n")
if __name__=="__main__":
    ref, port = ob.Oracle("ref"), ob.Oracle("port")
    base=base_text(ref); rng=np.random.default_rng(0); n_ok=n_err=0
    for it in range(6000):
        text=mutate(rng, base); outs=[]
        for o in (ref,port):
            try: outs.append(("ok",o.mgf_parse(text)))
            except ob.OracleError as e: outs.append(("err",str(e)))
        if outs[0][0]!=outs[1][0] or (outs[0][0]=="err" and outs[0][1]!=outs[1][1]) or (outs[0][0]=="ok" and not same(outs[0][1],outs[1][1])):
            print("MISMATCH", it, [o if o[0]=="err" else "ok" for o in outs]); open("/tmp/bad.mgf","wb").write(text); break
        n_ok+=outs[0][0]=="ok"; n_err+=outs[0][0]=="err"
    print("fuzz done", n_ok, n_err)
