import random
P=(1<<61)-1
def inv(a): return pow(a,P-2,P)
# polys as lists low->high
def pmulmod(a,b,m):
    r=[0]*(len(a)+len(b)-1)
    for i,x in enumerate(a):
        for j,y in enumerate(b): r[i+j]=(r[i+j]+x*y)%P
    return pmod(r,m)
def pmod(a,m):
    a=a[:]; dm=len(m)-1; im=inv(m[-1])
    while len(a)-1>=dm and len(a)>0:
        c=a[-1]*im%P
        if c:
            for i in range(dm+1): a[len(a)-1-dm+i]=(a[len(a)-1-dm+i]-c*m[i])%P
        a.pop()
    while a and a[-1]==0: a.pop()
    return a
def ppow(base,e,m):
    r=[1]; b=pmod(base,m)
    while e:
        if e&1: r=pmulmod(r,b,m)
        b=pmulmod(b,b,m); e>>=1
    return r
def pgcd(a,b):
    while b:
        a,b=b,pmod(a,b)
    return a
def psub(a,b):
    n=max(len(a),len(b)); r=[((a[i] if i<len(a) else 0)-(b[i] if i<len(b) else 0))%P for i in range(n)]
    while r and r[-1]==0: r.pop()
    return r
def find_root(c):  # c: cubic coefficients low->high; returns a root or None
    xp=ppow([0,1],P,c)
    g=pgcd(c,psub(xp,[0,1]))
    t=0
    while len(g)-1>1:
        t+=1
        h=psub(ppow([t,1],(P-1)//2,g),[1])
        k=pgcd(g,h) if h else g
        if 0<len(k)-1<len(g)-1:
            # take the smaller-degree factor
            if len(k)-1==1: g=k
            else:
                # k deg 2 of g deg 3 -> cofactor deg 1: divide
                # simple: continue splitting k
                g=k
    if len(g)-1==1: return (-g[0]*inv(g[1]))%P
    return None
def precondition(a, first_shift=0):  # a[0..7]
    a7=a[7]
    for s in range(first_shift,64):
        # divide u by (x+s): synthetic division
        q=[0]*7; rem=0
        # Horner at -s
        ms=(-s)%P
        acc=a[7]; q[6]=acc
        for i in range(6,0,-1):
            acc=(acc*ms+a[i])%P; q[i-1]=acc
        r0=(acc*ms+a[0])%P
        ia=inv(a7)
        U=[c*ia%P for c in q]  # monic, U[6]=1
        u0,u1,u2,u3,u4,u5=U[:6]
        p=(u5-1)*inv(2)%P
        A0=(u4-p*p-p)%P
        G0=(u3-A0*p)%P
        R0=(u2-G0*p)%P
        B=(A0-p)%P
        c3=(-2)%P; c2=(A0+2*B-1)%P; c1=(G0-2*R0-A0*B)%P; c0=(R0*A0-u1)%P
        qq=find_root([c0,c1,c2,c3])
        if qq is None: continue
        r=(R0+qq*qq-B*qq)%P
        aa=(A0-2*qq)%P
        g=(G0-qq-2*r)%P
        c=(p-aa)%P; b=(qq-aa*c)%P; d=(r-b*c)%P; e=(g-b)%P; f=(u0-r*r-g*r)%P
        return dict(s=s,a7=a7,r0=r0,al=[aa,b,c,d,e,f])
    return None
def eval_pre(pl,x):
    al=pl['al']; x%=P
    z=((x+al[0])*x+al[1])%P
    w=((x+al[2])*z+al[3])%P
    U=((w+z+al[4])*w+al[5])%P
    V=(x+pl['s'])*U%P
    return (pl['a7']*V+pl['r0'])%P
def horner(a,x):
    y=0
    for c in reversed(a): y=(y*x+c)%P
    return y
