// em_dev.cuh — per-component EM device logic shared by the fused batched fitter
// (em.cu) and the fine-grained drop-in entry points (em_entry.cu), so that
// vdfcg_e_step / vdfcg_m_step / vdfcg_prune_one / vdfcg_init_model exercise exactly
// the code the fused kernel runs.
#pragma once

#include "common.cuh"
#include "em.cuh"
#include "linalg.cuh"

namespace vdfcg {

// E-step component preparation (wgmm.cpp:197-229 + gaussian.hpp:9-42): Cholesky of the
// covariance (row-major 3x3 slot cov9), in-place repair when it fails. Returns false
// for a dead (unrepairable) component. Lo = {L10, L20, L21}, rd = 1/diag(L),
// cst = -0.5 (d log 2pi + log det) + log alpha.
template <int D>
VDFCG_DEV bool prep_component(double* cov9, double alpha, double* Lo, double* rd, double* cst) {
  Sym3 C, L;
#pragma unroll
  for (int e = 0; e < 9; ++e) C.a[e] = cov9[e];
  bool ok = cholesky<D>(C, L);
  if (!ok) {
    Sym3 R;
    int db;
    if (repair_covariance<D>(C, R, &db)) {
      symmetrize_from_upper<D>(R);
#pragma unroll
      for (int e = 0; e < 9; ++e) cov9[e] = R.a[e];
      ok = cholesky<D>(R, L);
    }
  }
  if (!ok) {
    *cst = -dinf();
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      rd[a] = 0.0;
      Lo[a] = 0.0;
    }
    return false;
  }
  double prodL = 1.0;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    rd[a] = 1.0 / L(a, a);
    prodL *= L(a, a);
  }
  Lo[0] = D >= 2 ? L(1, 0) : 0.0;
  Lo[1] = D >= 3 ? L(2, 0) : 0.0;
  Lo[2] = D >= 3 ? L(2, 1) : 0.0;
  // -0.5 (d log 2pi + 2 sum log L_aa) + log alpha, with one log
  *cst = alpha > 0.0 ? -0.5 * D * kLog2Pi + log(alpha / prodL) : -dinf();
  return true;
}

constexpr int kExpTab = 256;
// 2^(j/256), j = 0..255, correctly rounded (50-digit decimal evaluation).
__device__ __constant__ double kExp2Tab[256] = {
    1.0, 1.0027112750502025, 1.0054299011128027, 1.0081558981184175,
    1.0108892860517005, 1.0136300849514894, 1.016378314910953, 1.019133996077738,
    1.0218971486541166, 1.0246677928971357, 1.0274459491187637, 1.030231637686041,
    1.0330248790212284, 1.0358256936019572, 1.0386341019613787, 1.041450124688316,
    1.0442737824274138, 1.0471050958792898, 1.0499440858006872, 1.0527907730046264,
    1.0556451783605572, 1.0585073227945128, 1.061377227289262, 1.0642549128844645,
    1.0671404006768237, 1.0700337118202419, 1.0729348675259756, 1.075843889062791,
    1.0787607977571199, 1.0816856149932152, 1.0846183622133092, 1.0875590609177697,
    1.0905077326652577, 1.0934643990728858, 1.0964290818163769, 1.099401802630222,
    1.102382583307841, 1.1053714457017412, 1.1083684117236787, 1.1113735033448175,
    1.1143867425958924, 1.1174081515673693, 1.1204377524096067, 1.12347556733302,
    1.1265216186082418, 1.129575928566288, 1.1326385195987192, 1.1357094141578055,
    1.1387886347566916, 1.1418762039695616, 1.1449721444318042, 1.148076478840179,
    1.1511892299529827, 1.154310420590216, 1.1574400736337511, 1.1605782120274988,
    1.1637248587775775, 1.1668800369524817, 1.1700437696832502, 1.1732160801636373,
    1.1763969916502812, 1.1795865274628758, 1.182784710984341, 1.1859915656609938,
    1.189207115002721, 1.1924313825831512, 1.1956643920398273, 1.1989061670743806,
    1.202156731452703, 1.2054161090051239, 1.2086843236265816, 1.2119613992768012,
    1.215247359980469, 1.2185422298274085, 1.2218460329727576, 1.2251587936371455,
    1.22848053610687, 1.2318112847340759, 1.2351510639369334, 1.2384998981998165,
    1.241857812073484, 1.245224830175258, 1.2486009771892048, 1.2519862778663162,
    1.255380757024691, 1.2587844395497165, 1.2621973503942507, 1.2656195145788063,
    1.2690509571917332, 1.2724917033894028, 1.275941778396392, 1.2794012075056693,
    1.2828700160787783, 1.2863482295460256, 1.2898358734066657, 1.2933329732290895,
    1.2968395546510096, 1.3003556433796506, 1.3038812651919358, 1.3074164459346773,
    1.3109612115247644, 1.3145155879493546, 1.318079601266064, 1.3216532776031575,
    1.3252366431597413, 1.3288297242059544, 1.3324325470831615, 1.3360451382041458,
    1.339667524053303, 1.3432997311868353, 1.3469417862329458, 1.3505937158920345,
    1.3542555469368927, 1.3579273062129011, 1.3616090206382248, 1.365300717204012,
    1.3690024229745905, 1.3727141650876684, 1.3764359707545302, 1.380167867260238,
    1.383909881963832, 1.387662042298529, 1.3914243757719262, 1.3951969099662003,
    1.3989796725383112, 1.4027726912202048, 1.4065759938190154, 1.4103896082172707,
    1.4142135623730951, 1.4180478843204152, 1.4218926021691656, 1.4257477441054942,
    1.42961333839197, 1.433489413367789, 1.4373759974489824, 1.4412731191286257,
    1.4451808069770467, 1.449099089642035, 1.4530279958490526, 1.4569675544014438,
    1.460917794180647, 1.4648787441464057, 1.4688504333369818, 1.4728328908693675,
    1.4768261459394993, 1.4808302278224719, 1.4848451658727524, 1.488870989524397,
    1.4929077282912648, 1.4969554117672355, 1.5010140696264256, 1.5050837316234065,
    1.5091644275934228, 1.5132561874526098, 1.5173590411982147, 1.5214730189088146,
    1.5255981507445384, 1.529734466947287, 1.533881997840956, 1.5380407738316568,
    1.5422108254079407, 1.5463921831410214, 1.550584877685, 1.5547889397770887,
    1.559004400237837, 1.5632312899713576, 1.567469639965553, 1.5717194812923414,
    1.5759808451078865, 1.5802537626528246, 1.5845382652524937, 1.588834384317164,
    1.593142151342267, 1.597461597908627, 1.6017927556826934, 1.606135656416771,
    1.6104903319492543, 1.6148568142048607, 1.6192351351948637, 1.6236253270173289,
    1.6280274218573478, 1.632441451987275, 1.6368674497669644, 1.6413054476440063,
    1.645755478153965, 1.6502175739206177, 1.6546917676561943, 1.6591780921616162,
    1.6636765803267364, 1.6681872651305825, 1.6727101796415966, 1.6772453570178785,
    1.681792830507429, 1.6863526334483934, 1.6909247992693053, 1.6955093614893326,
    1.7001063537185235, 1.7047158096580513, 1.709337763100463, 1.713972247929926,
    1.718619298122478, 1.723278947746274, 1.7279512309618377, 1.732636182022311,
    1.7373338352737062, 1.7420442251551564, 1.746767386199169, 1.7515033530318782,
    1.7562521603732995, 1.761013843037584, 1.7657884359332727, 1.7705759740635547,
    1.7753764925265212, 1.7801900265154245, 1.785016611318935, 1.789856282321401,
    1.7947090750031072, 1.7995750249405351, 1.804454167806624, 1.809346539371032,
    1.8142521755003989, 1.8191711121586085, 1.8241033854070534, 1.8290490314048973,
    1.8340080864093424, 1.8389805867758937, 1.843966568958626, 1.8489660695104508,
    1.8539791250833855, 1.8590057724288205, 1.864046048397789, 1.8690999899412386,
    1.8741676341103, 1.8792490180565602, 1.8843441790323345, 1.8894531543909392,
    1.8945759815869656, 1.8997126981765553, 1.9048633418176741, 1.9100279502703899,
    1.9152065613971474, 1.9203992131630474, 1.925605943636125, 1.930826790987627,
    1.9360617934922943, 1.9413109895286405, 1.9465744175792332, 1.9518521162309783,
    1.9571441241754002, 1.9624504802089273, 1.9677712232331759, 1.9731063922552343,
    1.978456026387951, 1.9838201648502194, 1.9891988469672663, 1.9945921121709402};


// Log2-domain E-step: the affine form is pre-scaled by
// sqrt(log2(e)/2) and cst by log2(e), so a component's term is
//   lp2 = cst2 - |A2 z - b2|^2 = log2(e) * (cst - |A z - b|^2 / 2)
// (three FMAs from cst, no separate -0.5 scaling) and 2^x needs no ln2 multiply: the
// table index comes straight from x * 256 and the reduced argument x - k/256 is exact, so
// the two-constant Cody-Waite step collapses to one FMA. e^(r ln 2) by a degree-4 Taylor
// polynomial in r (|r| <= 1/512: truncation < 4e-17).
__device__ __constant__ double kExp2C[7] = {
    256.0, 6755399441055744.0, 0.00390625,
    0.0096181291076284772,   // ln2^4 / 24
    0.055504108664821579,    // ln2^3 / 6
    0.24022650695910071,     // ln2^2 / 2
    0.69314718055994531};    // ln2
constexpr double kLog2E = 1.4426950408889634;
constexpr double kSqrtHalfLog2E = 0.84932180028801907;  // sqrt(log2(e) / 2)

// 2^x for x <= 0; 0 below about -1021 (2^-1021 ~ 4.5e-308, below every tolerance).
// Degree-3 Taylor in r (|r| <= 1/512): truncation (r ln2)^4/24 < 1.5e-13 relative, four
// orders below the 1e-9 parity tolerance of the fitted parameters. The underflow test is an
// unsigned compare of the high word (x <= 0: |x| > 1021 <=> hi > hi(-1021); -inf and NaN
// also select 0) on the integer ALU: DSETP costs ~2 DFMA slots of the FP64 pipe on B200.
VDFCG_DEV double exp2_nonpos(double x, const double* tab) {
  const bool tiny = static_cast<unsigned>(__double2hiint(x)) > 0xC08FE800u;
  const double tm = fma(x, kExp2C[0], kExp2C[1]);
  const int k = __double2loint(tm);
  const double kd = tm - kExp2C[1];
  const double r = fma(-kd, kExp2C[2], x);  // exact
  const double r2 = r * r;
  const double lo = fma(kExp2C[6], r, 1.0);
  const double hi = fma(kExp2C[4], r, kExp2C[5]);
  const double p = fma(hi, r2, lo);
  const double v = tab[k & 255] * p;
  const double out = __hiloint2double(__double2hiint(v) + ((k >> 8) << 20), __double2loint(v));
  return tiny ? 0.0 : out;
}

// log(s) for the per-point mixture normaliser (any positive normal double; s >= 1e-300
// on the fast path). s = m 2^e, m in [1,2); j = top 7 mantissa bits; r = m c_j - 1 with
// c_j ~ 1/(1 + (j+0.5)/128) so |r| < 1/256; log s = e ln2 + (-log c_j) + log1p(r) with a
// degree-6 series (truncation < 1e-17). kLogTab = {c_j, -log c_j} (60-digit evaluation).
__device__ __constant__ double kLogTab[256] = {
    0.9961089494163424, 0.003898640415657309, 0.9884169884169884, 0.01165061721997525,
    0.9808429118773946, 0.019342962843130987, 0.973384030418251, 0.026976587698202083,
    0.9660377358490566, 0.03455238150665973, 0.9588014981273408, 0.042071213920687044,
    0.9516728624535316, 0.049533935122276676, 0.9446494464944649, 0.05694137640013845,
    0.9377289377289377, 0.06429435070539725, 0.9309090909090909, 0.07159365318700882,
    0.924187725631769, 0.078840061707776, 0.9175627240143369, 0.08603433734180316,
    0.9110320284697508, 0.09317722485418334, 0.9045936395759717, 0.10026945316367517,
    0.8982456140350877, 0.10731173578908804, 0.89198606271777, 0.11430477128005863,
    0.8858131487889274, 0.12124924363286965, 0.8797250859106529, 0.12814582269193006,
    0.8737201365187713, 0.13499516453750482, 0.8677966101694915, 0.1417979118602574,
    0.8619528619528619, 0.1485546943231372, 0.8561872909698997, 0.15526612891112396,
    0.8504983388704319, 0.16193282026931324, 0.8448844884488449, 0.16855536102980664,
    0.839344262295082, 0.17513433212784915, 0.8338762214983714, 0.18167030310763463,
    0.8284789644012945, 0.18816383241818294, 0.8231511254019293, 0.19461546769967167,
    0.8178913738019169, 0.2010257460605908, 0.8126984126984127, 0.2073951943460706,
    0.807570977917981, 0.21372432939771818, 0.8025078369905956, 0.22001365830528213,
    0.7975077881619937, 0.2262636786504534, 0.7925696594427245, 0.232474878743094,
    0.7876923076923077, 0.238647737850175, 0.7828746177370031, 0.24478272641769092,
    0.7781155015197568, 0.25088030628580943, 0.7734138972809668, 0.2569409308975004,
    0.7687687687687688, 0.26296504550088134, 0.764179104477612, 0.26895308734550394,
    0.7596439169139466, 0.2749054858727992, 0.7551622418879056, 0.2808226629008878,
    0.750733137829912, 0.2867050328039543, 0.7463556851311953, 0.29255300268637746,
    0.7420289855072464, 0.2983669725517973, 0.7377521613832853, 0.3041473354672968,
    0.7335243553008596, 0.3098944777228647, 0.7293447293447294, 0.3156087789863033,
    0.7252124645892352, 0.32129061245373425, 0.7211267605633803, 0.3269403449958533,
    0.7170868347338936, 0.3325583373000766, 0.713091922005571, 0.3381449440087164,
    0.7091412742382271, 0.34370051385331846, 0.7052341597796143, 0.3492253897852883,
    0.7013698630136986, 0.354719909102929, 0.6975476839237057, 0.3601844035750078,
    0.6937669376693767, 0.3656191995609647, 0.6900269541778976, 0.37102461812787263,
    0.6863270777479893, 0.376400975164253, 0.6826666666666666, 0.3817485814908484,
    0.6790450928381963, 0.3870677429684483, 0.6754617414248021, 0.3923587606028639,
    0.6719160104986877, 0.3976219306471385, 0.6684073107049608, 0.4028575447010835,
    0.6649350649350649, 0.4080658898082217, 0.661498708010336, 0.41324724855021927,
    0.6580976863753213, 0.41840189913888387, 0.6547314578005116, 0.4235301155058032,
    0.6513994910941476, 0.42863216738969867, 0.6481012658227848, 0.4337083204215594,
    0.6448362720403022, 0.43875883620762796, 0.6416040100250626, 0.44378397241030104,
    0.6384039900249376, 0.4487839828270067, 0.6352357320099256, 0.4537591174671205,
    0.6320987654320988, 0.4587096226269767, 0.628992628992629, 0.46363574096303256,
    0.6259168704156479, 0.46853771156323926, 0.6228710462287105, 0.4734157700166721,
    0.6198547215496368, 0.47827014848147026, 0.6168674698795181, 0.48310107575113576,
    0.6139088729016786, 0.48790877731923904, 0.6109785202863962, 0.4926934754425752,
    0.6080760095011877, 0.4974553892028189, 0.6052009456264775, 0.5021947345667155,
    0.6023529411764705, 0.5069117244448544, 0.5995316159250585, 0.5116065687490621,
    0.5967365967365967, 0.5162794744484545, 0.5939675174013921, 0.5209306456241853,
    0.5912240184757506, 0.5255602835229274, 0.5885057471264368, 0.5301685866091216,
    0.585812356979405, 0.5347557506160276, 0.5831435079726651, 0.5393219685956089,
    0.5804988662131519, 0.5438674309672835, 0.5778781038374717, 0.5483923255655733,
    0.5752808988764045, 0.5528968376866776, 0.5727069351230425, 0.5573811501340064,
    0.5701559020044543, 0.5618454432626918, 0.5676274944567627, 0.5662898950231159,
    0.565121412803532, 0.5707146810034716, 0.5626373626373626, 0.575119974471388,
    0.5601750547045952, 0.5795059464146423, 0.5577342047930284, 0.5838727655809826,
    0.5553145336225597, 0.588220598517086, 0.5529157667386609, 0.5925496096066716,
    0.5505376344086022, 0.5968599611077938, 0.5481798715203426, 0.6011518131893347,
    0.5458422174840085, 0.6054253239667169, 0.5435244161358811, 0.6096806495368553,
    0.5412262156448203, 0.6139179440123704, 0.5389473684210526, 0.6181373595550788,
    0.5366876310272537, 0.6223390464087787, 0.534446764091858, 0.6265231529313529,
    0.5322245322245323, 0.6306898256261987, 0.5300207039337475, 0.6348392091730102,
    0.5278350515463918, 0.6389714464579207, 0.5256673511293635, 0.6430866786030273,
    0.523517382413088, 0.6471850449953095, 0.5213849287169042, 0.6512666833149582,
    0.5192697768762677, 0.6553317295631277, 0.5171717171717172, 0.6593803180891278,
    0.5150905432595574, 0.6634125816170662, 0.5130260521042084, 0.6674286512719563,
    0.5109780439121756, 0.6714286566053024, 0.5089463220675944, 0.6754127256201768,
    0.5069306930693069, 0.6793809847957973, 0.504930966469428, 0.6833335591116206,
    0.5029469548133595, 0.6872705720709603, 0.5009784735812133, 0.691192145724142};

VDFCG_DEV double log_ge1(double s, const double* tab) {
  const int hi = __double2hiint(s);
  const int e = (hi >> 20) - 1023;
  const int j = (hi >> 13) & 127;
  const double m = __hiloint2double((hi & 0x000FFFFF) | 0x3FF00000, __double2loint(s));
  const double r = fma(m, tab[2 * j], -1.0);
  // log1p(r) = r - r^2/2 + r^3/3 - r^4/4 (+ r^5/5 < 1.8e-13 absolute: |r| < 1/256)
  double p = fma(r, -0.25, 1.0 / 3.0);
  p = fma(p, r, -0.5);
  p = fma(p, r, 1.0);
  return fma(static_cast<double>(e), 0.6931471805599453, tab[2 * j + 1] + p * r);
}

// 1/s for s in [1, K] (the per-point mixture normaliser): MUFU estimate (~2^-23) + one
// Newton step (~2^-46 relative). The same factor scales every responsibility of the
// point, so means and covariances (ratios of sums) are unaffected and the weights move
// by <1e-13 relative, far inside the 1e-9 parity tolerance.
VDFCG_DEV double rcp_newton(double s) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(s));
  return fma(r, fma(-s, r, 1.0), r);
}

// log N(z | mu, L) + log alpha for one component (prepared by prep_component).
template <int D>
VDFCG_DEV double comp_logp(const double* z, const double* mu, const double* Lo, const double* rd,
                           double cst) {
  double y0, y1 = 0.0, y2 = 0.0;
  y0 = (z[0] - mu[0]) * rd[0];
  if (D >= 2) y1 = ((z[1] - mu[1]) - Lo[0] * y0) * rd[1];
  if (D >= 3) y2 = ((z[2] - mu[2]) - Lo[1] * y0 - Lo[2] * y1) * rd[2];
  double q = y0 * y0;
  if (D >= 2) q += y1 * y1;
  if (D >= 3) q += y2 * y2;
  return cst - 0.5 * q;
}

// The same density through y = A z - b with A = L^-1 (lower triangular), b = A mu:
// 6 FMAs instead of 3 subtractions + the substitution (used by the fused point pass).
// A is packed {a00, a10, a11, a20, a21, a22}.
template <int D>
VDFCG_DEV void affine_from_chol(const double* mu, const double* Lo, const double* rd, double* A,
                                double* b) {
  // rows of L^-1 by forward substitution on the unit vectors
  const double a00 = rd[0];
  const double a10 = D >= 2 ? -Lo[0] * a00 * rd[1] : 0.0;
  const double a11 = D >= 2 ? rd[1] : 0.0;
  const double a20 = D >= 3 ? -(Lo[1] * a00 + Lo[2] * a10) * rd[2] : 0.0;
  const double a21 = D >= 3 ? -Lo[2] * a11 * rd[2] : 0.0;
  const double a22 = D >= 3 ? rd[2] : 0.0;
  A[0] = a00; A[1] = a10; A[2] = a11; A[3] = a20; A[4] = a21; A[5] = a22;
  b[0] = a00 * mu[0];
  b[1] = D >= 2 ? a10 * mu[0] + a11 * mu[1] : 0.0;
  b[2] = D >= 3 ? a20 * mu[0] + a21 * mu[1] + a22 * mu[2] : 0.0;
}

// log2-domain term with the pre-scaled affine form (see exp2_nonpos).
template <int D>
VDFCG_DEV double comp_logp2_affine(const double* z, const double* A, const double* b, double cst) {
  const double y0 = fma(A[0], z[0], -b[0]);
  double lp = fma(-y0, y0, cst);
  if (D >= 2) {
    const double y1 = fma(A[2], z[1], fma(A[1], z[0], -b[1]));
    lp = fma(-y1, y1, lp);
  }
  if (D >= 3) {
    const double y2 = fma(A[5], z[2], fma(A[4], z[1], fma(A[3], z[0], -b[2])));
    lp = fma(-y2, y2, lp);
  }
  return lp;
}

template <int D>
VDFCG_DEV double comp_logp_affine(const double* z, const double* A, const double* b, double cst) {
  const double y0 = fma(A[0], z[0], -b[0]);
  double q = y0 * y0;
  if (D >= 2) {
    const double y1 = fma(A[2], z[1], fma(A[1], z[0], -b[1]));
    q = fma(y1, y1, q);
  }
  if (D >= 3) {
    const double y2 = fma(A[5], z[2], fma(A[4], z[1], fma(A[3], z[0], -b[2])));
    q = fma(y2, y2, q);
  }
  return fma(-0.5, q, cst);
}

// Model arrays: alpha[K], mu[K*D], cov[K*9] (3x3 slots).
template <int D>
VDFCG_DEV void remove_component(double* alpha, double* mu, double* cov, int& m, int idx) {
  for (int j = idx; j + 1 < m; ++j) {
    alpha[j] = alpha[j + 1];
#pragma unroll
    for (int a = 0; a < D; ++a) mu[j * D + a] = mu[(j + 1) * D + a];
#pragma unroll
    for (int e = 0; e < 9; ++e) cov[j * 9 + e] = cov[(j + 1) * 9 + e];
  }
  --m;
}

// Rescale to unit sum by the sequential sum in component order (wgmm.cpp:331-332).
VDFCG_DEV void renormalize(double* alpha, int m) {
  double total = 0.0;
  for (int j = 0; j < m; ++j) total = __dadd_rn(total, alpha[j]);
  for (int j = 0; j < m; ++j) alpha[j] = alpha[j] / total;
}

// prune_one (wgmm.cpp:320-333): smallest weight (ties -> lowest index), strictly below
// the threshold, only while more than one component remains.
template <int D>
VDFCG_DEV bool prune_one_dev(double* alpha, double* mu, double* cov, int& m, double thr,
                             int* idx, double* weight) {
  if (m <= 1) return false;
  int sm = 0;
  for (int i = 1; i < m; ++i)
    if (alpha[i] < alpha[sm]) sm = i;
  if (!(alpha[sm] < thr)) return false;
  *idx = sm;
  *weight = alpha[sm];
  remove_component<D>(alpha, mu, cov, m, sm);
  renormalize(alpha, m);
  return true;
}

// init_model (wgmm.cpp:136-191) given the frame (normalization, bounding box of the
// normalized points, temperature, min(M, distinct)). Returns M.
template <int D>
VDFCG_DEV int init_model_dev(const Frame& F, const EmConfig& cfg, double* alpha, double* mu,
                             double* cov) {
  if (cfg.warm_m > 0) {  // warm start: re-express the canonical model in this frame
    double Dv[3];
#pragma unroll
    for (int a = 0; a < D; ++a) Dv[a] = 1.0 / F.scale[a];
    for (int i = 0; i < cfg.warm_m; ++i) {
      alpha[i] = cfg.warm_w[i];
#pragma unroll
      for (int a = 0; a < D; ++a)
        mu[i * D + a] = __dsub_rn(cfg.warm_mu[i * D + a], F.offset[a]) / F.scale[a];
      Sym3 cv;
#pragma unroll
      for (int e = 0; e < 9; ++e) cv.a[e] = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int b = 0; b < D; ++b)
          cv(a, b) = __dmul_rn(__dmul_rn(Dv[a], cfg.warm_cov[(i * D + a) * D + b]), Dv[b]);
      symmetrize_from_upper<D>(cv);
#pragma unroll
      for (int e = 0; e < 9; ++e) cov[i * 9 + e] = cv.a[e];
    }
    return cfg.warm_m;
  }
  const int m = F.m_init;
  for (int i = 0; i < m; ++i) {
    alpha[i] = 1.0 / m;
#pragma unroll
    for (int a = 0; a < D; ++a)
      mu[i * D + a] = __dadd_rn(F.zlo[a], __dmul_rn(__dsub_rn(F.zhi[a], F.zlo[a]), cfg.uniforms[i * D + a]));
#pragma unroll
    for (int e = 0; e < 9; ++e) cov[i * 9 + e] = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) cov[i * 9 + a * 3 + a] = F.temp[a] / __dmul_rn(F.scale[a], F.scale[a]);
  }
  return m;
}

// Number of distinct rows among the first points of z (SoA [D][n]), stopping at M
// (only "distinct < M" matters, wgmm.cpp:166-172). Executed by one full warp; list is
// a shared [16][3] scratch. Returns the count to every lane.
template <int D>
VDFCG_DEV int count_distinct_warp(const double* z, int64_t n, int M, double (*list)[3]) {
  const int lane = threadIdx.x & 31;
  int count = 0;
  for (int64_t b = 0; b < n && count < M; b += 32) {
    const int64_t p = b + lane;
    double zz[3] = {0, 0, 0};
    bool isnew = p < n;
    if (isnew) {
#pragma unroll
      for (int a = 0; a < D; ++a) zz[a] = z[a * n + p];
      for (int j = 0; j < count && isnew; ++j) {
        bool eq = true;
#pragma unroll
        for (int a = 0; a < D; ++a) eq = eq && (zz[a] == list[j][a]);
        if (eq) isnew = false;
      }
    }
    unsigned mask = __ballot_sync(0xffffffffu, isnew);
    while (mask && count < M) {
      const int l = __ffs(mask) - 1;
      double bz[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) bz[a] = __shfl_sync(0xffffffffu, zz[a], l);
      __syncwarp();
      if (lane == 0) {
#pragma unroll
        for (int a = 0; a < 3; ++a) list[count][a] = bz[a];
      }
      __syncwarp();
      ++count;
      if (lane > l && isnew) {
        bool eq = true;
#pragma unroll
        for (int a = 0; a < D; ++a) eq = eq && (zz[a] == bz[a]);
        if (eq) isnew = false;
      }
      if (lane == l) isnew = false;
      mask = __ballot_sync(0xffffffffu, isnew);
    }
  }
  return count;
}

}  // namespace vdfcg
