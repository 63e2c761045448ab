// wq_zhp_deg10.cu -- instantiation of the ZHP line kernel for p = 10 (one TU per degree: parallel builds)
#include "wq_zhp.cuh"
WQ_ZHP_DEG_DEF(10)
