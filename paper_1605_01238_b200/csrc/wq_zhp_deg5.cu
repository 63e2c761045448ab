// wq_zhp_deg5.cu -- instantiation of the ZHP line kernel for p = 5 (one TU per degree: parallel builds)
#include "wq_zhp.cuh"
WQ_ZHP_DEG_DEF(5)
