/*
 * ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.h). Precision-generic body of
 * the forward pass, included twice by forward.c: REAL=double (the parity
 * reference, with the absolute-value "mag" forward) and REAL=float (the CPU
 * baseline). Operator order follows work() (proj/src/model_zoo.cpp:177-245):
 * DenseFC, EmbeddingLookup+Pooling (Sum | Concat | AttentionFC |
 * AttentionRNN), Interaction, PredictFC; the predict input is laid out as
 * predict_input_dim (model_zoo.cpp:113-137) counts it:
 *   [dense_out | sparse_out | interaction pairs].
 */

/* Y[S][out] = act(A[S][in] W^T + b); YM = sum |W| AM + |b| (error scale). */
static void FN(fc)(const REAL* A, const REAL* AM, int64_t S, int64_t in, int64_t lda,
                   const float* W, const float* b, int64_t out, int relu, REAL* Y,
                   int64_t ldy, REAL* YM) {
#ifdef FAST_FC
  /* fp32 CPU-baseline path (no error scale): 4 items per pass over a weight
   * row, the dot vectorised (SIMD reduction: a different summation order than
   * the fp64 parity path, which is not used for timing). */
  if (!YM) {
    for (int64_t it0 = 0; it0 < S; it0 += 4) {
      const int64_t nr = S - it0 < 4 ? S - it0 : 4;
      const REAL* x0 = A + it0 * lda;
      const REAL* x1 = nr > 1 ? x0 + lda : x0;
      const REAL* x2 = nr > 2 ? x0 + 2 * lda : x0;
      const REAL* x3 = nr > 3 ? x0 + 3 * lda : x0;
      for (int64_t o = 0; o < out; ++o) {
        const float* w = W + o * in;
        REAL a0 = 0, a1 = 0, a2 = 0, a3 = 0;
#pragma omp simd reduction(+ : a0, a1, a2, a3)
        for (int64_t i = 0; i < in; ++i) {
          a0 += w[i] * x0[i];
          a1 += w[i] * x1[i];
          a2 += w[i] * x2[i];
          a3 += w[i] * x3[i];
        }
        const REAL r[4] = {a0, a1, a2, a3};
        for (int64_t k = 0; k < nr; ++k) {
          REAL y = r[k] + (REAL)b[o];
          if (relu && y < 0) y = 0;
          Y[(it0 + k) * ldy + o] = y;
        }
      }
    }
    return;
  }
#endif
  for (int64_t o = 0; o < out; ++o) {
    const float* w = W + o * in;
    for (int64_t it = 0; it < S; ++it) {
      const REAL* x = A + it * lda;
      REAL acc = 0;
      for (int64_t i = 0; i < in; ++i) acc += (REAL)w[i] * x[i];
      REAL y = acc + (REAL)b[o];
      if (relu && y < 0) y = 0;
      Y[it * ldy + o] = y;
      if (YM) {
        const REAL* xm = AM + it * lda;
        REAL m = 0;
        for (int64_t i = 0; i < in; ++i) m += (REAL)fabs((double)w[i]) * xm[i];
        YM[it * ldy + o] = m + (REAL)fabs((double)b[o]);
      }
    }
  }
}

static REAL FN(sigm)(REAL x) { return (REAL)1 / ((REAL)1 + (REAL)exp(-(double)x)); }

/* One GRU / AUGRU sequence; writes h[H] (and hm[H]). */
static int FN(gru_seq)(const or_state* s, int64_t t, const int64_t* bidx, REAL* h, REAL* hm,
                       REAL* work) {
  const int64_t D = s->m.D, H = s->m.hidden, L = s->m.L, H3 = 3 * H;
  const float* wih = s->wih + t * H3 * D;
  const float* whh = s->whh + t * H3 * H;
  const float* bih = s->bih + t * H3;
  const float* bhh = s->bhh + t * H3;
  REAL* x = work;            /* D */
  REAL* gi = x + D;          /* 3H */
  REAL* gh = gi + H3;        /* 3H */
  REAL* ua = gh + H3;        /* D */
  REAL* hn = ua + D;         /* H */
  float row[256];
  for (int64_t j = 0; j < H; ++j) { h[j] = 0; if (hm) hm[j] = 0; }
  for (int64_t l = 0; l < L; ++l) {
    const float* e = or_row(s, t, bidx[l], row);
    if (!e) return -7;
    for (int64_t c = 0; c < D; ++c) x[c] = e[c];
    if (s->augru && l == 0) { /* ua = W_a^T x_0 */
      const float* wa = s->watt + t * D * D;
      for (int64_t c = 0; c < D; ++c) {
        REAL a = 0;
        for (int64_t i = 0; i < D; ++i) a += x[i] * (REAL)wa[i * D + c];
        ua[c] = a;
      }
    }
    for (int64_t r = 0; r < H3; ++r) {
      REAL a = 0, g = 0;
      for (int64_t c = 0; c < D; ++c) a += (REAL)wih[r * D + c] * x[c];
      for (int64_t k = 0; k < H; ++k) g += (REAL)whh[r * H + k] * h[k];
      gi[r] = a + (REAL)bih[r];
      gh[r] = g + (REAL)bhh[r];
    }
    REAL att = 1;
    if (s->augru) {
      REAL sc = 0;
      for (int64_t c = 0; c < D; ++c) sc += ua[c] * x[c];
      att = FN(sigm)(sc);
    }
    for (int64_t j = 0; j < H; ++j) {
      const REAL pr = gi[j] + gh[j], pz = gi[H + j] + gh[H + j];
      const REAL r = FN(sigm)(pr), z = FN(sigm)(pz);
      const REAL pn = gi[2 * H + j] + r * gh[2 * H + j];
      const REAL n = (REAL)tanh((double)pn);
      REAL hv;
      if (s->augru) {
        const REAL u = att * ((REAL)1 - z);
        hv = ((REAL)1 - u) * h[j] + u * n;
      } else {
        hv = ((REAL)1 - z) * n + z * h[j];
      }
      hn[j] = hv;
    }
    /* Error scale of the hidden state: h is a convex mix of tanh outputs,
     * bounded in (-1, 1); carrying |terms| through the recurrence would grow
     * geometrically with the sequence length, so the scale is the unit scale
     * of h itself. */
    for (int64_t j = 0; j < H; ++j) { h[j] = hn[j]; if (hm) hm[j] = (REAL)1; }
  }
  return 0;
}

static int FN(forward)(const or_state* s, int64_t S, const float* dense, const int64_t* idx,
                       REAL* out, REAL* mag, REAL* pooled, REAL* pooled_mag) {
  const or_model* m = &s->m;
  const int64_t T = m->T, L = m->L, D = m->D;
  const int64_t p_in = s->p_in, dout = s->dense_out;
  const int want = mag != NULL;
  int rc = 0;
  REAL* X = (REAL*)calloc((size_t)(S * p_in), sizeof(REAL));
  REAL* XM = want ? (REAL*)calloc((size_t)(S * p_in), sizeof(REAL)) : NULL;
  float row[256];
  if (!X || (want && !XM)) { free(X); free(XM); return -6; }

  /* ---- DenseFC (ReLU after every layer) or raw dense features ---- */
  if (m->has_dense_fc) {
    int64_t in = m->dense_in;
    REAL* A = (REAL*)calloc((size_t)(S * (in > 0 ? in : 1)), sizeof(REAL));
    REAL* AM = want ? (REAL*)calloc((size_t)(S * (in > 0 ? in : 1)), sizeof(REAL)) : NULL;
    for (int64_t i = 0; i < S * in; ++i) {
      A[i] = dense[i];
      if (AM) AM[i] = (REAL)fabs((double)dense[i]);
    }
    for (int l = 0; l < m->dense_fc.n; ++l) {
      const int64_t o = m->dense_fc.dims[l];
      REAL* B = (REAL*)calloc((size_t)(S * o), sizeof(REAL));
      REAL* BM = want ? (REAL*)calloc((size_t)(S * o), sizeof(REAL)) : NULL;
      FN(fc)(A, AM, S, in, in, s->dW[l], s->db[l], o, 1, B, o, BM);
      free(A); free(AM);
      A = B; AM = BM; in = o;
    }
    for (int64_t it = 0; it < S; ++it)
      for (int64_t c = 0; c < dout; ++c) {
        X[it * p_in + c] = A[it * dout + c];
        if (XM) XM[it * p_in + c] = AM[it * dout + c];
      }
    free(A); free(AM);
  } else {
    for (int64_t it = 0; it < S; ++it)
      for (int64_t c = 0; c < m->dense_in; ++c) {
        X[it * p_in + c] = dense[it * m->dense_in + c];
        if (XM) XM[it * p_in + c] = (REAL)fabs((double)dense[it * m->dense_in + c]);
      }
  }

  /* ---- EmbeddingLookup + Pooling ---- */
  const int64_t pdim = s->pooled_dim;
  if (T > 0) {
    if (m->pooling == 0) { /* Sum, then Interaction */
      REAL* P = (REAL*)calloc((size_t)(T * D), sizeof(REAL));
      REAL* PM = (REAL*)calloc((size_t)(T * D), sizeof(REAL));
      for (int64_t it = 0; it < S && !rc; ++it) {
        for (int64_t t = 0; t < T && !rc; ++t) {
          REAL* p = P + t * D;
          REAL* pm = PM + t * D;
          for (int64_t c = 0; c < D; ++c) { p[c] = 0; pm[c] = 0; }
          for (int64_t l = 0; l < L; ++l) {
            const float* e = or_row(s, t, idx[(it * T + t) * L + l], row);
            if (!e) { rc = -7; break; }
            if (want) {
              for (int64_t c = 0; c < D; ++c) {
                p[c] += e[c];
                pm[c] += (REAL)fabs((double)e[c]);
              }
            } else {
              for (int64_t c = 0; c < D; ++c) p[c] += e[c];
            }
          }
        }
        if (pooled)
          for (int64_t k = 0; k < T * D; ++k) {
            pooled[it * pdim + k] = P[k];
            if (pooled_mag) pooled_mag[it * pdim + k] = PM[k];
          }
        REAL* x = X + it * p_in;
        REAL* xm = XM ? XM + it * p_in : NULL;
        for (int64_t c = 0; c < D; ++c) { /* summed embedding (D9) */
          REAL a = 0, am = 0;
          for (int64_t t = 0; t < T; ++t) { a += P[t * D + c]; am += PM[t * D + c]; }
          x[dout + c] = a;
          if (xm) xm[dout + c] = am;
        }
        if (m->has_dense_fc) { /* pairs over v0 = dense_out, v_t = pooled */
          int64_t p = 0;
          for (int64_t i = 1; i <= T; ++i)
            for (int64_t j = 0; j < i; ++j, ++p) {
              const REAL* vi = P + (i - 1) * D;
              const REAL* vim = PM + (i - 1) * D;
              const REAL* vj = j == 0 ? x : P + (j - 1) * D;
              const REAL* vjm = j == 0 ? xm : PM + (j - 1) * D;
              REAL d = 0, dm = 0;
              for (int64_t c = 0; c < D; ++c) {
                d += vi[c] * vj[c];
                if (xm) dm += vim[c] * (REAL)fabs((double)vj[c]) + (REAL)fabs((double)vi[c]) * vjm[c];
              }
              x[dout + D + p] = d;
              if (xm) xm[dout + D + p] = dm;
            }
        }
      }
      free(P); free(PM);
    } else if (m->pooling == 1) { /* Concat */
      for (int64_t it = 0; it < S && !rc; ++it)
        for (int64_t k = 0; k < T * L; ++k) {
          const float* e = or_row(s, k / L, idx[it * T * L + k], row);
          if (!e) { rc = -7; break; }
          for (int64_t c = 0; c < D; ++c) {
            X[it * p_in + dout + k * D + c] = e[c];
            if (XM) XM[it * p_in + dout + k * D + c] = (REAL)fabs((double)e[c]);
          }
        }
    } else if (m->pooling == 2) { /* AttentionFC: a_l = sig(q^T W_t e_l), pooled = sum a_l e_l */
      REAL* q = (REAL*)malloc(sizeof(REAL) * (size_t)D);
      REAL* we = (REAL*)malloc(sizeof(REAL) * (size_t)D);
      for (int64_t it = 0; it < S && !rc; ++it)
        for (int64_t t = 0; t < T && !rc; ++t) {
          const int64_t* b = idx + (it * T + t) * L;
          const float* W = s->att + t * D * D;
          const float* e0 = or_row(s, t, b[0], row);
          if (!e0) { rc = -7; break; }
          for (int64_t c = 0; c < D; ++c) q[c] = e0[c];
          REAL* o = X + it * p_in + dout + t * D;
          REAL* om = XM ? XM + it * p_in + dout + t * D : NULL;
          for (int64_t c = 0; c < D; ++c) { o[c] = 0; if (om) om[c] = 0; }
          for (int64_t l = 0; l < L; ++l) {
            const float* e = or_row(s, t, b[l], row);
            if (!e) { rc = -7; break; }
            REAL sc = 0, scm = 0;
            for (int64_t i = 0; i < D; ++i) {
              REAL a = 0, am = 0;
              for (int64_t j = 0; j < D; ++j) {
                a += (REAL)W[i * D + j] * (REAL)e[j];
                am += (REAL)fabs((double)W[i * D + j]) * (REAL)fabs((double)e[j]);
              }
              sc += q[i] * a;
              scm += (REAL)fabs((double)q[i]) * am;
            }
            const REAL a = FN(sigm)(sc);                 /* activation-unit weight */
            const REAL am = (REAL)0.25 * scm + a;
            for (int64_t c = 0; c < D; ++c) {
              o[c] += a * (REAL)e[c];
              if (om) om[c] += am * (REAL)fabs((double)e[c]);
            }
          }
        }
      free(q); free(we);
    } else { /* AttentionRNN */
      const int64_t H = m->hidden;
      REAL* work = (REAL*)malloc(sizeof(REAL) * (size_t)(4 * D + 14 * H + 16));
      REAL* hm = want ? (REAL*)malloc(sizeof(REAL) * (size_t)H) : NULL;
      REAL* h = (REAL*)malloc(sizeof(REAL) * (size_t)H);
      for (int64_t it = 0; it < S && !rc; ++it)
        for (int64_t t = 0; t < T && !rc; ++t) {
          rc = FN(gru_seq)(s, t, idx + (it * T + t) * L, h, hm, work);
          for (int64_t j = 0; j < H; ++j) {
            X[it * p_in + dout + t * H + j] = h[j];
            if (XM) XM[it * p_in + dout + t * H + j] = hm[j];
          }
        }
      free(work); free(hm); free(h);
    }
    if (pooled && m->pooling != 0)
      for (int64_t it = 0; it < S; ++it)
        for (int64_t k = 0; k < pdim; ++k) {
          pooled[it * pdim + k] = X[it * p_in + dout + k];
          if (pooled_mag) pooled_mag[it * pdim + k] = XM ? XM[it * p_in + dout + k] : 0;
        }
  }

  /* ---- PredictFC: N parallel stacks, ReLU on hidden layers ---- */
  const int64_t odim = m->predict_fc.dims[m->predict_fc.n - 1];
  const int64_t ow = m->stacks * odim;
  for (int64_t z = 0; z < m->stacks && !rc; ++z) {
    const REAL* A = X;
    const REAL* AM = XM;
    int64_t in = p_in;
    REAL* bufs[2] = {NULL, NULL};
    REAL* mbufs[2] = {NULL, NULL};
    for (int l = 0; l < m->predict_fc.n; ++l) {
      const int64_t o = m->predict_fc.dims[l];
      const int last = l + 1 == m->predict_fc.n;
      REAL* B = (REAL*)calloc((size_t)(S * o), sizeof(REAL));
      REAL* BM = want ? (REAL*)calloc((size_t)(S * o), sizeof(REAL)) : NULL;
      FN(fc)(A, AM, S, in, in, s->pW[l] + z * o * in, s->pb[l] + z * o, o, !last, B, o, BM);
      free(bufs[l & 1]); free(mbufs[l & 1]);
      bufs[l & 1] = B; mbufs[l & 1] = BM;
      A = B; AM = BM; in = o;
    }
    for (int64_t it = 0; it < S; ++it)
      for (int64_t c = 0; c < odim; ++c) {
        out[it * ow + z * odim + c] = A[it * odim + c];
        if (mag) mag[it * ow + z * odim + c] = AM[it * odim + c];
      }
    free(bufs[0]); free(bufs[1]); free(mbufs[0]); free(mbufs[1]);
  }
  free(X); free(XM);
  return rc;
}
