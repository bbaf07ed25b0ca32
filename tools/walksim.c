// walksim.c -- CPU model of the lockstep in-block walk schedule (tuning tool,
// not part of the product).  Reads a u8 D8 raster, cuts it into BR x BC
// blocks, and counts warp iterations of the walk loop under several
// scheduling policies, so lane efficiency can be compared before a kernel
// is written.
//   gcc -O2 -o /tmp/walksim tools/walksim.c && /tmp/walksim dirs.u8 H W BR BC L policy stopx
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static const int DX[9] = {0, 0, 1, 1, 1, 0, -1, -1, -1};
static const int DY[9] = {0, -1, -1, 0, 1, 1, 1, 0, -1};

int main(int argc, char** argv) {
  if (argc < 9) { fprintf(stderr, "usage\n"); return 1; }
  const char* fn = argv[1];
  int H = atoi(argv[2]), W = atoi(argv[3]), BR = atoi(argv[4]), BC = atoi(argv[5]), L = atoi(argv[6]);
  int policy = atoi(argv[7]), stopx = atoi(argv[8]);
  int steal_min = argc > 9 ? atoi(argv[9]) : 4;
  uint8_t* d = malloc((size_t)H * W);
  FILE* f = fopen(fn, "rb");
  if (fread(d, 1, (size_t)H * W, f) != (size_t)H * W) return 2;
  fclose(f);
  int BN = BR * BC;
  int* succ = malloc(sizeof(int) * BN);
  int* cnt = malloc(sizeof(int) * BN);
  int* pend = malloc(sizeof(int) * BN);
  int* srcq = malloc(sizeof(int) * BN);
  int* lane_c = malloc(sizeof(int) * L);
  int* lane_live = malloc(sizeof(int) * L);
  int* rowq = malloc(sizeof(int) * BN);  // per-lane source lists
  int* rowh = malloc(sizeof(int) * L);
  int* rown = malloc(sizeof(int) * L);
  long long tot_iter = 0, tot_cells = 0, tot_busy = 0, nblk = 0, tot_src = 0, max_iter = 0;
  long long tot_junc = 0;
  for (int by = 0; by + BR <= H; by += BR)
    for (int bx = 0; bx + BC <= W; bx += BC) {
      int ndata = 0;
      for (int i = 0; i < BN; ++i) { cnt[i] = 0; succ[i] = -2; }
      for (int ly = 0; ly < BR; ++ly)
        for (int lx = 0; lx < BC; ++lx) {
          int i = ly * BC + lx;
          int c = d[(size_t)(by + ly) * W + bx + lx];
          if (c == 255) { succ[i] = -3; continue; }
          ++ndata;
          succ[i] = -1;
          if (c >= 1 && c <= 8) {
            int ty = ly + DY[c], tx = lx + DX[c];
            if (ty >= 0 && ty < BR && tx >= 0 && tx < BC && d[(size_t)(by + ty) * W + bx + tx] != 255)
              succ[i] = ty * BC + tx;
          }
        }
      for (int i = 0; i < BN; ++i)
        if (succ[i] >= 0) cnt[succ[i]]++;
      int ns = 0;
      for (int i = 0; i < BN; ++i) {
        pend[i] = cnt[i];
        if (succ[i] >= -1 && cnt[i] == 0) srcq[ns++] = i;
        if (cnt[i] >= 2) tot_junc++;
      }
      // per-lane lists: lane = row % L (rows of the block)
      for (int l = 0; l < L; ++l) { rowh[l] = 0; rown[l] = 0; }
      int per = BN / L;  // capacity per lane
      for (int k = 0; k < ns; ++k) {
        int l = (srcq[k] / BC) % L;
        rowq[l * per + rown[l]++] = srcq[k];
      }
      if (policy == 2) {  // FIFO Kahn: each iteration pops min(L, ready) cells
        int* q = malloc(sizeof(int) * (BN + 1));
        int h0 = 0, t0 = 0;
        for (int k = 0; k < ns; ++k) q[t0++] = srcq[k];
        long long it2 = 0;
        while (h0 < t0) {
          int n = t0 - h0 < L ? t0 - h0 : L;
          int tt = t0;
          for (int k = 0; k < n; ++k) {
            int c = q[h0 + k];
            int t = succ[c];
            if (t >= 0 && --pend[t] == 0) q[tt++] = t;
          }
          h0 += n; t0 = tt; ++it2;
          tot_busy += n;
        }
        free(q);
        tot_iter += it2;
        if (it2 > max_iter) max_iter = it2;
        tot_cells += BN; tot_src += ns; nblk++;
        continue;
      }
      int qh = 0;
      for (int l = 0; l < L; ++l) lane_live[l] = 0;
      long long it = 0, retired = 0;
      for (;;) {
        // refill
        int nidle = 0, any_src = 0;
        for (int l = 0; l < L; ++l) {
          if (lane_live[l]) continue;
          int got = -1;
          if (policy == 0) { if (qh < ns) got = srcq[qh++]; }
          else if (rowh[l] < rown[l]) got = rowq[l * per + rowh[l]++];
          if (got >= 0) { lane_c[l] = got; lane_live[l] = 1; retired++; }
        }
        for (int l = 0; l < L; ++l) { if (!lane_live[l]) nidle++; if (rowh[l] < rown[l]) any_src = 1; }
        if (policy == 0) any_src = qh < ns;
        if (nidle == L && !any_src) break;
        if (policy == 1 && nidle >= steal_min) {
          // q-th rich lane gives its last source to the q-th idle lane
          int rich[64], nr = 0, idl[64], ni = 0;
          for (int l = 0; l < L; ++l) { if (rowh[l] < rown[l]) rich[nr++] = l; if (!lane_live[l]) idl[ni++] = l; }
          for (int k = 0; k < nr && k < ni; ++k) {
            int r = rich[k];
            int got = rowq[r * per + --rown[r]];
            lane_c[idl[k]] = got; lane_live[idl[k]] = 1; retired++;
          }
        }
        ++it;
        for (int l = 0; l < L; ++l) {
          if (!lane_live[l]) continue;
          tot_busy++;
          int c = lane_c[l];
          int t = succ[c];
          if (t < 0) { lane_live[l] = 0; continue; }  // stop (extra iteration)
          if (cnt[t] >= 2) {
            if (--pend[t] > 0) { lane_live[l] = 0; continue; }
          }
          retired++;
          lane_c[l] = t;
          if (!stopx && succ[t] < 0) lane_live[l] = 0;
        }
      }
      if (retired != ndata) { fprintf(stderr, "mismatch %lld %d\n", retired, ndata); }
      tot_iter += it;
      if (it > max_iter) max_iter = it;
      tot_cells += BN;
      tot_src += ns;
      nblk++;
    }
  printf("BR=%d BC=%d L=%d policy=%d stopx=%d steal=%d: blocks %lld  iters/block %.1f (max %lld)  cells/iter %.2f  "
         "lane-eff %.3f  sources/block %.1f  junctions/cell %.3f\n",
         BR, BC, L, policy, stopx, steal_min, nblk, (double)tot_iter / nblk, max_iter,
         (double)tot_cells / tot_iter, (double)tot_busy / (tot_iter * (double)L), (double)tot_src / nblk,
         (double)tot_junc / tot_cells);
  return 0;
}
